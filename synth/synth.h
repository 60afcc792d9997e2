/*
 * synth.h — seeded synthetic-input generator for the ARA hot path.
 *
 * This module holds NO arithmetic of the method (no lookups, no financial
 * terms, no sums of losses, no metrics).  It only draws the *inputs* the
 * paper's §IV-A describes:
 *   - a Year Event Table (Eq. 1): trials of event ids, 800-1500
 *     events per trial drawn from a global catalogue;
 *   - Event Loss Tables (Eq. 2): per-ELT sparse (event, loss) lists,
 *     10k-30k losses per ELT typical.
 * Both the oracle side (tests/, bench cpu_baseline) and the CUDA side (bench,
 * parity tests) consume these arrays as plain data; neither imports the other.
 *
 * The generator is counter-based (splitmix64 keyed by (seed, stream, index)),
 * so any trial or any ELT can be regenerated independently of the rest — which
 * is what lets the full-size parity tests recompute sampled trials on the CPU.
 */
#ifndef ARA_SYNTH_H
#define ARA_SYNTH_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Raw 64-bit counter-based draw: u64(seed, stream, index). */
uint64_t synth_u64(uint64_t seed, uint64_t stream, uint64_t index);

/* Events per trial n_t ~ U{nmin..nmax} for trials [first, first+n). */
void synth_trial_counts(uint64_t seed, uint64_t first, uint64_t n,
                        uint32_t nmin, uint32_t nmax, uint32_t* counts);

/* Global index of the first event of trial `first` (= sum of n_i, i < first). */
uint64_t synth_event_base(uint64_t seed, uint64_t first, uint32_t nmin, uint32_t nmax);

/* CSR offsets for trials [first, first+n): offsets[0] = 0, offsets[i+1] =
 * offsets[i] + n_{first+i}.  Returns total events. */
uint64_t synth_yet_offsets(uint64_t seed, uint64_t first, uint64_t n,
                           uint32_t nmin, uint32_t nmax, uint64_t* offsets);

/* Event ids for global event indices [begin, begin+n): uniform on [1, catalog]
 * (the "uniform" id distribution; pessimistic for L2).  Multi-threaded. */
void synth_yet_events(uint64_t seed, uint32_t catalog, uint64_t begin, uint64_t n,
                      uint32_t* ids, int nthreads);

/* Timestamps in [0,1) for one trial of n events, ascending (Eq. 1 ordering).
 * Not consumed by the hot path (reading A6). */
void synth_trial_timestamps(uint64_t seed, uint64_t trial, uint32_t n, double* ts);

/* ELT j: Bernoulli(rho) membership for each event e in [1, catalog].
 * Returns the number of (event, loss) records. */
uint64_t synth_elt_count(uint64_t seed, uint32_t j, uint32_t catalog, double rho);

/* ELT j records, ascending event id.  Loss ~ LogNormal(mu, sigma).  If
 * int_cap > 0 the loss is floor()-ed and clamped to int_cap - 1 (integer-valued
 * variant that makes all fp64 sums exact). */
void synth_elt_fill(uint64_t seed, uint32_t j, uint32_t catalog, double rho,
                    double mu, double sigma, double int_cap,
                    uint32_t* event_ids, double* losses);

#ifdef __cplusplus
}
#endif
#endif
