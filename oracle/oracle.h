/*
 * oracle.h — plain, slow, single-threaded CPU oracle for Aggregate Risk Analysis.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product path (paper_1606_04473_b200/) never links, imports or calls it, and
 * this file shares no code, header, table or constant with it.
 *
 * What it computes (PAPER.md = P, SPEC.md = S, DESIGN.md "Readings" = A#):
 *   Alg. 1  for each layer, for each trial  -> YLT
 *   Alg. 3  for each event, for each ELT of the layer:
 *                         lookup, apply I, sum;
 *                       occurrence terms per event, accumulate,
 *                       aggregate terms per trial
 *   PML / TVaR  as defined in S:203-220 (reading A9/A10)
 * IEEE fp64, round-to-nearest, compiled with -ffp-contract=off, no fast-math.
 *
 * Parity pins: every function below is pinned by a `-m "not gpu"` test in
 * tests/test_oracle_pins.py (worked examples, closed forms, invariants, brute
 * force).  No function is "parity unpinned".
 */
#ifndef ARA_ORACLE_H
#define ARA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { ORACLE_LOOKUP_MAP = 0, ORACLE_LOOKUP_DENSE = 1 };

/* The ELT set, Eq. 2: ELT j holds records
 * (event_ids[k], losses[k]) for k in [offsets[j], offsets[j+1]), event ids
 * strictly ascending within each ELT. */
typedef struct {
    uint32_t n_elts;
    const uint64_t* offsets;
    const uint32_t* event_ids;
    const double* losses;
} oracle_elts;

/* A layer L = (E, T), Eq. 3: its ELTs in listed order plus the
 * four layer terms of P:373/P:375. */
typedef struct {
    uint32_t n_elts;
    const uint32_t* elts;
    double occ_retention, occ_limit, agg_retention, agg_limit;
} oracle_layer;

/* l = min(max(l - R, 0), Lim): the term formula of P:373 / P:375 with the
 * missing max argument read as 0 (reading A1). */
double oracle_apply_terms(double loss, double retention, double limit);

/* Map-semantics lookup of event e in ELT j; a missing event gives 0 (A4).
 * Binary search over the ascending record list. */
double oracle_lookup_map(const oracle_elts* elts, uint32_t j, uint32_t e);

/* Direct-access tables ("Each ELT is implemented as an independent
 * table"): dense[j*(catalog+1) + e] = loss of e in ELT j, 0 if absent.
 * Returns 0, or -1 if an event id is outside [1, catalog]. */
int oracle_direct_access(const oracle_elts* elts, uint32_t catalog, double* dense);

/* Aggregate Risk Analysis (Alg. 1 + Alg. 3) over trials [0, n_trials) of a
 * CSR YET: trial t's events are event_ids[trial_off[t] - trial_off[0] ...].
 *   lookup_mode   ORACLE_LOOKUP_MAP or ORACLE_LOOKUP_DENSE (dense may be NULL
 *                 for MAP; for DENSE it is oracle_direct_access()'s output)
 *   fp32_storage  nonzero: every looked-up loss is read as (double)(float)x
 *                 (the fp32-storage variant, reading A13)
 *   elt_deductible/elt_limit  per-ELT terms I_j = (D_j, Lim_j) (A3), [n_elts]
 * Outputs (any may be NULL), layer-major [n_layers][n_trials]:
 *   ylt       Y[l][t]   year loss after aggregate terms
 *   scale     S[l][t] = sum over events of the per-event loss l_e (before
 *                        occurrence terms): the tolerance scale of A21
 *   lossy     m[l][t] = number of events with occurrence-net loss > 0
 *   portfolio P[t] = sum over layers in layer order of Y[l][t]  (A8)
 * Returns 0 or -1 on an event id outside [1, catalog] or an unknown ELT. */
int oracle_ara(const uint64_t* trial_off, const uint32_t* event_ids, uint64_t n_trials,
               const oracle_elts* elts, uint32_t catalog,
               const double* elt_deductible, const double* elt_limit,
               uint32_t n_layers, const oracle_layer* layers,
               int lookup_mode, const double* dense, int fp32_storage,
               double* ylt, double* scale, uint32_t* lossy, double* portfolio);

/* Programs (Alg. 1 l.1): program q's year loss = the sum of its
 * layers' year losses [program_layers[q], program_layers[q+1]) in layer
 * order, from 0.  ylt [n_layers][T] -> out [n_programs][T].  Returns 0 or -1
 * on a malformed program_layers. */
int oracle_programs(const double* ylt, uint64_t n_trials, uint32_t n_layers, uint32_t n_programs,
                    const uint32_t* program_layers, double* out);

/* k = ceil(T / R) for return period R, 1 <= R <= T (A10).  0 on domain error. */
uint64_t oracle_rank(uint64_t n_trials, double return_period);

/* PML(R) = k-th largest Y; TVaR(R) = mean of the k largest Y, summed
 * sequentially in descending order (A9).  Returns 0, or -1 on a
 * return period outside [1, T]. */
int oracle_metrics(const double* y, uint64_t n_trials, uint32_t n_rp,
                   const double* return_periods, uint64_t* k, double* pml, double* tvar);

/* Aggregate exceedance-probability curve of a YLT row (SURVEY 8f F4 "full EP
 * curve", reading A23): for each threshold x[i], the number of trials whose
 * year loss exceeds it, counts[i] = #{t : y[t] > x[i]}; EP(x[i]) =
 * counts[i] / T, the fraction of simulated years with a larger loss.  Plain
 * double loop. */
void oracle_ep_counts(const double* y, uint64_t n_trials, uint32_t n_points, const double* x, uint64_t* counts);

#ifdef __cplusplus
}
#endif
#endif
