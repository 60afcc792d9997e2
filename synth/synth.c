/*
 * synth.c — counter-based synthetic inputs for ARA (see synth.h).
 * Distribution recipe: DESIGN.md §"Input recipe".
 */
#include "synth.h"
#include <math.h>
#include <pthread.h>
#include <stddef.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

/* stream ids */
enum { ST_NT = 1, ST_EV = 2, ST_TS = 3, ST_MEMB = 16, ST_LU1 = 17, ST_LU2 = 18 };

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint64_t synth_u64(uint64_t seed, uint64_t stream, uint64_t index) {
    uint64_t key = mix64(seed + GOLDEN * (stream + 1));
    return mix64(key + GOLDEN * (index + 1));
}

/* uniform double in [0,1) with 53 random bits */
static inline double u01(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }
/* uniform integer in [0, m) via multiply-high (m <= 2^32) */
static inline uint32_t below(uint64_t r, uint64_t m) { return (uint32_t)(((r >> 32) * m) >> 32); }

static inline uint32_t trial_count(uint64_t seed, uint64_t t, uint32_t nmin, uint32_t nmax) {
    return nmin + below(synth_u64(seed, ST_NT, t), (uint64_t)(nmax - nmin) + 1);
}

void synth_trial_counts(uint64_t seed, uint64_t first, uint64_t n,
                        uint32_t nmin, uint32_t nmax, uint32_t* counts) {
    for (uint64_t i = 0; i < n; ++i) counts[i] = trial_count(seed, first + i, nmin, nmax);
}

uint64_t synth_event_base(uint64_t seed, uint64_t first, uint32_t nmin, uint32_t nmax) {
    uint64_t s = 0;
    for (uint64_t t = 0; t < first; ++t) s += trial_count(seed, t, nmin, nmax);
    return s;
}

uint64_t synth_yet_offsets(uint64_t seed, uint64_t first, uint64_t n,
                           uint32_t nmin, uint32_t nmax, uint64_t* offsets) {
    offsets[0] = 0;
    for (uint64_t i = 0; i < n; ++i)
        offsets[i + 1] = offsets[i] + trial_count(seed, first + i, nmin, nmax);
    return offsets[n];
}

typedef struct { uint64_t seed, begin, lo, hi; uint32_t catalog; uint32_t* ids; } ev_job;

static void* ev_worker(void* p) {
    ev_job* j = (ev_job*)p;
    for (uint64_t i = j->lo; i < j->hi; ++i)
        j->ids[i] = 1u + below(synth_u64(j->seed, ST_EV, j->begin + i), j->catalog);
    return NULL;
}

void synth_yet_events(uint64_t seed, uint32_t catalog, uint64_t begin, uint64_t n,
                      uint32_t* ids, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (n < (1u << 20)) nthreads = 1;
    pthread_t th[256];
    ev_job jobs[256];
    for (int k = 0; k < nthreads; ++k) {
        jobs[k] = (ev_job){seed, begin, n * k / nthreads, n * (k + 1) / nthreads, catalog, ids};
        if (k > 0) pthread_create(&th[k], NULL, ev_worker, &jobs[k]);
    }
    ev_worker(&jobs[0]);
    for (int k = 1; k < nthreads; ++k) pthread_join(th[k], NULL);
}

void synth_trial_timestamps(uint64_t seed, uint64_t trial, uint32_t n, double* ts) {
    /* sorted uniforms as normalised cumulative exponential spacings */
    double acc = 0.0;
    uint64_t base = trial << 12;
    for (uint32_t k = 0; k < n; ++k) {
        acc += -log(1.0 - u01(synth_u64(seed, ST_TS, base + k)));
        ts[k] = acc;
    }
    double tot = acc - log(1.0 - u01(synth_u64(seed, ST_TS, base + n)));
    for (uint32_t k = 0; k < n; ++k) ts[k] /= tot;
}

static inline int member(uint64_t seed, uint32_t j, uint32_t e, uint32_t catalog, double rho) {
    if (rho >= 1.0) return 1;
    uint64_t idx = (uint64_t)j * ((uint64_t)catalog + 1) + e;
    return u01(synth_u64(seed, ST_MEMB, idx)) < rho;
}

uint64_t synth_elt_count(uint64_t seed, uint32_t j, uint32_t catalog, double rho) {
    uint64_t c = 0;
    for (uint32_t e = 1; e <= catalog; ++e) c += (uint64_t)member(seed, j, e, catalog, rho);
    return c;
}

void synth_elt_fill(uint64_t seed, uint32_t j, uint32_t catalog, double rho,
                    double mu, double sigma, double int_cap,
                    uint32_t* event_ids, double* losses) {
    uint64_t w = 0;
    for (uint32_t e = 1; e <= catalog; ++e) {
        if (!member(seed, j, e, catalog, rho)) continue;
        uint64_t idx = (uint64_t)j * ((uint64_t)catalog + 1) + e;
        /* Box–Muller, hand-rolled so the stream is fixed by this file alone */
        double u1 = ((double)(synth_u64(seed, ST_LU1, idx) >> 11) + 1.0) * 0x1.0p-53; /* (0,1] */
        double u2 = u01(synth_u64(seed, ST_LU2, idx));
        double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        double x = exp(mu + sigma * z);
        if (int_cap > 0.0) {
            x = floor(x);
            if (x > int_cap - 1.0) x = int_cap - 1.0;
        }
        event_ids[w] = e;
        losses[w] = x;
        ++w;
    }
}
