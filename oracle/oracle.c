/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h).  Plain loops in the
 * paper's order and notation; no blocking, fusion or reordering.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

static double max2(double a, double b) { return a > b ? a : b; }
static double min2(double a, double b) { return a < b ? a : b; }

/* P:373 "l_T = min(max(l_T - T_OccR), T_OccL)", P:375 likewise for Agg;
 * reading A1: max(., 0).  Also used for I_j (reading A3). */
double oracle_apply_terms(double loss, double retention, double limit) {
    return min2(max2(loss - retention, 0.0), limit);
}

/* P:359 "Lookup E in the ELT and find corresponding loss"; miss -> 0 (A4). */
double oracle_lookup_map(const oracle_elts* elts, uint32_t j, uint32_t e) {
    uint64_t lo = elts->offsets[j], hi = elts->offsets[j + 1];
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        uint32_t k = elts->event_ids[mid];
        if (k == e) return elts->losses[mid];
        if (k < e) lo = mid + 1; else hi = mid;
    }
    return 0.0;
}

/* P:377 "ELTs ... implemented as direct access tables ... Each ELT is
 * implemented as an independent table". */
int oracle_direct_access(const oracle_elts* elts, uint32_t catalog, double* dense) {
    uint64_t stride = (uint64_t)catalog + 1;
    memset(dense, 0, sizeof(double) * stride * elts->n_elts);
    for (uint32_t j = 0; j < elts->n_elts; ++j) {
        for (uint64_t k = elts->offsets[j]; k < elts->offsets[j + 1]; ++k) {
            uint32_t e = elts->event_ids[k];
            if (e < 1 || e > catalog) return -1;
            dense[j * stride + e] = elts->losses[k];
        }
    }
    return 0;
}

static double lookup(const oracle_elts* elts, uint32_t catalog, int mode,
                     const double* dense, uint32_t j, uint32_t e) {
    if (mode == ORACLE_LOOKUP_DENSE) return dense[(uint64_t)j * ((uint64_t)catalog + 1) + e];
    return oracle_lookup_map(elts, j, e);
}

int oracle_ara(const uint64_t* trial_off, const uint32_t* event_ids, uint64_t n_trials,
               const oracle_elts* elts, uint32_t catalog,
               const double* elt_deductible, const double* elt_limit,
               uint32_t n_layers, const oracle_layer* layers,
               int lookup_mode, const double* dense, int fp32_storage,
               double* ylt, double* scale, uint32_t* lossy, double* portfolio) {
    const uint64_t base = trial_off[0];
    for (uint32_t l = 0; l < n_layers; ++l)                        /* Alg. 1 l.1-2 */
        for (uint32_t i = 0; i < layers[l].n_elts; ++i)
            if (layers[l].elts[i] >= elts->n_elts) return -1;     /* S:48 unresolved ELT */

    for (uint32_t l = 0; l < n_layers; ++l) {                      /* Alg. 1 l.2 */
        const oracle_layer* L = &layers[l];
        for (uint64_t t = 0; t < n_trials; ++t) {                  /* Alg. 3 l.2 */
            double G = 0.0;   /* trial aggregate: occurrence-net losses */
            double S = 0.0;   /* scale: sum of per-event losses (A21)          */
            uint32_t m = 0;
            for (uint64_t i = trial_off[t]; i < trial_off[t + 1]; ++i) {   /* Alg. 3 l.3 */
                uint32_t e = event_ids[i - base];
                if (e < 1 || e > catalog) return -1;                         /* A14 */
                double le = 0.0;                                  /* per-event loss l_E */
                for (uint32_t q = 0; q < L->n_elts; ++q) {        /* Alg. 3 l.4 */
                    uint32_t j = L->elts[q];
                    double x = lookup(elts, catalog, lookup_mode, dense, j, e);     /* l.5 */
                    if (fp32_storage) x = (double)(float)x;                          /* A13 */
                    le = le + oracle_apply_terms(x, elt_deductible[j], elt_limit[j]);/* l.6-7 */
                }
                S = S + le;
                double o = oracle_apply_terms(le, L->occ_retention, L->occ_limit);
                if (o > 0.0) m = m + 1;
                G = G + o;                      /* P:373 "accumulated into a single aggregate loss" */
            }
            double y = oracle_apply_terms(G, L->agg_retention, L->agg_limit);
            if (ylt) ylt[(uint64_t)l * n_trials + t] = y;
            if (scale) scale[(uint64_t)l * n_trials + t] = S;
            if (lossy) lossy[(uint64_t)l * n_trials + t] = m;
        }
    }
    if (portfolio) {                                               /* A8 */
        for (uint64_t t = 0; t < n_trials; ++t) {
            double p = 0.0;
            for (uint32_t l = 0; l < n_layers; ++l) {
                double y;
                if (ylt) y = ylt[(uint64_t)l * n_trials + t];
                else return -1;
                p = p + y;
            }
            portfolio[t] = p;
        }
    }
    return 0;
}

/* P:248-252 "PF = {P1, P2, ...}" with Alg. 1's loops over programs and layers. */
int oracle_programs(const double* ylt, uint64_t n_trials, uint32_t n_layers, uint32_t n_programs,
                    const uint32_t* program_layers, double* out) {
    if (n_programs && (program_layers[0] != 0 || program_layers[n_programs] != n_layers)) return -1;
    for (uint32_t q = 0; q < n_programs; ++q) {
        if (program_layers[q + 1] <= program_layers[q]) return -1;
        for (uint64_t t = 0; t < n_trials; ++t) {
            double s = 0.0;
            for (uint32_t l = program_layers[q]; l < program_layers[q + 1]; ++l) s = s + ylt[(uint64_t)l * n_trials + t];
            out[(uint64_t)q * n_trials + t] = s;
        }
    }
    return 0;
}

/* Reading A10: integer R -> (T + R - 1) / R in u64; otherwise ceil in long double. */
uint64_t oracle_rank(uint64_t n_trials, double R) {
    if (!(R >= 1.0) || R > (double)n_trials) return 0;
    if (R == floor(R) && R < 18446744073709551616.0) {
        uint64_t r = (uint64_t)R;
        return (n_trials + r - 1) / r;
    }
    return (uint64_t)ceill((long double)n_trials / (long double)R);
}

static int desc(const void* a, const void* b) {
    double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}

/* S:206 "sort losses descending; return the value at rank ceil(n/R)";
 * S:215 "mean of the worst ceil(q n) losses" with q = 1/R (A9). */
int oracle_metrics(const double* y, uint64_t n_trials, uint32_t n_rp,
                   const double* return_periods, uint64_t* k, double* pml, double* tvar) {
    double* s = (double*)malloc(sizeof(double) * (n_trials ? n_trials : 1));
    if (!s) return -1;
    memcpy(s, y, sizeof(double) * n_trials);
    qsort(s, n_trials, sizeof(double), desc);
    for (uint32_t r = 0; r < n_rp; ++r) {
        uint64_t kk = oracle_rank(n_trials, return_periods[r]);
        if (kk == 0) { free(s); return -1; }
        double sum = 0.0;
        for (uint64_t i = 0; i < kk; ++i) sum = sum + s[i];
        if (k) k[r] = kk;
        if (pml) pml[r] = s[kk - 1];
        if (tvar) tvar[r] = sum / (double)kk;
    }
    free(s);
    return 0;
}

/* A23: counts[i] = #{t : y[t] > x[i]} (strict exceedance), by brute force. */
void oracle_ep_counts(const double* y, uint64_t n_trials, uint32_t n_points, const double* x, uint64_t* counts) {
    for (uint32_t i = 0; i < n_points; ++i) {
        uint64_t c = 0;
        for (uint64_t t = 0; t < n_trials; ++t)
            if (y[t] > x[i]) c = c + 1;
        counts[i] = c;
    }
}
