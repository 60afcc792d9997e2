// kernel_fold.cu -- catalogue-fold mode (ARA_RUN_FOLD) and
// the program-row sums of ara_run_portfolio (Alg. 1 l.1).
#include <cstdlib>

#include "ara_device.cuh"

namespace ara {
namespace {

// ---------------------------------------------------------------------------
// Catalogue-fold mode.  Occurrence terms act on each event
// occurrence independently, so o(e) = min(max(l_e - OccR, 0), OccL)
// with l_e = sum_j min(max(tab[e][j] - D_j, 0), Lim_j) depends on the event id
// and the terms only.  fold_kernel evaluates it once per catalogue event (a
// coalesced streaming pass over the table, same arithmetic and ELT order as
// the trial kernel, so the values are bit-identical); trial_fold_kernel then
// gathers one small row o(e)[layers] per occurrence from an L2-resident array
// and accumulates exactly as the direct kernel does (same lane mapping, same
// per-lane order, same tree): the YLT and the lossy counts are bit-identical
// to the direct path.
template <typename TV, int NSEC, int NLB>
__global__ void __launch_bounds__(kThreads) fold_kernel(const __grid_constant__ TrialParams p) {
    constexpr int EPS = SecT<TV>::N;
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
    __shared__ double2 s_term[SM ? NLB : 1][kMaxWin];
    if (SM) {
        for (int i = threadIdx.x; i < NLB * kMaxWin; i += kThreads)
            s_term[i / kMaxWin][i % kMaxWin] = p.term[i / kMaxWin][i % kMaxWin];
        __syncthreads();
    }
    // The table is streamed once: its lines are read with an L2::evict_first
    // policy, so that they do not stay in L2 ahead of the data the trial pass
    // gathers next (the YET ids it streams are evict-first too, so stale
    // normal-priority table lines would otherwise hold most of L2 through the
    // whole trial pass).
    const uint64_t pol = policy_evict_first();
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e <= p.catalog;
         e += (uint64_t)gridDim.x * kThreads) {
        Row<TV, NSEC> r;
        {
            const TV* tab = static_cast<const TV*>(p.table) + (uint64_t)e * p.row_stride;
#pragma unroll
            for (int sct = 0; sct < NSEC; ++sct) {
                const TV* q = tab + p.sec_off[sct];
                if constexpr (sizeof(TV) == 8)
                    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
                        : "=d"(r.x[sct][0]), "=d"(r.x[sct][1]), "=d"(r.x[sct][2]), "=d"(r.x[sct][3])
                        : "l"(q), "l"(pol));
                else
                    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                        : "=f"(r.x[sct][0]), "=f"(r.x[sct][1]), "=f"(r.x[sct][2]), "=f"(r.x[sct][3]),
                          "=f"(r.x[sct][4]), "=f"(r.x[sct][5]), "=f"(r.x[sct][6]), "=f"(r.x[sct][7])
                        : "l"(q), "l"(pol));
            }
        }
#pragma unroll
        for (int l = 0; l < NLB; ++l) {
            if (l >= (int)p.n_layers) break;
            double le = 0.0;
#pragma unroll
            for (int s = 0; s < NSEC; ++s)
#pragma unroll
                for (int c = 0; c < EPS; ++c) {
                    const double2 tc = SM ? lds_term(&s_term[l][s * EPS + c]) : p.term[l][s * EPS + c];
                    le = __dadd_rn(le, terms((double)r.x[s][c], tc.x, tc.y));
                }
            p.fold[e * p.fold_stride + p.fold_col0 + l] = terms(le, p.lw[l].occ_r, p.lw[l].occ_l);
        }
    }
}

template <int NL>
__device__ __forceinline__ void ld_fold(const double* src, double (&o)[NL]) {
    if constexpr (NL == 1) {
        asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(o[0]) : "l"(src));
    } else if constexpr (NL == 2) {
        asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(o[0]), "=d"(o[1]) : "l"(src));
    } else {
#pragma unroll
        for (int h = 0; h < NL; h += 4)
            asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                : "=d"(o[h]), "=d"(o[h + 1]), "=d"(o[h + 2]), "=d"(o[h + 3]) : "l"(src + h));
    }
}

template <int NL>
__global__ void __launch_bounds__(kThreads) trial_fold_kernel(const __grid_constant__ TrialParams p) {
    constexpr int QB = NL <= 2 ? 4 : 2;
    constexpr uint64_t STEP = 32u * QB;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gw = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
    const uint64_t pol = policy_evict_first();
    const uint64_t base = __ldg(p.off);
    const double* fold = p.fold;
    uint32_t err = 0;
    // (gating the fold-row loads with the occupancy bitmap measured slower here:
    // 5.85 vs 3.98 ms -- the dependent bitmap load lengthens the load chain;
    // the scan-based kernel below does gate)
    TrialSched sched;
    sched.init(p, gw, nw);
    uint64_t t = sched.next(p), tn = sched.next(p);
    uint64_t a_nxt = 0, b_nxt = 0;
    if (t != ~0ull) { a_nxt = __ldg(p.off + t); b_nxt = __ldg(p.off + t + 1); }
    for (; t != ~0ull; t = tn, tn = sched.next(p)) {
        uint64_t a = a_nxt, b = b_nxt;
        if (tn != ~0ull) { a_nxt = __ldg(p.off + tn); b_nxt = __ldg(p.off + tn + 1); }
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        const uint64_t n = b - a;
        const uint32_t* ids = p.ids + (a - base);
        double G[NL];
        uint32_t m[NL];
#pragma unroll
        for (int l = 0; l < NL; ++l) { G[l] = 0.0; m[l] = 0u; }
        auto load_ids = [&](uint64_t k0, uint32_t (&e)[QB]) {
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                const uint64_t k = k0 + 32u * q + lane;
                uint32_t v = 0u;
                if (k < n) {
                    v = ld_stream_u32(ids + k, pol);
                    if (v == 0u || v > p.catalog) { err |= ERRBIT_EVENT_RANGE; v = 0u; }
                }
                e[q] = v;
            }
        };
        uint32_t e1[QB];
        double o0[QB][NL];
        {
            uint32_t e0[QB];
            load_ids(0, e0);
            load_ids(STEP, e1);
#pragma unroll
            for (int q = 0; q < QB; ++q) ld_fold<NL>(fold + (uint64_t)e0[q] * p.fold_stride, o0[q]);
        }
#pragma unroll 1
        for (uint64_t k0 = 0; k0 < n; k0 += STEP) {
            uint32_t e2[QB];
            load_ids(k0 + 2 * STEP, e2);
            double o1[QB][NL];
            if (k0 + STEP < n) {
#pragma unroll
                for (int q = 0; q < QB; ++q) ld_fold<NL>(fold + (uint64_t)e1[q] * p.fold_stride, o1[q]);
            }
#pragma unroll
            for (int q = 0; q < QB; ++q)
#pragma unroll
                for (int l = 0; l < NL; ++l) {
                    G[l] = __dadd_rn(G[l], o0[q][l]);
                    m[l] += (o0[q][l] > 0.0) ? 1u : 0u;
                }
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                e1[q] = e2[q];
#pragma unroll
                for (int l = 0; l < NL; ++l) o0[q][l] = o1[q][l];
            }
        }
#pragma unroll
        for (int l = 0; l < NL; ++l) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
                m[l] += __shfl_xor_sync(0xffffffffu, m[l], off);
            }
        }
        if (lane == 0) {
            store_trial(p, t, G, m);
        }
    }
    peer_fence(p);
    if (err) atomicOr(p.err, err);
}

template <typename TV>
void* pick_fold(uint32_t nsec, int nl) {
#define ARA_FOLD_NL(NS)                                                   \
    if (nl <= 1) return (void*)fold_kernel<TV, NS, 1>;                    \
    if (nl <= 2) return (void*)fold_kernel<TV, NS, 2>;                    \
    return (void*)fold_kernel<TV, NS, 4>;
    if (nsec <= 1) { ARA_FOLD_NL(1) }
    if (nsec <= 2) { ARA_FOLD_NL(2) }
    if (nsec <= 4) { ARA_FOLD_NL(4) }
    ARA_FOLD_NL(8)
#undef ARA_FOLD_NL
}

}  // namespace

cudaError_t launch_fold(const TrialParams& p, int fp32, uint32_t nsec, cudaStream_t s) {
    void* fn = fp32 ? pick_fold<float>(nsec, (int)p.n_layers) : pick_fold<double>(nsec, (int)p.n_layers);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t need = ((uint64_t)p.catalog + 1 + kThreads - 1) / kThreads;
    const uint64_t g = need < (uint64_t)nsm * 8 ? need : (uint64_t)nsm * 8;
    void* args[] = {(void*)&p};
    return cudaLaunchKernel(fn, dim3((unsigned)g), dim3(kThreads), args, 0, s);
}


cudaError_t launch_trials_folded(const TrialParams& p, int grid_mult_x100, cudaStream_t s) {
    if (p.t_end <= p.t_begin) return cudaSuccess;
    void* fn = p.fold_stride <= 1 ? (void*)trial_fold_kernel<1>
               : p.fold_stride <= 2 ? (void*)trial_fold_kernel<2>
               : p.fold_stride <= 4 ? (void*)trial_fold_kernel<4>
                                    : (void*)trial_fold_kernel<8>;
    int dev = 0, nsm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    uint64_t grid = (uint64_t)nsm * per_sm * grid_mult_x100 / 100;
    const uint64_t need = ((p.t_end - p.t_begin) * 32 + kThreads - 1) / kThreads;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    void* args[] = {(void*)&p};
    return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(kThreads), args, 0, s);
}

// Program rows (Alg. 1 l.1): Y_prog[q][t] = sum of the program's layer rows, in
// layer order, from +0 (the oracle's sequential order).
__global__ void __launch_bounds__(256) program_sum_kernel(double* __restrict__ ylt, uint64_t ld, uint64_t t_local,
                                                          uint32_t n_programs, const uint32_t* __restrict__ pl,
                                                          uint32_t n_layers) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < t_local;
         t += (uint64_t)gridDim.x * blockDim.x) {
        for (uint32_t q = 0; q < n_programs; ++q) {
            double acc = 0.0;
            for (uint32_t l = __ldg(pl + q); l < __ldg(pl + q + 1); ++l) acc = __dadd_rn(acc, ylt[(uint64_t)l * ld + t]);
            ylt[(uint64_t)(n_layers + q) * ld + t] = acc;
        }
    }
}

cudaError_t launch_program_sums(double* ylt, uint64_t ld, uint64_t t_local, uint32_t n_programs,
                                const uint32_t* d_program_layers, uint32_t n_layers, cudaStream_t s) {
    if (!n_programs || !t_local) return cudaSuccess;
    uint64_t blocks = (t_local + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    program_sum_kernel<<<(unsigned)blocks, 256, 0, s>>>(ylt, ld, t_local, n_programs, d_program_layers, n_layers);
    return cudaGetLastError();
}

}  // namespace ara
