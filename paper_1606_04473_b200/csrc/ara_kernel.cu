// ara_kernel.cu — the ARA hot loop on sm_100a.
//
// PAPER.md Alg. 3 + P:371-377: for each trial, for each event,
// for each ELT of the layer: look the event up, apply the per-ELT
// terms I, sum across ELTs; apply occurrence terms to the
// event's combined loss; accumulate the trial; apply aggregate terms
// -> the trial's YLT entry.
//
// B200 mapping:
//   * one warp per trial (the paper used one thread per trial);
//   * the trial's event ids stream through coalesced 128-B warp loads with an
//     L2 evict_first policy (the YET is read exactly once);
//   * event k of the trial goes to lane k % 32, slot (k / 32) % 4 — a mapping
//     that depends only on the trial's own event order, so the per-trial
//     summation order (and therefore the YLT bits) is independent of how the
//     YET is sharded, chunked or aligned in memory (partition invariance);
//   * one lane reads one event's whole interleaved row tab[e][*] — the layer's
//     window of 32-B sectors — with 256-bit non-allocating loads
//     (LDG.E.NA.ENL2.256), then sums the ELT terms sequentially in ELT order
//     (bit-identical per-event loss to the sequential oracle);
//   * the trial sum is a fixed lane-strided + 5-step xor-shuffle tree; lossy
//     occurrence counts are integers (exact);
//   * validation of YET ids / offsets is fused (error bits, no extra pass).
// This is a gather-and-reduce path: no tensor cores (not a contraction).
#include "ara_internal.cuh"

namespace ara {
namespace {

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}

// One 32-B sector of a row, predicated (pred == 0 leaves x untouched).
__device__ __forceinline__ void ld_sector(const double* p, double (&x)[4], uint32_t pred) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %4, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%5];\n\t}"
        : "+d"(x[0]), "+d"(x[1]), "+d"(x[2]), "+d"(x[3]) : "r"(pred), "l"(p));
}
__device__ __forceinline__ void ld_sector(const float* p, float (&x)[8], uint32_t pred) {
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %8, 0;\n\t"
        "@q ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%9];\n\t}"
        : "+f"(x[0]), "+f"(x[1]), "+f"(x[2]), "+f"(x[3]),
          "+f"(x[4]), "+f"(x[5]), "+f"(x[6]), "+f"(x[7])
        : "r"(pred), "l"(p));
}

// min(max(x - r, 0), lim): P:373/P:375 with reading A1; also I_j (A3).
__device__ __forceinline__ double terms(double x, double r, double lim) {
    return fmin(fmax(__dsub_rn(x, r), 0.0), lim);
}

template <typename TV> struct SecT;
template <> struct SecT<double> { static constexpr int N = 4; };
template <> struct SecT<float> { static constexpr int N = 8; };

// Per-event work for all layers of the launch: a3 lookup, a4 per-ELT terms,
// a5 sequential ELT sum, a6 occurrence terms, a7 accumulate.
// Terms of small windows stay in uniform registers (constant bank); larger
// sets are read from shared memory at the point of use (volatile, so the
// compiler cannot hoist them into vector registers and spill).
__device__ __forceinline__ double2 lds_term(const double2* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

template <typename TV, int NSEC, int NLB, bool SHARE>
struct TermsInSmem {
    static constexpr bool value = NLB * NSEC * SecT<TV>::N > 16;
};

template <typename TV, int NSEC, int NLB, bool SHARE>
__device__ __forceinline__ void event_step(const TrialParams& p, const double2 (*s_term)[kMaxWin], uint32_t e,
                                           double (&G)[NLB], uint32_t (&m)[NLB]) {
    constexpr int EPS = SecT<TV>::N;
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB, SHARE>::value;
    const TV* row = static_cast<const TV*>(p.table) + (uint64_t)e * p.row_elems;
    TV x[NSEC][EPS];
#pragma unroll
    for (int l = 0; l < NLB; ++l) {
        if (l >= (int)p.n_layers) break;
        if (!SHARE || l == 0) {
            const TV* w = row + (uint64_t)p.lw[l].sec0 * EPS;
#pragma unroll
            for (int s = 0; s < NSEC; ++s) {
#pragma unroll
                for (int c = 0; c < EPS; ++c) x[s][c] = TV(0);
                ld_sector(w + s * EPS, x[s], e != 0u && (uint32_t)s < p.lw[l].nsec);
            }
        }
        double le = 0.0;
#pragma unroll
        for (int s = 0; s < NSEC; ++s)
#pragma unroll
            for (int c = 0; c < EPS; ++c) {
                const double2 tc = SM ? lds_term(&s_term[l][s * EPS + c]) : p.term[l][s * EPS + c];
                le = __dadd_rn(le, terms((double)x[s][c], tc.x, tc.y));
            }
        const double o = terms(le, p.lw[l].occ_r, p.lw[l].occ_l);
        G[l] = __dadd_rn(G[l], o);
        m[l] += (o > 0.0) ? 1u : 0u;
    }
}

// Events per lane in flight per iteration: one 32-B sector per fp64 window
// column group costs 8 registers, so keep ~64 registers of rows in flight.
template <typename TV, int NSEC, int NLB, bool SHARE>
struct Batch {
    static constexpr int R = NSEC * SecT<TV>::N * (int)sizeof(TV) / 4 * (SHARE ? 1 : NLB);  // row regs/event
    static constexpr int QB = R >= 64 ? 1 : (R >= 32 ? 2 : 4);
};

template <typename TV, int NSEC, int NLB, bool SHARE>
__global__ void __launch_bounds__(kThreads, 2) trial_kernel(const __grid_constant__ TrialParams p) {
    constexpr int QB = Batch<TV, NSEC, NLB, SHARE>::QB;
    constexpr uint64_t STEP = 32u * QB;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gw = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
    const uint64_t pol = policy_evict_first();
    const uint64_t base = __ldg(p.off);
    uint32_t err = 0;
    __shared__ double2 s_term[TermsInSmem<TV, NSEC, NLB, SHARE>::value ? NLB : 1][kMaxWin];
    if (TermsInSmem<TV, NSEC, NLB, SHARE>::value) {
        for (int i = threadIdx.x; i < NLB * kMaxWin; i += kThreads) s_term[i / kMaxWin][i % kMaxWin] = p.term[i / kMaxWin][i % kMaxWin];
        __syncthreads();
    }

    for (uint64_t t = p.t_begin + gw; t < p.t_end; t += nw) {
        uint64_t a = __ldg(p.off + t), b = __ldg(p.off + t + 1);
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        const uint64_t n = b - a;
        const uint32_t* ids = p.ids + (a - base);
        double G[NLB];
        uint32_t m[NLB];
#pragma unroll
        for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }

        // Event k of the trial -> lane k % 32; each lane visits its events in
        // increasing k.  Ids of the next step are prefetched one step ahead.
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
        uint32_t e_cur[QB];
        load_ids(0, e_cur);
#pragma unroll 1
        for (uint64_t k0 = 0; k0 < n; k0 += STEP) {
            uint32_t e_nxt[QB];
            load_ids(k0 + STEP, e_nxt);
#pragma unroll
            for (int q = 0; q < QB; ++q) event_step<TV, NSEC, NLB, SHARE>(p, s_term, e_cur[q], G, m);
#pragma unroll
            for (int q = 0; q < QB; ++q) e_cur[q] = e_nxt[q];
        }
        // a7: fixed xor-tree over lanes; every lane ends with the same bits.
#pragma unroll
        for (int l = 0; l < NLB; ++l) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
                G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
                m[l] += __shfl_xor_sync(0xffffffffu, m[l], off);
            }
        }
        // a8: aggregate terms, store the YLT entries (+ portfolio, A8).
        if (lane == 0) {
            double port = 0.0;
            if (p.portfolio_mode == 1) port = p.ylt[(uint64_t)p.portfolio_row * p.ld + t];
#pragma unroll
            for (int l = 0; l < NLB; ++l) {
                if (l >= (int)p.n_layers) break;
                const double y = terms(G[l], p.lw[l].agg_r, p.lw[l].agg_l);
                p.ylt[(uint64_t)(p.ylt_row0 + l) * p.ld + t] = y;
                if (p.lossy) p.lossy[(uint64_t)(p.ylt_row0 + l) * p.ld + t] = m[l];
                port = __dadd_rn(port, y);
            }
            if (p.portfolio_mode >= 0) p.ylt[(uint64_t)p.portfolio_row * p.ld + t] = port;
        }
    }
    if (err) atomicOr(p.err, err);
}

// Wide layers (window > kMaxSec sectors): same arithmetic and lane mapping,
// one layer per launch, scalar loads, runtime column loop.
template <typename TV>
__global__ void __launch_bounds__(kThreads) trial_kernel_wide(const __grid_constant__ TrialParams p,
                                                              const double2* __restrict__ cterm,
                                                              uint32_t col0, uint32_t ncol) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gw = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
    const uint64_t base = __ldg(p.off);
    const TV* tab = static_cast<const TV*>(p.table);
    uint32_t err = 0;
    for (uint64_t t = p.t_begin + gw; t < p.t_end; t += nw) {
        uint64_t a = __ldg(p.off + t), b = __ldg(p.off + t + 1);
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        const uint64_t n = b - a;
        const uint32_t* ids = p.ids + (a - base);
        double G = 0.0;
        uint32_t m = 0;
        for (uint64_t k0 = 0; k0 < n; k0 += 128) {
            for (int q = 0; q < 4; ++q) {
                const uint64_t k = k0 + 32u * q + lane;
                uint32_t v = 0u;
                if (k < n) {
                    v = __ldg(ids + k);
                    if (v == 0u || v > p.catalog) { err |= ERRBIT_EVENT_RANGE; v = 0u; }
                }
                double le = 0.0;
                if (v) {
                    const TV* row = tab + (uint64_t)v * p.row_elems + col0;
                    for (uint32_t c = 0; c < ncol; ++c) {
                        const double2 tc = cterm[c];
                        le = __dadd_rn(le, terms((double)__ldg(row + c), tc.x, tc.y));
                    }
                }
                const double o = terms(le, p.lw[0].occ_r, p.lw[0].occ_l);
                G = __dadd_rn(G, o);
                m += (o > 0.0) ? 1u : 0u;
            }
        }
        for (int off = 16; off >= 1; off >>= 1) {
            G = __dadd_rn(G, __shfl_xor_sync(0xffffffffu, G, off));
            m += __shfl_xor_sync(0xffffffffu, m, off);
        }
        if (lane == 0) {
            const double y = terms(G, p.lw[0].agg_r, p.lw[0].agg_l);
            p.ylt[(uint64_t)p.ylt_row0 * p.ld + t] = y;
            if (p.lossy) p.lossy[(uint64_t)p.ylt_row0 * p.ld + t] = m;
            if (p.portfolio_mode >= 0) {
                double port = p.portfolio_mode == 1 ? p.ylt[(uint64_t)p.portfolio_row * p.ld + t] : 0.0;
                p.ylt[(uint64_t)p.portfolio_row * p.ld + t] = __dadd_rn(port, y);
            }
        }
    }
    if (err) atomicOr(p.err, err);
}

template <typename TV, int NSEC, int NLB, bool SHARE>
struct Inst {
    static void* fn() { return (void*)trial_kernel<TV, NSEC, NLB, SHARE>; }
};

template <typename TV, int NLB, bool SHARE>
void* pick_nsec(uint32_t nsec) {
    if (nsec <= 1) return Inst<TV, 1, NLB, SHARE>::fn();
    if (nsec <= 2) return Inst<TV, 2, NLB, SHARE>::fn();
    if (nsec <= 4) return Inst<TV, 4, NLB, SHARE>::fn();
    return Inst<TV, 8, NLB, SHARE>::fn();
}

template <typename TV>
void* pick(uint32_t nsec, bool share, int nl) {
    if (nl <= 1) return pick_nsec<TV, 1, false>(nsec);
    if (nl <= 2) return share ? pick_nsec<TV, 2, true>(nsec) : pick_nsec<TV, 2, false>(nsec);
    return share ? pick_nsec<TV, 4, true>(nsec) : pick_nsec<TV, 4, false>(nsec);
}

void* pick_kernel(int fp32, uint32_t nsec, bool share, int nl) {
    return fp32 ? pick<float>(nsec, share, nl) : pick<double>(nsec, share, nl);
}

}  // namespace

int trial_kernel_grid(int fp32, uint32_t max_nsec, bool shared_window, int n_layers) {
    int dev = 0, nsm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    void* fn = max_nsec > (uint32_t)kMaxSec
                   ? (fp32 ? (void*)trial_kernel_wide<float> : (void*)trial_kernel_wide<double>)
                   : pick_kernel(fp32, max_nsec, shared_window, n_layers);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess ||
        per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    return nsm * per_sm;
}

cudaError_t launch_trials(const TrialParams& p, int fp32, uint32_t max_nsec, bool shared_window,
                          int grid, cudaStream_t s) {
    if (p.t_end <= p.t_begin) return cudaSuccess;
    const uint64_t warps = p.t_end - p.t_begin;
    const uint64_t need = (warps * 32 + kThreads - 1) / kThreads;
    const int g = (int)((uint64_t)grid < need ? (uint64_t)grid : need);
    void* fn = pick_kernel(fp32, max_nsec, shared_window, (int)p.n_layers);
    void* args[] = {(void*)&p};
    return cudaLaunchKernel(fn, dim3(g), dim3(kThreads), args, 0, s);
}

cudaError_t launch_trials_wide(const TrialParams& p, int fp32, const double2* d_cterm, uint32_t col0,
                               uint32_t ncol, int grid, cudaStream_t s) {
    if (p.t_end <= p.t_begin) return cudaSuccess;
    const uint64_t need = ((p.t_end - p.t_begin) * 32 + kThreads - 1) / kThreads;
    const int g = (int)((uint64_t)grid < need ? (uint64_t)grid : need);
    if (fp32)
        trial_kernel_wide<float><<<g, kThreads, 0, s>>>(p, d_cterm, col0, ncol);
    else
        trial_kernel_wide<double><<<g, kThreads, 0, s>>>(p, d_cterm, col0, ncol);
    return cudaGetLastError();
}

}  // namespace ara
