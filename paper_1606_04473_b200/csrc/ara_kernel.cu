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
//   * event k of the trial goes to lane k % 32 and each lane visits its events
//     in increasing k — a mapping that depends only on the trial's own event
//     order, so the per-trial summation order (and the YLT bits) is
//     independent of how the YET is sharded, chunked or aligned in memory;
//   * one lane reads one event's row window of the column-blocked
//     direct-access table — the layer's 32-B sectors — with 256-bit
//     non-allocating loads (LDG.E.NA.ENL2.256), then sums the ELT terms
//     sequentially in ELT order (bit-identical per-event loss to the
//     sequential oracle, hence exact lossy-occurrence counts);
//   * software pipeline per warp: ids two steps ahead, rows one step ahead of
//     the fp64 term arithmetic, so every lane keeps a row in flight;
//   * the trial sum is a fixed lane-strided + 5-step xor-shuffle tree;
//   * validation of YET ids / offsets is fused (error bits, no extra pass).
// This is a gather-and-reduce path: no tensor cores (not a contraction).
#include <cstdlib>
#include <cstring>

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

// One 32-B sector of a row, unconditional 256-bit non-allocating load.
// Lanes without an event load row 0 (all zeros, L2-resident), and sectors
// beyond a layer's window carry deductible +inf, so neither needs a predicate.
__device__ __forceinline__ void ld_sector(const double* p, double (&x)[4]) {
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(x[0]), "=d"(x[1]), "=d"(x[2]), "=d"(x[3]) : "l"(p));
}
__device__ __forceinline__ void ld_sector(const float* p, float (&x)[8]) {
    asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=f"(x[0]), "=f"(x[1]), "=f"(x[2]), "=f"(x[3]), "=f"(x[4]), "=f"(x[5]), "=f"(x[6]), "=f"(x[7])
        : "l"(p));
}

// min(max(x - r, 0), lim): P:373/P:375 with reading A1; also I_j (A3).
// max(v, 0) is the oracle's (v > 0 ? v : 0) done on the sign bit (integer
// pipe; v is never NaN); min is (v < lim ? v : lim).  Identical results to
// the oracle for every non-NaN input, signed zeros included.
__device__ __forceinline__ double terms(double x, double r, double lim) {
    double v = __dsub_rn(x, r);
    v = (__double2hiint(v) >= 0) ? v : 0.0;
    return (v < lim) ? v : lim;
}

template <typename TV> struct SecT;
template <> struct SecT<double> { static constexpr int N = 4; };
template <> struct SecT<float> { static constexpr int N = 8; };

// Terms of small windows stay in uniform registers (constant bank); larger
// sets are read from shared memory at the point of use (volatile, so the
// compiler cannot hoist them into vector registers and spill).
__device__ __forceinline__ double2 lds_term(const double2* p) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y)
                 : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

template <typename TV, int NSEC, int NLB>
struct TermsInSmem {
    static constexpr bool value = NLB * NSEC * SecT<TV>::N > 16;
};

// One event's window (NSEC sectors) of the column-blocked table (a3 lookup).
// Layers sharing a launch share their window (tower layers), so one load
// serves all of them.
template <typename TV, int NSEC>
struct Row {
    static constexpr int EPS = SecT<TV>::N;
    TV x[NSEC][EPS];

    __device__ __forceinline__ void load(const TrialParams& p, uint32_t e) {
        const TV* tab = static_cast<const TV*>(p.table) + (uint64_t)e * p.row_stride;
#pragma unroll
        for (int s = 0; s < NSEC; ++s) ld_sector(tab + p.sec_off[s], x[s]);
    }
};

// Per-event work for the layers of the launch: a4 per-ELT terms, a5
// sequential ELT sum, a6 occurrence terms, a7 accumulate.
template <typename TV, int NSEC, int NLB>
__device__ __forceinline__ void event_compute(const TrialParams& p, const double2 (*s_term)[kMaxWin],
                                              const Row<TV, NSEC>& r, double (&G)[NLB], uint32_t (&m)[NLB]) {
    constexpr int EPS = SecT<TV>::N;
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
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
        const double o = terms(le, p.lw[l].occ_r, p.lw[l].occ_l);
        G[l] = __dadd_rn(G[l], o);
        m[l] += (o > 0.0) ? 1u : 0u;
    }
}

// event_compute for a window staged in shared memory (swizzled 16-B chunks):
// each sector is read right before its ELTs are summed, so only one sector of
// the row is live in registers.  Same arithmetic and order as event_compute.
template <typename TV, int NSEC, int NLB>
__device__ __forceinline__ void event_compute_smem(const TrialParams& p, const double2 (*s_term)[kMaxWin],
                                                   uint32_t src, uint32_t swz, double (&G)[NLB],
                                                   uint32_t (&m)[NLB]) {
    constexpr int EPS = SecT<TV>::N;
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
#pragma unroll
    for (int l = 0; l < NLB; ++l) {
        if (l >= (int)p.n_layers) break;
        double le = 0.0;
#pragma unroll
        for (int s = 0; s < NSEC; ++s) {
            TV x[EPS];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(src + (((uint32_t)(2 * s + h) ^ swz) << 4))
                             : "memory");
                memcpy(&x[h * (EPS / 2)], &v, 16);
            }
#pragma unroll
            for (int c = 0; c < EPS; ++c) {
                const double2 tc = SM ? lds_term(&s_term[l][s * EPS + c]) : p.term[l][s * EPS + c];
                le = __dadd_rn(le, terms((double)x[c], tc.x, tc.y));
            }
        }
        const double o = terms(le, p.lw[l].occ_r, p.lw[l].occ_l);
        G[l] = __dadd_rn(G[l], o);
        m[l] += (o > 0.0) ? 1u : 0u;
    }
}

// a8 epilogue of one trial (lane 0): aggregate terms per layer, the YLT and
// lossy-count stores, the portfolio row (A8) -- and, when the run assembles
// the global YLT over NVLink (p.n_peers > 0), the same values stored straight
// into every rank's global YLT (peer memory mapped by CUDA IPC), which fuses
// the YLT all-gather (a9) into the kernel epilogue.
template <int NL>
__device__ __forceinline__ void store_trial(const TrialParams& p, uint64_t t, const double (&G)[NL],
                                            const uint32_t (&m)[NL]) {
    double port = 0.0;
    if (p.portfolio_mode == 1) port = p.ylt[(uint64_t)p.portfolio_row * p.ld + t];
    const uint64_t tg = p.peer_t0 + t;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        if (l >= (int)p.n_layers) break;
        const double y = terms(G[l], p.lw[l].agg_r, p.lw[l].agg_l);
        p.ylt[(uint64_t)(p.ylt_row0 + l) * p.ld + t] = y;
        if (p.lossy) p.lossy[(uint64_t)(p.ylt_row0 + l) * p.ld + t] = m[l];
        port = __dadd_rn(port, y);
        for (uint32_t r = 0; r < p.n_peers; ++r) p.peer_ylt[r][(uint64_t)(p.ylt_row0 + l) * p.peer_ld + tg] = y;
    }
    if (p.portfolio_mode >= 0) {
        p.ylt[(uint64_t)p.portfolio_row * p.ld + t] = port;
        for (uint32_t r = 0; r < p.n_peers; ++r) p.peer_ylt[r][(uint64_t)p.portfolio_row * p.peer_ld + tg] = port;
    }
}

// peer stores of this warp are performed before the kernel is seen complete
__device__ __forceinline__ void peer_fence(const TrialParams& p) {
    if (p.n_peers && (threadIdx.x & 31u) == 0) __threadfence_system();
}

// event_compute for the sparse path: on the paper's ELTs an occupied row holds
// about one non-zero loss in 16, and a +0 loss adds an exact +0 to l_e (every
// deductible is >= 0 and l_e >= +0), so only the non-zero elements of the
// window are visited -- in ascending ELT order, which keeps l_e bit-identical
// to the dense sum.  The lane reads its staged row once to build the non-zero
// mask, then loads each non-zero element (and its terms) by index.
__device__ __forceinline__ uint4 lds_v4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a)
                 : "memory");
    return v;
}
template <typename TV, int NSEC, int NLB>
__device__ __forceinline__ void event_compute_sparse(const TrialParams& p, const double2 (*s_term)[kMaxWin],
                                                     uint32_t src, uint32_t swz, double (&G)[NLB],
                                                     uint32_t (&m)[NLB]) {
    constexpr int CH = NSEC * 2;                 // 16-B chunks of the window
    constexpr int EPC = 16 / (int)sizeof(TV);    // elements per chunk
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
    uint32_t nz = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const uint4 v = lds_v4(src + (((uint32_t)c ^ swz) << 4));
        if (EPC == 2) {
            nz |= ((v.x | v.y) != 0u ? 1u : 0u) << (2 * c);
            nz |= ((v.z | v.w) != 0u ? 1u : 0u) << (2 * c + 1);
        } else {
            nz |= (v.x != 0u ? 1u : 0u) << (4 * c);
            nz |= (v.y != 0u ? 1u : 0u) << (4 * c + 1);
            nz |= (v.z != 0u ? 1u : 0u) << (4 * c + 2);
            nz |= (v.w != 0u ? 1u : 0u) << (4 * c + 3);
        }
    }
#pragma unroll
    for (int l = 0; l < NLB; ++l) {
        if (l >= (int)p.n_layers) break;
        double le = 0.0;
        uint32_t mm = nz;
        while (mm) {
            const uint32_t j = (uint32_t)(__ffs(mm) - 1);
            mm &= mm - 1u;
            const uint32_t a = src + (((j / EPC) ^ swz) << 4) + (j % EPC) * (uint32_t)sizeof(TV);
            double x;
            if (EPC == 2) {
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a) : "memory");
            } else {
                float xf;
                asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xf) : "r"(a) : "memory");
                x = (double)xf;
            }
            const double2 tc = SM ? lds_term(&s_term[l][j]) : p.term[l][j];
            le = __dadd_rn(le, terms(x, tc.x, tc.y));
        }
        const double o = terms(le, p.lw[l].occ_r, p.lw[l].occ_l);
        G[l] = __dadd_rn(G[l], o);
        m[l] += (o > 0.0) ? 1u : 0u;
    }
}

// event_compute over a staged packed row (TrialParams::pk): the slot's mask
// names the block's non-zero columns, so the window's non-zeros are visited in
// ascending column order -- the order (and the values) event_compute_sparse
// visits, so l_e is bit-identical.  The v-th non-zero of the row sits in the
// slot when v < 24 / esz, else it is read from the dense table (rows with more
// non-zeros than the slot holds: ~1e-4 of the occupied rows at rho = 0.01).
template <typename TV, int NLB>
__device__ __forceinline__ void event_compute_packed(const TrialParams& p, const double2 (*s_term)[kMaxWin],
                                                     uint32_t src, uint32_t swz, double (&G)[NLB],
                                                     uint32_t (&m)[NLB], double (&Gn)[NLB], uint32_t (&mn)[NLB],
                                                     bool nxt) {
    // nxt: the event belongs to the trial after the one G accumulates (rounds
    // packed across a trial boundary): it is added to Gn / mn instead
    constexpr int CAP = (kPackBytes - 8) / (int)sizeof(TV);
    constexpr bool SM = true;   // lanes look up different columns: shared memory, not the constant bank
    uint32_t mask, e;
    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(mask), "=r"(e) : "r"(src + (swz << 4)) : "memory");
    // one pass over the window's non-zeros (ascending column), every layer of
    // the launch accumulating its own l_e in that order
    double le[NLB];
#pragma unroll
    for (int l = 0; l < NLB; ++l) le[l] = 0.0;
    auto add = [&](double x, uint32_t j) {
#pragma unroll
        for (int l = 0; l < NLB; ++l) {
            if (l == 0 || l < (int)p.n_layers) {   // a launch has >= 1 layer
                const double2 tc = SM ? lds_term(&s_term[l][j]) : p.term[l][j];
                le[l] = __dadd_rn(le[l], terms(x, tc.x, tc.y));
            }
        }
    };
    auto lds_val = [&](uint32_t o) {   // value at byte o of the staged slot
        const uint32_t a = src + (((o >> 4) ^ swz) << 4) + (o & 15u);
        double x;
        if (sizeof(TV) == 8) {
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a) : "memory");
        } else {
            float xf;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xf) : "r"(a) : "memory");
            x = (double)xf;
        }
        return x;
    };
    if (__popc(mask) <= CAP) {
        // the slot holds all of the row's non-zeros (the common case): walk
        // them in column order, the v-th at byte 8 + v * esz
        uint32_t mm = mask, o = 8u;
        while (mm) {
            const uint32_t b = (uint32_t)(__ffs(mm) - 1);
            mm &= mm - 1u;
            const uint32_t j = b - p.pk_col0;   // window element (wraps when b < col0)
            if (j < 32u && ((p.pk_wmask >> j) & 1u)) add(lds_val(o), j);
            o += (uint32_t)sizeof(TV);
        }
    } else {
        // more non-zeros than the slot holds: the first CAP from the slot,
        // the rest from the dense table
        uint32_t mm = (mask >> p.pk_col0) & p.pk_wmask;
        while (mm) {
            const uint32_t j = (uint32_t)(__ffs(mm) - 1);
            mm &= mm - 1u;
            const uint32_t v = __popc(mask & ((1u << (j + p.pk_col0)) - 1u));   // rank among the row's non-zeros
            const double x = v < (uint32_t)CAP
                                 ? lds_val(8u + v * (uint32_t)sizeof(TV))
                                 : (double)__ldg(static_cast<const TV*>(p.table) + p.sec_off[0] +
                                                 (uint64_t)e * p.row_stride + j);
            add(x, j);
        }
    }
#pragma unroll
    for (int l = 0; l < NLB; ++l) {
        if (l >= (int)p.n_layers) break;
        const double o = terms(le[l], p.lw[l].occ_r, p.lw[l].occ_l);
        if (nxt) {
            Gn[l] = __dadd_rn(Gn[l], o);
            mn[l] += (o > 0.0) ? 1u : 0u;
        } else {
            G[l] = __dadd_rn(G[l], o);
            m[l] += (o > 0.0) ? 1u : 0u;
        }
    }
}

// The same for a multi-window launch: the staged row belongs to the window of
// layer u (one layer per window); only that layer's accumulators change.
template <typename TV, int NSEC, int NLB>
__device__ __forceinline__ void event_compute_sparse_win(const TrialParams& p, const double2 (*s_term)[kMaxWin],
                                                         uint32_t src, uint32_t swz, double (&G)[NLB],
                                                         uint32_t (&m)[NLB], uint32_t u) {
    constexpr int CH = NSEC * 2;
    constexpr int EPC = 16 / (int)sizeof(TV);
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
    uint32_t nz = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        const uint4 v = lds_v4(src + (((uint32_t)c ^ swz) << 4));
        if (EPC == 2) {
            nz |= ((v.x | v.y) != 0u ? 1u : 0u) << (2 * c);
            nz |= ((v.z | v.w) != 0u ? 1u : 0u) << (2 * c + 1);
        } else {
            nz |= (v.x != 0u ? 1u : 0u) << (4 * c);
            nz |= (v.y != 0u ? 1u : 0u) << (4 * c + 1);
            nz |= (v.z != 0u ? 1u : 0u) << (4 * c + 2);
            nz |= (v.w != 0u ? 1u : 0u) << (4 * c + 3);
        }
    }
    double le = 0.0;
    while (nz) {
        const uint32_t j = (uint32_t)(__ffs(nz) - 1);
        nz &= nz - 1u;
        const uint32_t a = src + (((j / EPC) ^ swz) << 4) + (j % EPC) * (uint32_t)sizeof(TV);
        double x;
        if (EPC == 2) {
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(a) : "memory");
        } else {
            float xf;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(xf) : "r"(a) : "memory");
            x = (double)xf;
        }
        const double2 tc = SM ? lds_term(&s_term[u][j]) : p.term[u][j];
        le = __dadd_rn(le, terms(x, tc.x, tc.y));
    }
    const double o = terms(le, p.lw[u].occ_r, p.lw[u].occ_l);
    const uint32_t hit = (o > 0.0) ? 1u : 0u;
#pragma unroll
    for (int l = 0; l < NLB; ++l) {
        const double gl = __dadd_rn(G[l], o);
        G[l] = (l == (int)u) ? gl : G[l];
        m[l] += (l == (int)u) ? hit : 0u;
    }
}

// Events per lane per pipeline step (~16-32 row registers per stage); windows
// wider than 32 registers run without the row double buffer (PIPE = false).
template <typename TV, int NSEC>
struct Batch {
    static constexpr int R = NSEC * SecT<TV>::N * (int)sizeof(TV) / 4;   // row registers per event
    static constexpr int QB = R >= 16 ? 1 : (R >= 8 ? 2 : 4);
    static constexpr bool PIPE = R <= 32;
};

// L2 prefetch of one event's window (no register destination: CCTL.E.PF2).
__device__ __forceinline__ void prefetch_l2(const void* ptr) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
}

// D = id-queue depth: rows of step i+1 are demand-loaded into registers while
// step i is computed; for D > 1 the rows of step i+D are also prefetched into
// L2 (no registers held), so the demand loads mostly hit L2.
// Warp-level trial scheduler.  Static: trials gw, gw+nw, ... (work_ctr ==
// null).  Dynamic: batches of p.batch consecutive trials claimed from a
// global counter shared by every warp of every kernel of the launch group —
// this is what lets the LDG and TMA kernels run side by side (hybrid) and
// balance themselves.  Per-trial arithmetic does not depend on which warp
// takes a trial, so the YLT bits do not either.
struct TrialSched {
    uint64_t cur, end, stride;
    bool dyn;
    __device__ __forceinline__ void init(const TrialParams& p, uint64_t gw, uint64_t nw) {
        dyn = p.work_ctr != nullptr;
        if (dyn) { cur = end = 0; stride = 0; }
        else { cur = p.t_begin + gw; end = ~0ull; stride = nw; }
    }
    // next trial index for this warp, or ~0 when the range is exhausted
    __device__ __forceinline__ uint64_t next(const TrialParams& p) {
        if (!dyn) {
            const uint64_t t = cur;
            cur += stride;
            return t < p.t_end ? t : ~0ull;
        }
        if (cur >= end) {
            unsigned long long b = 0;
            if ((threadIdx.x & 31u) == 0) b = atomicAdd(p.work_ctr, (unsigned long long)p.batch);
            b = __shfl_sync(0xffffffffu, b, 0);
            cur = p.t_begin + b;
            end = cur + p.batch < p.t_end ? cur + p.batch : p.t_end;
            if (cur >= p.t_end) { end = cur; return ~0ull; }
        }
        return cur++;
    }
};

template <typename TV, int NSEC, int NLB, int D, int MINB = 2>
__global__ void __launch_bounds__(kThreads, MINB) trial_kernel(const __grid_constant__ TrialParams p) {
    constexpr int QB = Batch<TV, NSEC>::QB;
    constexpr bool PIPE = Batch<TV, NSEC>::PIPE;
    constexpr uint64_t STEP = 32u * QB;
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
    using R = Row<TV, NSEC>;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t gw = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const uint64_t nw = (uint64_t(gridDim.x) * kThreads) >> 5;
    const uint64_t pol = policy_evict_first();
    const uint64_t base = __ldg(p.off);
    uint32_t err = 0;
    __shared__ double2 s_term[SM ? NLB : 1][kMaxWin];
    if (SM) {
        for (int i = threadIdx.x; i < NLB * kMaxWin; i += kThreads)
            s_term[i / kMaxWin][i % kMaxWin] = p.term[i / kMaxWin][i % kMaxWin];
        __syncthreads();
    }

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
        double G[NLB];
        uint32_t m[NLB];
#pragma unroll
        for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }

        // Event k of the trial -> lane k % 32, visited in increasing k.
        // Software pipeline: ids two steps ahead, rows one step ahead.
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
        auto prefetch_rows = [&](const uint32_t (&e)[QB]) {
#pragma unroll
            for (int q = 0; q < QB; ++q) {
                const TV* row = static_cast<const TV*>(p.table) + (uint64_t)e[q] * p.row_stride;
#pragma unroll
                for (int sct = 0; sct < NSEC; ++sct)
                    if (sct < p.pf_sectors) prefetch_l2(row + p.sec_off[sct]);
            }
        };
        if (PIPE) {
            uint32_t qe[D][QB];   // ids of steps i+1 .. i+D
            R r0[QB];
            {
                uint32_t e0[QB];
                load_ids(0, e0);
#pragma unroll
                for (int d = 0; d < D; ++d) load_ids((d + 1) * STEP, qe[d]);
#pragma unroll
                for (int q = 0; q < QB; ++q) r0[q].load(p, e0[q]);
#pragma unroll
                for (int d = 1; d < D; ++d)
                    if ((d + 1) * STEP < n) prefetch_rows(qe[d]);
            }
#pragma unroll 1
            for (uint64_t k0 = 0; k0 < n; k0 += STEP) {
                uint32_t en[QB];
                load_ids(k0 + (D + 1) * STEP, en);
                if (D > 1 && k0 + D * STEP < n) prefetch_rows(qe[D - 1]);
                R r1[QB];
                if (k0 + STEP < n) {
#pragma unroll
                    for (int q = 0; q < QB; ++q) r1[q].load(p, qe[0][q]);
                }
#pragma unroll
                for (int q = 0; q < QB; ++q) event_compute<TV, NSEC, NLB>(p, s_term, r0[q], G, m);
#pragma unroll
                for (int q = 0; q < QB; ++q) {
                    r0[q] = r1[q];
#pragma unroll
                    for (int d = 0; d + 1 < D; ++d) qe[d][q] = qe[d + 1][q];
                    qe[D - 1][q] = en[q];
                }
            }
        } else {
            uint32_t e1[QB];
            load_ids(0, e1);
#pragma unroll 1
            for (uint64_t k0 = 0; k0 < n; k0 += STEP) {
                uint32_t e2[QB];
                load_ids(k0 + STEP, e2);
                R r0[QB];
#pragma unroll
                for (int q = 0; q < QB; ++q) r0[q].load(p, e1[q]);
#pragma unroll
                for (int q = 0; q < QB; ++q) event_compute<TV, NSEC, NLB>(p, s_term, r0[q], G, m);
#pragma unroll
                for (int q = 0; q < QB; ++q) e1[q] = e2[q];
            }
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
            store_trial(p, t, G, m);
        }
    }
    peer_fence(p);
    if (err) atomicOr(p.err, err);
}

// ---------------------------------------------------------------------------
// Shared-memory staged variant (default for the paper-shaped path).  The
// register-pipelined kernel above can keep at most ~2 row windows per lane in
// flight before the register file (256 KB/SM) is exhausted; with 128-B windows
// that is too little memory-level parallelism to cover loaded DRAM latency
// (ncu: long-scoreboard stalls, DRAM ~55 % busy).  Here each lane copies its
// event's window straight into a per-warp shared-memory ring with cp.async
// (LDGSTS, no registers held), NS steps deep, so ~(NS-1) x 4 KB per warp is in
// flight continuously; the fp64 arithmetic reads the window back with swizzled
// (bank-conflict-free) LDS.128.  The ring runs across trial boundaries: a step
// iterator two steps ahead loads ids, the producer issues step j, the consumer
// retires step j-(NS-1) and finishes a trial on its last step.  Same lane
// mapping, same per-lane order, same arithmetic as trial_kernel: identical
// YLT bits.
struct StepMeta {
    uint64_t t;      // trial (UINT64_MAX: no more steps)
    uint32_t n, k0;  // trial length, first event index of the step
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename TV, int NSEC>
struct SmGeo {
    static constexpr int WARPS = kThreads / 32;
    static constexpr int CH = NSEC * 2;                // 16-B chunks per lane slot
    static constexpr int SLOT = CH * 16;               // bytes per lane slot
    static constexpr int STAGE = 32 * SLOT;            // bytes per warp stage
    static constexpr int NS0 = (196 * 1024) / (WARPS * STAGE);
    static constexpr int NS = NS0 > 8 ? 8 : (NS0 < 2 ? 2 : NS0);
    static constexpr int RING = WARPS * NS * STAGE;
    static constexpr int BYTES = RING + WARPS * NS * (int)sizeof(StepMeta);
};

template <typename TV, int NSEC, int NLB>
__global__ void __launch_bounds__(kThreads, 1) trial_kernel_sm(const __grid_constant__ TrialParams p) {
    using Geo = SmGeo<TV, NSEC>;
    constexpr int NS = Geo::NS, CH = Geo::CH;
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double2 s_term[SM ? NLB : 1][kMaxWin];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + wib * NS * Geo::STAGE + lane * Geo::SLOT;
    StepMeta* meta = reinterpret_cast<StepMeta*>(smem + Geo::RING) + wib * NS;
    if (SM) {
        for (int i = threadIdx.x; i < NLB * kMaxWin; i += kThreads)
            s_term[i / kMaxWin][i % kMaxWin] = p.term[i / kMaxWin][i % kMaxWin];
    }
    __syncthreads();

    const uint64_t nw = (uint64_t)gridDim.x * Geo::WARPS;
    const uint64_t pol = policy_evict_first();
    const uint64_t base = __ldg(p.off);
    const TV* tab = static_cast<const TV*>(p.table);
    uint32_t err = 0;

    // ---- id iterator (two steps ahead of the producer)
    uint64_t it_t = p.t_begin + (uint64_t)blockIdx.x * Geo::WARPS + wib;
    uint64_t it_a = 0, nx_a = 0, nx_b = 0;
    uint32_t it_n = 0, it_k0 = 0;
    bool it_valid = it_t < p.t_end;
    auto fetch_next_offsets = [&](uint64_t tn) {
        if (tn < p.t_end) { nx_a = __ldg(p.off + tn); nx_b = __ldg(p.off + tn + 1); }
    };
    auto enter_trial = [&](uint64_t a, uint64_t b) {
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        it_a = a - base;
        it_n = (uint32_t)(b - a);
        it_k0 = 0;
    };
    if (it_valid) {
        enter_trial(__ldg(p.off + it_t), __ldg(p.off + it_t + 1));
        fetch_next_offsets(it_t + nw);
    }
    auto it_advance = [&]() {
        it_k0 += 32u;
        if (it_k0 >= it_n) {
            it_t += nw;
            it_valid = it_t < p.t_end;
            if (it_valid) {
                enter_trial(nx_a, nx_b);
                fetch_next_offsets(it_t + nw);
            }
        }
    };
    // queue of two steps whose ids are in flight
    uint64_t q_t[2];
    uint32_t q_n[2], q_k0[2], q_e[2];
    uint64_t q_a[2];
    auto load_step = [&](int slot) {
        if (it_valid) {
            q_t[slot] = it_t;
            q_a[slot] = it_a;
            q_n[slot] = it_n;
            q_k0[slot] = it_k0;
            const uint32_t k = it_k0 + lane;
            uint32_t v = 0u;
            if (k < it_n) {
                v = ld_stream_u32(p.ids + it_a + k, pol);
                if (v == 0u || v > p.catalog) { err |= ERRBIT_EVENT_RANGE; v = 0u; }
            }
            q_e[slot] = v;
            it_advance();
        } else {
            q_t[slot] = ~0ull;
            q_e[slot] = 0u;
        }
    };
    load_step(0);
    load_step(1);

    double G[NLB];
    uint32_t m[NLB];
#pragma unroll
    for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }

#pragma unroll 1
    for (uint32_t j = 0;; ++j) {
        // ---- producer: issue the rows of step j into ring slot j % NS
        {
            const uint64_t ct = q_t[0];
            const uint32_t cn = q_n[0], ck0 = q_k0[0], ce = q_e[0];
            q_t[0] = q_t[1]; q_n[0] = q_n[1]; q_k0[0] = q_k0[1]; q_e[0] = q_e[1]; q_a[0] = q_a[1];
            load_step(1);
            const uint32_t slot = j % NS;
            if (ct != ~0ull) {
                const TV* row = tab + (uint64_t)ce * p.row_stride;
                const uint32_t src_bytes = ce ? 16u : 0u;   // lanes without an event: zero-fill
                const uint32_t dst = ring + slot * Geo::STAGE;
#pragma unroll
                for (int c = 0; c < CH; ++c) {
                    const TV* src = row + p.sec_off[c >> 1] + (c & 1) * (8 / sizeof(TV) * 2);
                    cp_async16(dst + ((c ^ (lane & (CH - 1))) << 4), src, src_bytes);
                }
            }
            if (lane == 0) meta[slot] = StepMeta{ct, cn, ck0};
            cp_commit();
        }
        // ---- consumer: retire step j - (NS - 1)
        if (j + 1 >= (uint32_t)NS) {
            cp_wait<NS - 1>();
            __syncwarp();
            const uint32_t slot = (j + 1) % NS;   // == (j - (NS - 1)) % NS
            const StepMeta md = meta[slot];
            if (md.t == ~0ull) break;
            Row<TV, NSEC> r;
            const uint32_t src = ring + slot * Geo::STAGE;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(src + ((c ^ (lane & (CH - 1))) << 4)));
                memcpy(&r.x[c >> 1][(c & 1) * (16 / sizeof(TV))], &v, 16);
            }
            event_compute<TV, NSEC, NLB>(p, s_term, r, G, m);
            if (md.k0 + 32u >= md.n) {   // last step of trial md.t: a7 + a8
#pragma unroll
                for (int l = 0; l < NLB; ++l) {
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) {
                        G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
                        m[l] += __shfl_xor_sync(0xffffffffu, m[l], off);
                    }
                }
                if (lane == 0) {
                    const uint64_t t = md.t;
                    store_trial(p, t, G, m);
                }
#pragma unroll
                for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }
            }
            __syncwarp();
        }
    }
    cp_wait<0>();
    if (err) atomicOr(p.err, err);
}

// ---------------------------------------------------------------------------
// TMA variant (default for fp64 128-B windows).  The row windows are gathered
// by the Tensor Memory Accelerator with tile::gather4 (4 rows per instruction,
// UTMALDG.2D.GATHER4) into a per-warp shared-memory ring NS stages deep; an
// mbarrier per stage counts the landed bytes (complete_tx).  No registers are
// held by in-flight rows, so ~(NS-1) x 4 KB per warp stays in flight and the
// TMA's own address translation keeps the random 128-B gathers off the LSU
// and TLB paths (measured: 9.5 TB/s vs 8.0 TB/s for LDG gathers of 128-B rows
// from a 256 MB table, tools/microbench.py).  The TMA box is the layer's
// window in its column block, swizzled (128/64/32B) so that each lane's read
// of its own row is bank-conflict free.  Same lane mapping, per-lane order
// and arithmetic as trial_kernel: identical YLT bits.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_gather4(uint32_t dst, const CUtensorMap* map, uint32_t bar, int32_t col,
                                            uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst), "l"(map), "r"(bar), "r"(col), "r"(r0), "r"(r1),
        "r"(r2), "r"(r3)
        : "memory");
}

template <typename TV, int NSEC>
struct TmaGeo {
    static constexpr int WARPS = kThreads / 32;
    static constexpr int ROWB = NSEC * kSectorBytes;   // bytes per gathered row (= TMA box)
    static constexpr int CH = ROWB / 16;
    static constexpr int STAGE = 32 * ROWB;            // one row per lane
    static constexpr int NS0 = (192 * 1024) / (WARPS * STAGE);
    static constexpr int NS = NS0 > 8 ? 8 : (NS0 < 2 ? 2 : NS0);
    static constexpr int BYTES = WARPS * NS * STAGE + 1024;   // + alignment slack
};

template <typename TV, int NSEC, int NLB>
__global__ void __launch_bounds__(kThreads, 1) trial_kernel_tma(const __grid_constant__ TrialParams p) {
    using Geo = TmaGeo<TV, NSEC>;
    constexpr int NS = Geo::NS, CH = Geo::CH;
    constexpr int QD = 8;              // id stage runs QD steps ahead of the gathers
    constexpr int IR = QD + 1;         // id ring slots
    constexpr int MR = QD + NS;        // step-metadata ring slots
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
    extern __shared__ unsigned char smem_dyn[];
    __shared__ __align__(8) uint64_t bars[Geo::WARPS][NS];
    __shared__ StepMeta meta[Geo::WARPS][MR];
    __shared__ __align__(16) uint32_t idring[Geo::WARPS][IR][32];
    __shared__ double2 s_term[SM ? NLB : 1][kMaxWin];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t sbase = ((uint32_t)__cvta_generic_to_shared(smem_dyn) + 1023u) & ~1023u;
    const uint32_t ring = sbase + wib * NS * Geo::STAGE;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&bars[wib][0]);
    const uint32_t id0 = (uint32_t)__cvta_generic_to_shared(&idring[wib][0][0]);
    if (lane == 0)
        for (int s = 0; s < NS; ++s) mbar_init(bar0 + 8u * s, 1u);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (SM) {
        for (int i = threadIdx.x; i < NLB * kMaxWin; i += kThreads)
            s_term[i / kMaxWin][i % kMaxWin] = p.term[i / kMaxWin][i % kMaxWin];
    }
    __syncthreads();

    const uint64_t nw = (uint64_t)gridDim.x * Geo::WARPS;
    const uint64_t base = __ldg(p.off);
    uint32_t err = 0;
    // lane's conflict-free chunk permutation (matches the map's swizzle mode)
    const uint32_t swz = (lane * (uint32_t)Geo::ROWB / 128u) & (uint32_t)(CH - 1);

    // ---- id stage: a step iterator QD steps ahead of the gathers.  Each lane
    // copies its event id of the step straight into the id ring (cp.async,
    // zero-filled past the trial's end); lane 0 records the step metadata.
    TrialSched sched;
    sched.init(p, (uint64_t)blockIdx.x * Geo::WARPS + wib, nw);
    uint64_t it_t = sched.next(p), it_tn = sched.next(p);
    uint64_t it_a = 0, nx_a = 0, nx_b = 0;
    uint32_t it_n = 0, it_k0 = 0;
    bool it_valid = it_t != ~0ull;
    auto fetch_next_offsets = [&](uint64_t tn) {
        if (tn != ~0ull) { nx_a = __ldg(p.off + tn); nx_b = __ldg(p.off + tn + 1); }
    };
    auto enter_trial = [&](uint64_t a, uint64_t b) {
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        it_a = a - base;
        it_n = (uint32_t)(b - a);
        it_k0 = 0;
    };
    if (it_valid) {
        enter_trial(__ldg(p.off + it_t), __ldg(p.off + it_t + 1));
        fetch_next_offsets(it_tn);
    }
    auto id_stage = [&](uint32_t step) {
        StepMeta md{~0ull, 0u, 0u};
        if (it_valid) {
            md = StepMeta{it_t, it_n, it_k0};
            const uint32_t k = it_k0 + lane;
            const uint32_t* src = p.ids + it_a + (k < it_n ? k : 0u);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(id0 + ((step % IR) * 32u + lane) * 4u),
                         "l"(src), "r"(k < it_n ? 4u : 0u)
                         : "memory");
            it_k0 += 32u;
            if (it_k0 >= it_n) {
                it_t = it_tn;
                it_valid = it_t != ~0ull;
                if (it_valid) {
                    enter_trial(nx_a, nx_b);
                    it_tn = sched.next(p);
                    fetch_next_offsets(it_tn);
                }
            }
        }
        if (lane == 0) meta[wib][step % MR] = md;
        cp_commit();
    };
    for (uint32_t s = 0; s < (uint32_t)QD; ++s) id_stage(s);

    double G[NLB];
    uint32_t m[NLB];
#pragma unroll
    for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }
    const int32_t col = (int32_t)p.tma_col;

#pragma unroll 1
    for (uint32_t j = 0;; ++j) {
        id_stage(j + QD);
        // ---- producer: ids of step j are in the ring; gather its rows into slot j % NS
        cp_wait<QD>();
        __syncwarp();
        {
            const StepMeta md = meta[wib][j % MR];
            const uint32_t slot = j % NS;
            if (md.t != ~0ull) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the slot
                if (lane == 0) mbar_expect_tx(bar0 + 8u * slot, (uint32_t)Geo::STAGE);
                __syncwarp();
                if (lane < 8u) {
                    uint4 e4;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(e4.x), "=r"(e4.y), "=r"(e4.z), "=r"(e4.w)
                                 : "r"(id0 + ((j % IR) * 32u + lane * 4u) * 4u));
                    uint32_t e[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {   // fused YET validation (A14)
                        const bool live = md.k0 + lane * 4u + i < md.n;
                        if (live && (e[i] == 0u || e[i] > p.catalog)) err |= ERRBIT_EVENT_RANGE;
                        if (!live || e[i] > p.catalog) e[i] = 0u;
                    }
                    tma_gather4(ring + slot * Geo::STAGE + lane * 4u * Geo::ROWB, &p.tmap, bar0 + 8u * slot, col,
                                e[0], e[1], e[2], e[3]);
                }
            }
        }
        // ---- consumer: retire step c = j - (NS - 1)
        if (j + 1 >= (uint32_t)NS) {
            const uint32_t c = j + 1 - NS;
            const uint32_t slot = c % NS;
            const StepMeta md = meta[wib][c % MR];
            if (md.t == ~0ull) break;
            mbar_wait(bar0 + 8u * slot, (c / NS) & 1u);
            Row<TV, NSEC> r;
            const uint32_t src = ring + slot * Geo::STAGE + lane * Geo::ROWB;
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                uint4 v;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                             : "r"(src + (((uint32_t)q ^ swz) << 4)));
                memcpy(&r.x[q >> 1][(q & 1) * (16 / sizeof(TV))], &v, 16);
            }
            event_compute<TV, NSEC, NLB>(p, s_term, r, G, m);
            if (md.k0 + 32u >= md.n) {   // last step of trial md.t: a7 + a8
#pragma unroll
                for (int l = 0; l < NLB; ++l) {
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) {
                        G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
                        m[l] += __shfl_xor_sync(0xffffffffu, m[l], off);
                    }
                }
                if (lane == 0) {
                    const uint64_t t = md.t;
                    store_trial(p, t, G, m);
                }
#pragma unroll
                for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }
            }
        }
        __syncwarp();   // id-ring / slot reads of this iteration precede the next writes
    }
    cp_wait<0>();
    if (err) atomicOr(p.err, err);
}

// ---------------------------------------------------------------------------
// Cooperative cp.async ring.  Like trial_kernel_sm, the row windows of a step
// land in a per-warp shared-memory ring NS steps deep, so in-flight rows hold
// no registers and the ring runs across trial boundaries (no pipeline drain
// per trial).  Unlike trial_kernel_sm (each lane copying its own row in 16-B
// pieces, which re-fetches every 32-B sector twice), each cp.async
// instruction here copies 32/CH whole rows, CH lanes per row, so one warp
// request covers every sector of a row exactly once — the L2->SM traffic
// equals the algorithmic bytes.  Rows are stored with a per-row chunk swizzle
// so that each lane's read of its own row is bank-conflict free.  Same lane
// mapping, per-lane order and arithmetic as trial_kernel: identical YLT bits.
template <typename TV, int NSEC, int BUDGET_KB>
struct CoGeo {
    static constexpr int WARPS = kThreads / 32;
    static constexpr int ROWB = NSEC * kSectorBytes;   // bytes per row window
    static constexpr int CH = ROWB / 16;               // 16-B chunks per row
    static constexpr int LPR = CH < 32 ? CH : 32;      // lanes per row in one copy instruction
    static constexpr int RPI = 32 / LPR;               // rows per copy instruction
    static constexpr int STAGE = 32 * ROWB;            // one row per lane
    static constexpr int NS0 = (BUDGET_KB * 1024) / (WARPS * (STAGE + (int)sizeof(StepMeta)));
    static constexpr int NS = NS0 > 16 ? 16 : (NS0 < 1 ? 1 : NS0);   // 1: compacted rounds only
    static constexpr int BYTES = WARPS * NS * STAGE + WARPS * NS * (int)sizeof(StepMeta);
    // conflict-free chunk permutation of row r (8 consecutive rows of a
    // quarter-warp phase hit 8 distinct 16-B bank groups)
    static __device__ __forceinline__ uint32_t swz(uint32_t r) {
        return (r * (uint32_t)ROWB / 128u) & (uint32_t)(CH - 1);
    }
};

template <typename TV, int NSEC, int NLB, int BUDGET_KB, int MINB, bool EARLY>
__global__ void __launch_bounds__(kThreads, MINB) trial_kernel_co(const __grid_constant__ TrialParams p) {
    using Geo = CoGeo<TV, NSEC, BUDGET_KB>;
    constexpr int NS = Geo::NS;
    constexpr int CH = Geo::CH, LPR = Geo::LPR, RPI = Geo::RPI;
    constexpr bool SM = TermsInSmem<TV, NSEC, NLB>::value;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double2 s_term[SM ? NLB : 1][kMaxWin];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + wib * NS * Geo::STAGE;
    StepMeta* meta = reinterpret_cast<StepMeta*>(smem + Geo::WARPS * NS * Geo::STAGE) + wib * NS;
    if (SM) {
        for (int i = threadIdx.x; i < NLB * kMaxWin; i += kThreads)
            s_term[i / kMaxWin][i % kMaxWin] = p.term[i / kMaxWin][i % kMaxWin];
    }
    __syncthreads();

    const uint64_t nw = (uint64_t)gridDim.x * Geo::WARPS;
    const uint64_t pol = policy_evict_first();
    const uint64_t base = __ldg(p.off);
    uint32_t err = 0;
    // This lane's part of every cooperative copy: chunk c_chunk of row
    // i * RPI + c_row in copy instruction i.  Row addresses are one
    // IMAD.WIDE.U32 (id x row bytes + per-lane base); the destination's
    // swizzle repeats with period 2 in i (swz(i*RPI + c_row) for any window).
    const uint32_t c_chunk = lane % LPR, c_row = lane / LPR;
    const uint32_t row_bytes = (uint32_t)(p.row_stride * sizeof(TV));
    const char* c_src = reinterpret_cast<const char*>(p.table) +
                        (p.sec_off[c_chunk >> 1] + (c_chunk & 1) * (16 / sizeof(TV))) * sizeof(TV);
    uint32_t c_dst[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t r = (uint32_t)h * RPI + c_row;
        c_dst[h] = c_row * Geo::ROWB + ((c_chunk ^ Geo::swz(r)) << 4);
    }
    const uint32_t my_row = ring + lane * Geo::ROWB;
    const uint32_t my_swz = Geo::swz(lane);

    // ---- step iterator (ids two steps ahead of the copies)
    uint64_t it_t = p.t_begin + (uint64_t)blockIdx.x * Geo::WARPS + wib;
    uint64_t it_a = 0, nx_a = 0, nx_b = 0;
    uint32_t it_n = 0, it_k0 = 0;
    bool it_valid = it_t < p.t_end;
    auto fetch_next_offsets = [&](uint64_t tn) {
        if (tn < p.t_end) { nx_a = __ldg(p.off + tn); nx_b = __ldg(p.off + tn + 1); }
    };
    auto enter_trial = [&](uint64_t a, uint64_t b) {
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        it_a = a - base;
        it_n = (uint32_t)(b - a);
        it_k0 = 0;
    };
    if (it_valid) {
        enter_trial(__ldg(p.off + it_t), __ldg(p.off + it_t + 1));
        fetch_next_offsets(it_t + nw);
    }
    // Two-slot queue of steps whose ids are in flight; step j lives in slot
    // j & 1 (compile-time below: the loops are unrolled by two).
    uint64_t q_t[2];
    uint32_t q_n[2], q_k0[2], q_e[2], q_w[2];
    auto load_step = [&](const int slot) {
        if (it_valid) {
            q_t[slot] = it_t;
            q_n[slot] = it_n;
            q_k0[slot] = it_k0;
            const uint32_t k = it_k0 + lane;
            uint32_t v = 0u;
            if (k < it_n) {
                v = ld_stream_u32(p.ids + it_a + k, pol);
                if (v == 0u || v > p.catalog) { err |= ERRBIT_EVENT_RANGE; v = 0u; }
            }
            q_e[slot] = v;
            it_k0 += 32u;
            if (it_k0 >= it_n) {
                it_t += nw;
                it_valid = it_t < p.t_end;
                if (it_valid) {
                    enter_trial(nx_a, nx_b);
                    fetch_next_offsets(it_t + nw);
                }
            }
        } else {
            q_t[slot] = ~0ull;
            q_e[slot] = 0u;
        }
    };
    // copy the rows of step j (queue slot j & 1) into ring slot j % NS, then
    // reuse the queue slot for the ids of step j + 2
    // The occupancy word of a step's id is fetched one iteration after the id
    // (and one before the copies): a clear bit marks an all-zero row, whose
    // copy becomes a zero-fill with no memory request.  The arithmetic is
    // unchanged (it runs on the zeros), so the YLT bits are too.
    const uint32_t* bm = p.bm;
    auto load_occupancy = [&](const int slot) {
        q_w[slot] = bm ? __ldg(bm + (q_e[slot] >> 5)) : ~0u;
    };
    auto issue = [&](const uint32_t j, const int qs) {
        const uint64_t ct = q_t[qs];
        const uint32_t cn = q_n[qs], ck0 = q_k0[qs];
        const uint32_t ce = ((q_w[qs] >> (q_e[qs] & 31u)) & 1u) ? q_e[qs] : 0u;
        load_occupancy(qs ^ 1);
        load_step(qs);
        const uint32_t slot = j % NS;
        if (ct != ~0ull) {
            const uint32_t dst = ring + slot * Geo::STAGE;
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                const uint32_t e = __shfl_sync(0xffffffffu, ce, (uint32_t)i * RPI + c_row);
                // rows without an event (e == 0): zero-fill, no memory request
                cp_async16(dst + (uint32_t)i * RPI * Geo::ROWB + c_dst[i & 1], c_src + (uint64_t)e * row_bytes,
                           e ? 16u : 0u);
            }
        }
        if (lane == 0) meta[slot] = StepMeta{ct, cn, ck0};
        cp_commit();
    };
    load_step(0);
    load_occupancy(0);
    load_step(1);
#pragma unroll
    for (int j = 0; j < NS; ++j) issue((uint32_t)j, j & 1);

    double G[NLB];
    uint32_t m[NLB];
#pragma unroll
    for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }

    // consumer: step c lands, its rows move to registers, the slot is
    // refilled with step c + NS (before or after the fp64 work, EARLY).
#pragma unroll 1
    for (uint32_t c0 = 0;; c0 += 2) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t c = c0 + (uint32_t)h;
            cp_wait<NS - 1>();
            __syncwarp();   // other lanes' copies of my row are complete and visible
            const uint32_t slot = c % NS;
            const StepMeta md = meta[slot];
            if (md.t == ~0ull) goto done;
            const uint32_t src = my_row + slot * Geo::STAGE;
            if (EARLY) {
                Row<TV, NSEC> r;
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    uint4 v;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                                 : "r"(src + (((uint32_t)q ^ my_swz) << 4))
                                 : "memory");
                    memcpy(&r.x[q >> 1][(q & 1) * (16 / sizeof(TV))], &v, 16);
                }
                __syncwarp();   // every lane's reads of the slot precede the copies refilling it
                issue(c + NS, (h + NS) & 1);   // NS steps in flight during the arithmetic
                event_compute<TV, NSEC, NLB>(p, s_term, r, G, m);
            } else {
                // the row is consumed from shared memory one sector at a time
                // (8 live row registers instead of 32), then the slot is refilled
                event_compute_smem<TV, NSEC, NLB>(p, s_term, src, my_swz, G, m);
                __syncwarp();   // every lane's reads of the slot precede the copies refilling it
                issue(c + NS, (h + NS) & 1);
            }
            if (md.k0 + 32u >= md.n) {   // last step of trial md.t: a7 + a8
#pragma unroll
                for (int l = 0; l < NLB; ++l) {
#pragma unroll
                    for (int off = 16; off >= 1; off >>= 1) {
                        G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
                        m[l] += __shfl_xor_sync(0xffffffffu, m[l], off);
                    }
                }
                if (lane == 0) {
                    const uint64_t t = md.t;
                    store_trial(p, t, G, m);
                }
#pragma unroll
                for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }
            }
        }
    }
done:
    cp_wait<0>();
    peer_fence(p);
    if (err) atomicOr(p.err, err);
}

// ---------------------------------------------------------------------------
// Compacted rounds (sparse ELTs).  On the paper's ELTs most rows of the
// direct-access table are all zero (10k-30k losses per ELT over a catalogue of
// millions), and a zero row adds an exact +0 to every sum.  This kernel
// keeps the warp-per-trial mapping (event k -> lane k % 32, each lane in
// increasing k) but lets every lane skip its zero-row events: a scan stage
// walks the trial 32 events per step, tests each event's row in the
// occupancy bitmap and appends occupied events to a per-lane FIFO (QC deep);
// a round -- one occupied event per lane -- is emitted into the cooperative
// cp.async ring whenever a lane's FIFO is full and, at the end of the trial,
// until every FIFO is empty (the last round of a trial finalises it).  Each
// lane still adds its occupied events' losses in increasing k, so G per lane,
// the xor tree and the YLT bits equal trial_kernel's, while the fp64 term
// arithmetic runs once per round (~0.3 rounds per step at the paper's
// occupancy) instead of once per step.
//
// Latency: the scan's ids (QD steps ahead) and occupancy words (DW steps
// ahead) are cp.async copies into small per-warp rings, so nothing in flight
// holds a register; every copy belongs to a commit group whose sequence
// number is tracked, and each consumer waits for exactly the group it needs
// (cp.async.wait_group with a run-time count).
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
// Scan steps cover 128 events of one trial (4 sub-steps of 32: event
// k0 + 32 j + lane), so the fixed per-step work (waits, step metadata, the id
// iterator) is paid once per 128 events.  A step's ids arrive as one aligned
// 16-B-chunk copy of the id range (33 chunks); its occupancy words as one
// 4-B gather per event.
struct CqStep {
    uint64_t t;            // trial (UINT64_MAX: no more steps)
    uint32_t n, k0;        // trial length, first event of the step
    uint32_t sh, pad;      // position of event k0 in the step's id slot
};

template <int MINB_, int SE_ = 128>
struct CqRings {
    static constexpr int QD = 3;        // ids are copied QD steps ahead
    static constexpr int DW = 1;        // occupancy words DW steps ahead (QD >= 2 DW + 1)
    static constexpr int IR = QD + 1;   // id ring slots (SE/4 + 1 chunks of 16 B)
    static constexpr int WR = DW + 1;   // occupancy ring slots (SE x u32)
    static constexpr int MR = 8;        // step-meta ring slots (> QD)
    static constexpr int IDB = (SE_ / 4 + 1) * 16;
    static constexpr int BYTES = IR * IDB + WR * SE_ * 4 + MR * (int)sizeof(CqStep);   // per warp
};

template <typename TV, int NSEC, int BUDGET_KB, int MINB, int SE = 128>
struct CqGeo {
    using Ring = CoGeo<TV, NSEC, BUDGET_KB>;
    using R = CqRings<MINB, SE>;
    static constexpr int BYTES = Ring::WARPS * Ring::NS * Ring::STAGE + Ring::WARPS * Ring::NS * (int)sizeof(StepMeta) +
                                 Ring::WARPS * R::BYTES;
};

// cp.async.wait_group with a run-time count n, clamped to 7 (a smaller count
// only waits for more groups)
__device__ __forceinline__ void cp_wait_upto(uint32_t n) {
    if (n >= 4) {
        if (n >= 6) { if (n >= 7) cp_wait<7>(); else cp_wait<6>(); }
        else { if (n >= 5) cp_wait<5>(); else cp_wait<4>(); }
    } else {
        if (n >= 2) { if (n >= 3) cp_wait<3>(); else cp_wait<2>(); }
        else { if (n >= 1) cp_wait<1>(); else cp_wait<0>(); }
    }
}

template <typename TV, int NSEC, int NLB, int BUDGET_KB, int MINB, int NWIN, bool PK = false, bool OL = false,
          int SE = 128, bool XT = false>
__global__ void __launch_bounds__(kThreads, MINB) trial_kernel_cq(const __grid_constant__ TrialParams p) {
    // PK: the rounds gather packed rows (one 32-B slot per event, p.pk; NSEC == 1)
    // OL: a step's occupancy words are plain L1-cached loads into registers,
    //     issued one step ahead, instead of cp.async copies into the ring
    static_assert(!PK || (NSEC == 1 && NWIN == 1), "packed rounds: one sector per event, one window");
    static_assert(!OL || NWIN == 1, "register occupancy words: one window");
    // XT: rounds packed across trial boundaries -- a trial whose scan has
    // ended stays "pending" while the next trial's events enter the FIFOs
    // (tagged), so its last rounds also carry the next trial's events; each
    // lane adds a tagged event to a second accumulator, and the pending
    // trial is finalised with the round that pops its last event
    static_assert(!XT || PK, "cross-trial rounds: packed rows");
    // SE: events per scan step (SUB = SE / 32 sub-steps, scanned 4 at a time)
    static_assert(SE == 128 || (SE == 256 && NWIN == 1 && !OL), "256-event steps: one window, cp.async words");
    constexpr int SUB = SE / 32;
    constexpr int NCH = SE / 4 + 1;   // 16-B id chunks spanning a step's ids
    // NWIN == 1: one row window (layers 0..n_layers-1 share it: towers);
    // NWIN > 1: p.n_layers disjoint windows, one layer each, scanned together
    // (one id stream, one combined 4-bit occupancy word per event, one FIFO
    // per window; the last round of a trial is an empty finalising marker)
    static_assert(NWIN == 1 || NWIN == NLB, "one layer per window");
    using Geo = CoGeo<TV, NSEC, BUDGET_KB>;
    using RG = typename CqGeo<TV, NSEC, BUDGET_KB, MINB, SE>::R;
    constexpr int NS = Geo::NS;
    constexpr int CH = Geo::CH, LPR = Geo::LPR, RPI = Geo::RPI;
    constexpr int QD = RG::QD, DW = RG::DW, IR = RG::IR, WR = RG::WR, MR = RG::MR, IDB = RG::IDB;
    constexpr int QC = NWIN > 1 ? 2 : 6;   // per-lane FIFO of occupied events (per window)
    constexpr bool SM = PK || TermsInSmem<TV, NSEC, NLB>::value;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double2 s_term[SM ? NLB : 1][kMaxWin];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem) + wib * NS * Geo::STAGE;
    StepMeta* rmeta = reinterpret_cast<StepMeta*>(smem + Geo::WARPS * NS * Geo::STAGE) + wib * NS;
    unsigned char* wsm = smem + Geo::WARPS * NS * (Geo::STAGE + (int)sizeof(StepMeta)) + wib * RG::BYTES;
    const uint32_t idr = (uint32_t)__cvta_generic_to_shared(wsm);   // id ring [IR][33 x 16 B]
    const uint32_t ocr = idr + IR * IDB;                            // occupancy ring [WR][128]
    CqStep* smeta = reinterpret_cast<CqStep*>(wsm + IR * IDB + WR * SE * 4);
    if (SM) {
        for (int i = threadIdx.x; i < NLB * kMaxWin; i += kThreads)
            s_term[i / kMaxWin][i % kMaxWin] = p.term[i / kMaxWin][i % kMaxWin];
    }
    __syncthreads();

    const uint64_t nw = (uint64_t)gridDim.x * Geo::WARPS;
    const uint64_t base = __ldg(p.off);
    const uint32_t* bm = p.bm;
    uint32_t err = 0;
    const uint32_t c_chunk = lane % LPR, c_row = lane / LPR;
    const uint32_t row_bytes = PK ? (uint32_t)kPackBytes : (uint32_t)(p.row_stride * sizeof(TV));
    const char* c_src = PK ? static_cast<const char*>(p.pk) + c_chunk * 16u
                           : reinterpret_cast<const char*>(p.table) +
                                 (p.sec_off[c_chunk >> 1] + (c_chunk & 1) * (16 / sizeof(TV))) * sizeof(TV);
    uint32_t c_dst[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) c_dst[h] = c_row * Geo::ROWB + ((c_chunk ^ Geo::swz((uint32_t)h * RPI + c_row)) << 4);
    const uint32_t my_row = ring + lane * Geo::ROWB;
    const uint32_t my_swz = Geo::swz(lane);

    uint32_t gseq = 0;   // commit groups so far (warp-uniform)
    auto commit = [&]() { cp_commit(); return gseq++; };
    auto wait_group = [&](uint32_t g) { cp_wait_upto(gseq - 1u - g); };
    auto lds_u32 = [&](uint32_t a) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        return v;
    };

    // ---- fetch iterator: QD steps ahead of the scan
    uint64_t it_t = p.t_begin + (uint64_t)blockIdx.x * Geo::WARPS + wib;
    uint64_t it_a = 0, nx_a = 0, nx_b = 0;
    uint32_t it_n = 0, it_k0 = 0;
    bool it_valid = it_t < p.t_end;
    auto fetch_next_offsets = [&](uint64_t tn) {
        if (tn < p.t_end) { nx_a = __ldg(p.off + tn); nx_b = __ldg(p.off + tn + 1); }
    };
    auto enter_trial = [&](uint64_t a, uint64_t b) {
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        it_a = a - base;
        it_n = (uint32_t)(b - a);
        it_k0 = 0;
    };
    if (it_valid) {
        enter_trial(__ldg(p.off + it_t), __ldg(p.off + it_t + 1));
        fetch_next_offsets(it_t + nw);
    }
    // copy step x's ids (the 16-B chunks spanning them; bytes past the step's
    // last id are zero-filled, never read) and record the step's metadata;
    // validation happens at the scan
    auto fetch_ids = [&](uint32_t x) {
        CqStep md{~0ull, 0u, 0u, 0u, 0u};
        if (it_valid) {
            const uint32_t cnt = it_n - it_k0 < (uint32_t)SE ? it_n - it_k0 : (uint32_t)SE;
            const uintptr_t ab = reinterpret_cast<uintptr_t>(p.ids + it_a + it_k0);
            const char* al = reinterpret_cast<const char*>(ab & ~(uintptr_t)15);
            const uint32_t rem = (uint32_t)(ab & 15u) + 4u * cnt;   // bytes from al to the step's last id
            const uint32_t dst = idr + (x % IR) * IDB;
#pragma unroll
            for (int r = 0; r < (NCH + 31) / 32; ++r) {
                const uint32_t off = 16u * (lane + 32u * (uint32_t)r);
                if (32 * (r + 1) <= NCH || off < 16u * (uint32_t)NCH) {
                    const uint32_t nb = off >= rem ? 0u : (rem - off >= 16u ? 16u : rem - off);
                    cp_async16(dst + off, al + (nb ? off : 0u), nb);
                }
            }
            md = CqStep{it_t, it_n, it_k0, (uint32_t)(ab & 15u) / 4u, gseq};   // pad: the ids' commit group
            it_k0 += (uint32_t)SE;
            if (it_k0 >= it_n) {
                it_t += nw;
                it_valid = it_t < p.t_end;
                if (it_valid) {
                    enter_trial(nx_a, nx_b);
                    fetch_next_offsets(it_t + nw);
                }
            }
        }
        if (lane == 0) smeta[x % MR] = md;
    };
    // copy the occupancy words of step x's events (its ids have landed); the
    // lane's 4 ids stay in nid for the scan of step x (NWIN == 1: the words
    // land lane-major, [lane][j], so the scan reads its 4 with one load)
    uint32_t nid[SUB];
#pragma unroll
    for (int j = 0; j < SUB; ++j) nid[j] = 0u;
    auto fetch_occupancy = [&](uint32_t x) {
        const uint32_t sh = smeta[x % MR].sh;
#pragma unroll
        for (int j = 0; j < SUB; ++j) {
            uint32_t e = lds_u32(idr + (x % IR) * IDB + (sh + 32u * j + lane) * 4u);
            nid[j] = e;
            e = e <= p.catalog ? e : 0u;   // not validated yet
            const uint32_t slot = NWIN == 1 ? lane * (uint32_t)SUB + (uint32_t)j : 32u * j + lane;
            cp_async4(ocr + ((x % WR) * (uint32_t)SE + slot) * 4u, bm + (e >> (NWIN > 1 ? 3 : 5)), bm ? 4u : 0u);
        }
    };

    // OL: step x's occupancy words into registers (its ids have landed)
    auto load_occupancy = [&](uint32_t x, uint32_t (&o)[4]) {
        const uint32_t sh = smeta[x % MR].sh;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t e = lds_u32(idr + (x % IR) * IDB + (sh + 32u * j + lane) * 4u);
            nid[j] = e;
            e = e <= p.catalog ? e : 0u;   // not validated yet
            o[j] = bm ? __ldg(bm + (e >> 5)) : 0u;
        }
    };

    // prologue: ids of steps 0..QD-1 (one group), then occupancy of steps 0..DW-1
#pragma unroll 1
    for (uint32_t x = 0; x < (uint32_t)QD; ++x) fetch_ids(x);
    wait_group(commit());
    __syncwarp();
    uint32_t g_occ = 0;   // commit group of the occupancy words of the next step to scan
    uint32_t onx[4] = {0u, 0u, 0u, 0u};   // OL: occupancy words of the next step to scan
    if (OL) {
        load_occupancy(0, onx);
    } else {
#pragma unroll 1
        for (uint32_t x = 0; x < (uint32_t)DW; ++x) {
            fetch_occupancy(x);
            g_occ = commit();
        }
    }

    // ---- per-lane FIFOs of occupied events, one per window (NWIN == 1:
    // right-aligned; NWIN > 1: left-aligned, entries at and beyond fc are 0)
    uint32_t f[NWIN][QC], fc[NWIN];
#pragma unroll
    for (int u = 0; u < NWIN; ++u) {
        fc[u] = 0;
#pragma unroll
        for (int i = 0; i < QC; ++i) f[u][i] = 0u;
    }

    double G[NLB], Gn[NLB];
    uint32_t m[NLB], mn[NLB];
#pragma unroll
    for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; Gn[l] = 0.0; mn[l] = 0u; }
    uint32_t ft = 0;          // XT: tag bits of the FIFO entries (bit i <-> f[0][i]): 1 = event of the
                              //     open trial while another trial is pending
    uint64_t pend = ~0ull;    // XT: the pending trial, or none
    uint32_t head = 0, tail = 0;   // ring slots: next to consume / next to fill (warp-uniform)
    uint32_t rg[NS];               // commit group of each ring slot's rows

    auto consume = [&]() {
        const uint32_t slot = head % NS;
        uint32_t g = rg[0];
#pragma unroll
        for (int i = 1; i < NS; ++i) g = (slot == (uint32_t)i) ? rg[i] : g;
        wait_group(g);
        __syncwarp();   // other lanes' copies of my row are complete and visible
        const StepMeta rm = rmeta[slot];
        if (PK) event_compute_packed<TV, NLB>(p, s_term, my_row + slot * Geo::STAGE, my_swz, G, m, Gn, mn,
                                              XT && ((rm.k0 >> lane) & 1u));
        else if (NWIN == 1) event_compute_sparse<TV, NSEC, NLB>(p, s_term, my_row + slot * Geo::STAGE, my_swz, G, m);
        else event_compute_sparse_win<TV, NSEC, NLB>(p, s_term, my_row + slot * Geo::STAGE, my_swz, G, m, rm.k0);
        __syncwarp();   // every lane's reads of the slot precede the copies refilling it
        ++head;
        if (rm.n) {   // last round of trial rm.t: a7 + a8
#pragma unroll
            for (int l = 0; l < NLB; ++l) {
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
                    m[l] += __shfl_xor_sync(0xffffffffu, m[l], off);
                }
            }
            if (lane == 0) {
                const uint64_t t = rm.t;
                store_trial(p, t, G, m);
            }
#pragma unroll
            for (int l = 0; l < NLB; ++l) {   // XT: the next trial's partial sums move up
                G[l] = XT ? Gn[l] : 0.0;
                m[l] = XT ? mn[l] : 0u;
                Gn[l] = 0.0;
                mn[l] = 0u;
            }
        }
    };
    // XT: emit a round (pop: every lane pops its FIFO head; !pop: an empty
    // marker round); the round that leaves the pending trial without entries
    // finalises it.  StepMeta: {finalised trial, last, tag mask of the lanes'
    // events}
    auto emit_xt = [&](bool pop) {
        uint32_t ce = 0, tg = 0;
        if (pop) {
#pragma unroll
            for (int i = 0; i < QC; ++i) ce = (fc[0] == (uint32_t)(QC - i)) ? f[0][i] : ce;
            tg = fc[0] ? (ft >> (QC - fc[0])) & 1u : 0u;
            fc[0] -= fc[0] ? 1u : 0u;
        }
        const uint32_t tagmask = __ballot_sync(0xffffffffu, tg != 0u);
        uint32_t last = 0;
        uint64_t tf = 0;
        if (pend != ~0ull) {
            const uint32_t valid = fc[0] ? (((1u << fc[0]) - 1u) << (QC - fc[0])) : 0u;
            if (!__any_sync(0xffffffffu, (~ft & valid) != 0u)) {   // no pending-trial entry left
                last = 1u;
                tf = pend;
                pend = ~0ull;
                ft = 0u;   // the remaining entries belong to the open trial, now untagged
            }
        }
        const uint32_t slot = tail % NS;
        const uint32_t dst = ring + slot * Geo::STAGE;
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            const uint32_t e = __shfl_sync(0xffffffffu, ce, (uint32_t)i * RPI + c_row);
            cp_async16(dst + (uint32_t)i * RPI * Geo::ROWB + c_dst[i & 1], c_src + (uint64_t)e * row_bytes,
                       e ? 16u : 0u);
        }
        if (lane == 0) rmeta[slot] = StepMeta{tf, last, tagmask};
        const uint32_t g = commit();
#pragma unroll
        for (int i = 0; i < NS; ++i) rg[i] = (slot == (uint32_t)i) ? g : rg[i];
        ++tail;
    };
    // emit a round of window u: every lane pops that FIFO's head (0 = nothing:
    // zero-fill); u == NWIN: the empty finalising marker (multi-window)
    // (the caller has made room in the ring)
    auto emit = [&](uint64_t t, uint32_t last, uint32_t u) {
        uint32_t ce = 0;
#pragma unroll
        for (int w = 0; w < NWIN; ++w) {
            if ((uint32_t)w != u) continue;
            if (NWIN == 1) {   // right-aligned FIFO: the head is f[QC - fc]
#pragma unroll
                for (int i = 0; i < QC; ++i) ce = (fc[0] == (uint32_t)(QC - i)) ? f[0][i] : ce;
            } else {
                ce = f[w][0];
#pragma unroll
                for (int i = 0; i + 1 < QC; ++i) f[w][i] = f[w][i + 1];
                f[w][QC - 1] = 0u;
            }
            fc[w] -= fc[w] ? 1u : 0u;
        }
        const char* src = c_src;
        if (NWIN > 1)
            src = reinterpret_cast<const char*>(p.table) +
                  (p.win0[u < (uint32_t)NWIN ? u : 0u] + c_chunk * (16 / sizeof(TV))) * sizeof(TV);
        const uint32_t slot = tail % NS;
        const uint32_t dst = ring + slot * Geo::STAGE;
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            const uint32_t e = __shfl_sync(0xffffffffu, ce, (uint32_t)i * RPI + c_row);
            cp_async16(dst + (uint32_t)i * RPI * Geo::ROWB + c_dst[i & 1], src + (uint64_t)e * row_bytes,
                       e ? 16u : 0u);
        }
        if (lane == 0) rmeta[slot] = StepMeta{t, last, u < (uint32_t)NWIN ? u : 0u};
        const uint32_t g = commit();
#pragma unroll
        for (int i = 0; i < NS; ++i) rg[i] = (slot == (uint32_t)i) ? g : rg[i];
        ++tail;
    };

    // One call site each for emit and (in the loop) consume keeps the loop
    // body small enough for the instruction cache.
#pragma unroll 1
    for (uint32_t sc = 0;; ++sc) {
        uint32_t ocur[4];
        if (OL) {
            // ids of step sc+1 (and, older, sc's) have landed; its occupancy
            // loads are issued now and consumed by the next step
            wait_group(smeta[(sc + 1) % MR].pad);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 4; ++j) ocur[j] = onx[j];
        } else {
            // step sc's occupancy words (and, older, its ids) have landed
            wait_group(g_occ);
            __syncwarp();
        }
        const CqStep md = smeta[sc % MR];
        if (md.t == ~0ull) break;
        uint32_t cid[SUB];   // this step's ids (lane's events k0 + 32 j + lane)
#pragma unroll
        for (int j = 0; j < SUB; ++j) cid[j] = nid[j];
        // refill first: occupancy of step sc+DW (its ids landed: QD >= 2 DW + 1),
        // then ids of step sc+QD; separate groups, so the next scan waits for
        // the occupancy words only
        if (OL) {
            load_occupancy(sc + 1, onx);
        } else {
            fetch_occupancy(sc + DW);
            g_occ = commit();
        }
        fetch_ids(sc + QD);
        commit();
        const bool trial_end = md.k0 + (uint32_t)SE >= md.n;
        const uint32_t id_base = idr + (sc % IR) * IDB + (md.sh + lane) * 4u;
        const uint32_t oc_base = ocr + ((sc % WR) * 128u + lane) * 4u;
        const uint32_t n_here = md.n - md.k0;   // events of the trial from this step on
        if constexpr (NWIN == 1) {
            uint32_t wv[SUB];
            if (OL) {
#pragma unroll
                for (int j = 0; j < 4; ++j) wv[j] = ocur[j];
            } else {
#pragma unroll
                for (int q = 0; q < SUB / 4; ++q) {
                    const uint4 w4 = lds_v4(ocr + ((sc % WR) * (uint32_t)SE + lane * (uint32_t)SUB + 4u * q) * 4u);
                    wv[4 * q] = w4.x; wv[4 * q + 1] = w4.y; wv[4 * q + 2] = w4.z; wv[4 * q + 3] = w4.w;
                }
            }
#pragma unroll 1
            for (uint32_t h = 0; h < (uint32_t)(SUB / 4); ++h) {
            // (1) 4 sub-steps tested at once (independent loads and compares:
            // instruction-level parallelism); ev[j] = event k0 + 128 h + 32 j
            // + lane if its row is occupied, else 0
            uint32_t ev[4], na = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t e = cid[j];
                const uint32_t w = wv[j];
                const bool live = 128u * h + 32u * j + lane < n_here;
                const bool bad = live && e - 1u >= p.catalog;            // id 0 or > C (A14)
                err |= bad ? (uint32_t)ERRBIT_EVENT_RANGE : 0u;
                ev[j] = (live && !bad && (!bm || ((w >> (e & 31u)) & 1u))) ? e : 0u;
                na += ev[j] ? 1u : 0u;
            }
            // the next 4 sub-steps move down (constant register indices)
#pragma unroll
            for (int j = 0; j + 4 < SUB; ++j) { cid[j] = cid[j + 4]; wv[j] = wv[j + 4]; }
            const bool flush = trial_end && h + 1u == (uint32_t)(SUB / 4);
            // (2) rounds are emitted until every lane's FIFO has room for the
            // appends, (3) the appends (right-aligned FIFO: an append shifts
            // it left by one -- predicated moves), (4) at the end of the
            // trial, rounds until every FIFO is empty, the last one
            // finalising the trial.  The FIFO keeps each lane's events in
            // increasing k, so the emission points do not change any sum.
            bool appended = false;
            if constexpr (XT) {
                // flush: finalise the pending trial (rounds until its entries
                // are gone), then the open trial becomes pending -- finalised
                // at once by an empty marker round if it left no entries
                bool made_pending = false;
#pragma unroll 1
                for (;;) {
                    bool pop = true;
                    if (!appended) {
                        if (!__any_sync(0xffffffffu, fc[0] + na > (uint32_t)QC)) {
                            const uint32_t tag = pend != ~0ull ? 1u : 0u;
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                if (ev[j]) {
#pragma unroll
                                    for (int i = 0; i + 1 < QC; ++i) f[0][i] = f[0][i + 1];
                                    f[0][QC - 1] = ev[j];
                                    ft = (ft >> 1) | (tag << (QC - 1));
                                }
                            }
                            fc[0] += na;
                            appended = true;
                            if (!flush) break;
                            continue;
                        }
                    } else if (pend == ~0ull) {
                        if (made_pending) break;
                        pend = md.t;
                        made_pending = true;
                        if (__any_sync(0xffffffffu, fc[0] > 0u)) break;
                        pop = false;   // no entries: the marker round finalises it
                    }
                    if (tail - head == (uint32_t)NS) consume();
                    emit_xt(pop);
                }
            } else {
#pragma unroll 1
            for (;;) {
                uint32_t last = 0;
                if (!appended) {
                    if (!__any_sync(0xffffffffu, fc[0] + na > (uint32_t)QC)) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            if (ev[j]) {
#pragma unroll
                                for (int i = 0; i + 1 < QC; ++i) f[0][i] = f[0][i + 1];
                                f[0][QC - 1] = ev[j];
                            }
                        }
                        fc[0] += na;
                        appended = true;
                        if (!flush) break;
                        continue;
                    }
                } else {
                    last = __any_sync(0xffffffffu, fc[0] > 1u) ? 0u : 1u;
                }
                if (tail - head == (uint32_t)NS) consume();
                emit(md.t, last, 0u);
                if (last) break;
            }
            }
            }
        } else {
#pragma unroll 1
        for (uint32_t j = 0; j < 4u; ++j) {
            uint32_t e = lds_u32(id_base + 128u * j);
            const uint32_t w = lds_u32(oc_base + 128u * j);
            const bool live = 32u * j + lane < n_here;
            const bool bad = live && e - 1u >= p.catalog;            // id 0 or > C (A14)
            err |= bad ? (uint32_t)ERRBIT_EVENT_RANGE : 0u;
            {
                const uint32_t bits = (live && !bad) ? (bm ? (w >> ((e & 7u) * 4u)) & 15u : 15u) : 0u;
#pragma unroll
                for (int u = 0; u < NWIN; ++u) {
                    const bool add = (bits >> u) & 1u;
#pragma unroll
                    for (int i = 0; i < QC; ++i) f[u][i] = (add && fc[u] == (uint32_t)i) ? e : f[u][i];
                    fc[u] += add ? 1u : 0u;
                }
            }
            // a full FIFO emits one round (per window); the end of the trial
            // emits rounds until every FIFO is empty, then finalises the trial
            const bool flush = trial_end && j == 3u;
            uint32_t fullmask = 0;
#pragma unroll
            for (int u = 0; u < NWIN; ++u) fullmask |= __any_sync(0xffffffffu, fc[u] == (uint32_t)QC) ? 1u << u : 0u;
            if (fullmask || flush) {
                for (;;) {
                    // the first window with a full FIFO (or, flushing, any entry)
                    uint32_t pend = 0;
#pragma unroll
                    for (int w = 0; w < NWIN; ++w)
                        pend |= __any_sync(0xffffffffu, flush ? fc[w] > 0u : fc[w] == (uint32_t)QC) ? 1u << w : 0u;
                    if (!pend && !flush) break;
                    const uint32_t u = pend ? (uint32_t)(__ffs(pend) - 1) : (uint32_t)NWIN;   // NWIN: the marker
                    const uint32_t last = pend ? 0u : 1u;
                    if (tail - head == (uint32_t)NS) consume();
                    emit(md.t, last, u);
                    if (last) break;
                }
            }
        }
        }
        __syncwarp();   // reads of this step's slots precede their refills
    }
    if constexpr (XT) {   // the last pending trial
#pragma unroll 1
        while (pend != ~0ull) {
            if (tail - head == (uint32_t)NS) consume();
            emit_xt(true);
        }
    }
    while (head != tail) consume();
    cp_wait<0>();
    peer_fence(p);
    if (err) atomicOr(p.err, err);
}

// Wide layers (window > kMaxSec sectors): same arithmetic and lane mapping,
// one layer per launch, scalar loads through the column-block address map.
template <typename TV>
__global__ void __launch_bounds__(kThreads) trial_kernel_wide(const __grid_constant__ TrialParams p,
                                                              const uint32_t* __restrict__ cols,
                                                              const double2* __restrict__ cterm, uint32_t ncol) {
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
        for (uint64_t k0 = 0; k0 < n; k0 += 32) {
            const uint64_t k = k0 + lane;
            uint32_t v = 0u;
            if (k < n) {
                v = __ldg(ids + k);
                if (v == 0u || v > p.catalog) { err |= ERRBIT_EVENT_RANGE; v = 0u; }
            }
            double le = 0.0;
            for (uint32_t c = 0; c < ncol; ++c) {
                const uint32_t j = __ldg(cols + c);
                const double2 tc = cterm[c];
                const double x = (double)__ldg(tab + (uint64_t)(j / p.row_stride) * p.block_stride +
                                               (uint64_t)v * p.row_stride + j % p.row_stride);
                le = __dadd_rn(le, terms(x, tc.x, tc.y));
            }
            const double o = terms(le, p.lw[0].occ_r, p.lw[0].occ_l);
            G = __dadd_rn(G, o);
            m += (o > 0.0) ? 1u : 0u;
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
                const double port = p.portfolio_mode == 1 ? p.ylt[(uint64_t)p.portfolio_row * p.ld + t] : 0.0;
                p.ylt[(uint64_t)p.portfolio_row * p.ld + t] = __dadd_rn(port, y);
            }
        }
    }
    if (err) atomicOr(p.err, err);
}

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
    for (uint64_t e = (uint64_t)blockIdx.x * kThreads + threadIdx.x; e <= p.catalog;
         e += (uint64_t)gridDim.x * kThreads) {
        Row<TV, NSEC> r;
        r.load(p, (uint32_t)e);
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

// ---------------------------------------------------------------------------
// Folded trial pass over the compacted-rounds scan (fold mode default).  The
// same cross-trial scan as trial_kernel_cq (128-event steps, ids and
// occupancy words by cp.async into per-warp rings) -- with the union
// occupancy bitmap of the fold chunk's blocks, L1-resident because this
// kernel keeps its shared memory small -- and, per event, the fold row
// o(e)[layers] copied by cp.async only when the event's row is occupied
// (an unoccupied event's fold row is exactly +0: zero-fill, no memory
// request).  The fold rows of step s land in a ring slot FR-1 steps before
// they are added, with trial_fold_kernel's lane mapping, per-lane order and
// tree: identical YLT bits.
template <int NL>
struct FoldCqGeo {
    using R = CqRings<2>;
    static constexpr int FR = 3;                                  // fold-row ring slots (steps)
    static constexpr int SLOT = 128 * NL * 8;                     // one step's fold rows
    static constexpr int PER_WARP = R::BYTES + FR * SLOT;
    static constexpr int BYTES = (kThreads / 32) * PER_WARP;
};

template <int NL>
__global__ void __launch_bounds__(kThreads, 2) trial_fold_kernel_cq(const __grid_constant__ TrialParams p) {
    using FG = FoldCqGeo<NL>;
    using RG = typename FG::R;
    constexpr int QD = RG::QD, DW = RG::DW, IR = RG::IR, WR = RG::WR, MR = RG::MR, IDB = RG::IDB;
    constexpr int FR = FG::FR;
    constexpr int WARPS = kThreads / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    unsigned char* wsm = smem + wib * FG::PER_WARP;
    const uint32_t idr = (uint32_t)__cvta_generic_to_shared(wsm);   // id ring [IR][33 x 16 B]
    const uint32_t ocr = idr + IR * IDB;                            // occupancy ring [WR][128]
    CqStep* smeta = reinterpret_cast<CqStep*>(wsm + IR * IDB + WR * 512);
    const uint32_t fr = idr + RG::BYTES;                            // fold rows [FR][4 sub-steps][NL][32]
    const uint64_t nw = (uint64_t)gridDim.x * WARPS;
    const uint64_t base = __ldg(p.off);
    const uint32_t* bm = p.bm;
    const double* fold = p.fold;
    uint32_t err = 0;

    uint32_t gseq = 0;
    auto commit = [&]() { cp_commit(); return gseq++; };
    auto wait_group = [&](uint32_t g) { cp_wait_upto(gseq - 1u - g); };
    auto lds_u32 = [&](uint32_t a) {
        uint32_t v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
        return v;
    };

    uint64_t it_t = p.t_begin + (uint64_t)blockIdx.x * WARPS + wib;
    uint64_t it_a = 0, nx_a = 0, nx_b = 0;
    uint32_t it_n = 0, it_k0 = 0;
    bool it_valid = it_t < p.t_end;
    auto fetch_next_offsets = [&](uint64_t tn) {
        if (tn < p.t_end) { nx_a = __ldg(p.off + tn); nx_b = __ldg(p.off + tn + 1); }
    };
    auto enter_trial = [&](uint64_t a, uint64_t b) {
        if (b < a) { err |= ERRBIT_OFFSETS; b = a; }
        it_a = a - base;
        it_n = (uint32_t)(b - a);
        it_k0 = 0;
    };
    if (it_valid) {
        enter_trial(__ldg(p.off + it_t), __ldg(p.off + it_t + 1));
        fetch_next_offsets(it_t + nw);
    }
    auto fetch_ids = [&](uint32_t x) {
        CqStep md{~0ull, 0u, 0u, 0u, 0u};
        if (it_valid) {
            const uint32_t cnt = it_n - it_k0 < 128u ? it_n - it_k0 : 128u;
            const uintptr_t ab = reinterpret_cast<uintptr_t>(p.ids + it_a + it_k0);
            const uintptr_t al = ab & ~(uintptr_t)15;
            const uintptr_t end = ab + 4u * cnt;
            const uint32_t dst = idr + (x % IR) * IDB;
#pragma unroll
            for (int r = 0; r < 2; ++r) {
                const uint32_t c = lane + 32u * (uint32_t)r;
                if (r == 0 || lane == 0) {
                    const uintptr_t cs = al + 16u * c;
                    const uint32_t nb = cs >= end ? 0u : (end - cs >= 16u ? 16u : (uint32_t)(end - cs));
                    cp_async16(dst + 16u * c, reinterpret_cast<const void*>(nb ? cs : al), nb);
                }
            }
            md = CqStep{it_t, it_n, it_k0, (uint32_t)(ab - al) / 4u, 0u};
            it_k0 += 128u;
            if (it_k0 >= it_n) {
                it_t += nw;
                it_valid = it_t < p.t_end;
                if (it_valid) {
                    enter_trial(nx_a, nx_b);
                    fetch_next_offsets(it_t + nw);
                }
            }
        }
        if (lane == 0) smeta[x % MR] = md;
    };
    auto fetch_occupancy = [&](uint32_t x) {
        const uint32_t sh = smeta[x % MR].sh;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t e = lds_u32(idr + (x % IR) * IDB + (sh + 32u * j + lane) * 4u);
            e = e <= p.catalog ? e : 0u;
            cp_async4(ocr + ((x % WR) * 128u + 32u * j + lane) * 4u, bm + (e >> 5), bm ? 4u : 0u);
        }
    };

#pragma unroll 1
    for (uint32_t x = 0; x < (uint32_t)QD; ++x) fetch_ids(x);
    wait_group(commit());
    __syncwarp();
    uint32_t g_occ = 0;
#pragma unroll 1
    for (uint32_t x = 0; x < (uint32_t)DW; ++x) {
        fetch_occupancy(x);
        g_occ = commit();
    }

    double G[NL];
    uint32_t m[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) { G[l] = 0.0; m[l] = 0u; }
    uint32_t gf[FR];   // commit group of each fold-row slot

    // add step x's fold rows (landed) to the lanes' sums; finalise its trial
    auto consume = [&](uint32_t x) {
        uint32_t g = gf[0];
#pragma unroll
        for (int i = 1; i < FR; ++i) g = ((x % FR) == (uint32_t)i) ? gf[i] : g;
        wait_group(g);
        __syncwarp();
        const CqStep md = smeta[x % MR];
        const uint32_t src = fr + (x % FR) * FG::SLOT + lane * 8u;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int l = 0; l < NL; ++l) {
                double o;
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(o) : "r"(src + ((uint32_t)(j * NL + l) * 32u) * 8u)
                             : "memory");
                G[l] = __dadd_rn(G[l], o);
                m[l] += (o > 0.0) ? 1u : 0u;
            }
        if (md.k0 + 128u >= md.n) {   // last step of trial md.t: a7 + a8
#pragma unroll
            for (int l = 0; l < NL; ++l) {
#pragma unroll
                for (int off = 16; off >= 1; off >>= 1) {
                    G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
                    m[l] += __shfl_xor_sync(0xffffffffu, m[l], off);
                }
            }
            if (lane == 0) store_trial(p, md.t, G, m);
#pragma unroll
            for (int l = 0; l < NL; ++l) { G[l] = 0.0; m[l] = 0u; }
        }
    };

    uint32_t sc = 0;
#pragma unroll 1
    for (;; ++sc) {
        wait_group(g_occ);
        __syncwarp();
        const CqStep md = smeta[sc % MR];
        if (md.t == ~0ull) break;
        fetch_occupancy(sc + DW);
        g_occ = commit();
        fetch_ids(sc + QD);
        commit();
        // this step's fold rows: lanes with an occupied event copy o(e)[0..NL)
        const uint32_t id_base = idr + (sc % IR) * IDB + (md.sh + lane) * 4u;
        const uint32_t oc_base = ocr + ((sc % WR) * 128u + lane) * 4u;
        const uint32_t n_here = md.n - md.k0;
        const uint32_t dst = fr + (sc % FR) * FG::SLOT + lane * 8u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            uint32_t e = lds_u32(id_base + 128u * j);
            const uint32_t w = lds_u32(oc_base + 128u * j);
            const bool live = 32u * (uint32_t)j + lane < n_here;
            const bool bad = live && e - 1u >= p.catalog;
            err |= bad ? (uint32_t)ERRBIT_EVENT_RANGE : 0u;
            e = (live && !bad && (!bm || ((w >> (e & 31u)) & 1u))) ? e : 0u;
            const double* row = fold + (uint64_t)e * p.fold_stride;
#pragma unroll
            for (int l = 0; l < NL; ++l)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst + ((uint32_t)(j * NL + l) * 32u) * 8u),
                             "l"(row + l), "r"(e ? 8u : 0u)
                             : "memory");
        }
        const uint32_t g = commit();
#pragma unroll
        for (int i = 0; i < FR; ++i) gf[i] = ((sc % FR) == (uint32_t)i) ? g : gf[i];
        if (sc + 1 >= (uint32_t)FR) consume(sc + 1 - FR);
        __syncwarp();
    }
    for (uint32_t x = sc + 1 >= (uint32_t)FR ? sc + 1 - FR : 0; x < sc; ++x) consume(x);
    cp_wait<0>();
    peer_fence(p);
    if (err) atomicOr(p.err, err);
}

template <typename TV, int NLB, int D, int MINB = 2>
void* pick_nsec(uint32_t nsec) {
    if (nsec <= 1) return (void*)trial_kernel<TV, 1, NLB, D, MINB>;
    if (nsec <= 2) return (void*)trial_kernel<TV, 2, NLB, D, MINB>;
    if (nsec <= 4) return (void*)trial_kernel<TV, 4, NLB, D, MINB>;
    return (void*)trial_kernel<TV, 8, NLB, D, MINB>;
}

// variant: 0 = no prefetch (D = 1), 2 = prefetch 2 steps ahead (D = 3),
// 3 = 4 steps ahead (D = 5), 4 = 7 steps ahead (D = 8).
template <typename TV>
void* pick(uint32_t nsec, int nl, int variant) {
    if (nl <= 1) {
        if (variant == 2) return pick_nsec<TV, 1, 3>(nsec);
        if (variant == 3) return pick_nsec<TV, 1, 5>(nsec);
        if (variant == 4) return pick_nsec<TV, 1, 8>(nsec);
        if (variant == 5) return pick_nsec<TV, 1, 1, 3>(nsec);
        if (variant == 6) return pick_nsec<TV, 1, 1, 4>(nsec);
        if (variant == 7) return pick_nsec<TV, 1, 3, 3>(nsec);
        return pick_nsec<TV, 1, 1>(nsec);
    }
    if (nl <= 2) return pick_nsec<TV, 2, 1>(nsec);
    return pick_nsec<TV, 4, 1>(nsec);
}

template <typename TV, int NLB>
void* pick_nsec_sm(uint32_t nsec, int* smem) {
    if (nsec <= 1) { *smem = SmGeo<TV, 1>::BYTES; return (void*)trial_kernel_sm<TV, 1, NLB>; }
    if (nsec <= 2) { *smem = SmGeo<TV, 2>::BYTES; return (void*)trial_kernel_sm<TV, 2, NLB>; }
    if (nsec <= 4) { *smem = SmGeo<TV, 4>::BYTES; return (void*)trial_kernel_sm<TV, 4, NLB>; }
    *smem = SmGeo<TV, 8>::BYTES;
    return (void*)trial_kernel_sm<TV, 8, NLB>;
}

template <typename TV>
void* pick_sm(uint32_t nsec, int nl, int* smem) {
    if (nl <= 1) return pick_nsec_sm<TV, 1>(nsec, smem);
    if (nl <= 2) return pick_nsec_sm<TV, 2>(nsec, smem);
    return pick_nsec_sm<TV, 4>(nsec, smem);
}

template <typename TV, int NLB>
void* pick_nsec_tma(uint32_t nsec, int* smem) {
    if (nsec <= 1) { *smem = TmaGeo<TV, 1>::BYTES; return (void*)trial_kernel_tma<TV, 1, NLB>; }
    if (nsec <= 2) { *smem = TmaGeo<TV, 2>::BYTES; return (void*)trial_kernel_tma<TV, 2, NLB>; }
    *smem = TmaGeo<TV, 4>::BYTES;
    return (void*)trial_kernel_tma<TV, 4, NLB>;
}

template <typename TV>
void* pick_tma(uint32_t nsec, int nl, int* smem) {
    if (nl <= 1) return pick_nsec_tma<TV, 1>(nsec, smem);
    if (nl <= 2) return pick_nsec_tma<TV, 2>(nsec, smem);
    return pick_nsec_tma<TV, 4>(nsec, smem);
}

template <typename TV, int NLB, int BUDGET_KB, int MINB, bool EARLY>
void* pick_nsec_co(uint32_t nsec, int* smem) {
    if (nsec <= 1) {
        *smem = CoGeo<TV, 1, BUDGET_KB>::BYTES;
        return (void*)trial_kernel_co<TV, 1, NLB, BUDGET_KB, MINB, EARLY>;
    }
    if (nsec <= 2) {
        *smem = CoGeo<TV, 2, BUDGET_KB>::BYTES;
        return (void*)trial_kernel_co<TV, 2, NLB, BUDGET_KB, MINB, EARLY>;
    }
    *smem = CoGeo<TV, 4, BUDGET_KB>::BYTES;
    return (void*)trial_kernel_co<TV, 4, NLB, BUDGET_KB, MINB, EARLY>;
}

// 10: one CTA/SM, ~200 KB ring; 11: two CTAs/SM, ~100 KB each; 12: three CTAs/SM,
// ~66 KB each (refill after the arithmetic); 13: as 12, refill before it
template <typename TV>
void* pick_co(uint32_t nsec, int nl, int variant, int* smem) {
#define ARA_CO_V(NLB)                                                             \
    if (variant == 11) return pick_nsec_co<TV, NLB, 100, 2, true>(nsec, smem);    \
    if (variant == 12) return pick_nsec_co<TV, NLB, 66, 3, false>(nsec, smem);    \
    if (variant == 13) return pick_nsec_co<TV, NLB, 66, 3, true>(nsec, smem);     \
    return pick_nsec_co<TV, NLB, 200, 1, true>(nsec, smem);
    if (nl <= 1) { ARA_CO_V(1) }
    if (nl <= 2) { ARA_CO_V(2) }
    ARA_CO_V(4)
#undef ARA_CO_V
}

template <typename TV, int NLB, int BUDGET_KB, int MINB>
void* pick_nsec_cq(uint32_t nsec, int* smem) {
    if (nsec <= 1) {
        *smem = CqGeo<TV, 1, BUDGET_KB, MINB>::BYTES;
        return (void*)trial_kernel_cq<TV, 1, NLB, BUDGET_KB, MINB, 1>;
    }
    if (nsec <= 2) {
        *smem = CqGeo<TV, 2, BUDGET_KB, MINB>::BYTES;
        return (void*)trial_kernel_cq<TV, 2, NLB, BUDGET_KB, MINB, 1>;
    }
    *smem = CqGeo<TV, 4, BUDGET_KB, MINB>::BYTES;
    return (void*)trial_kernel_cq<TV, 4, NLB, BUDGET_KB, MINB, 1>;
}

// packed rounds (17): one 32-B slot per event; the row ring (BUDGET_KB) holds
// NS 1-KB stages per warp
template <typename TV, int NLB, int B, bool OL, int SE = 128, bool XT = false>
void* pick_pk(int* smem) {
    *smem = CqGeo<TV, 1, B, 2, SE>::BYTES;
    return (void*)trial_kernel_cq<TV, 1, NLB, B, 2, 1, true, OL, SE, XT>;
}

// two CTAs/SM: a 2-stage row ring (64 KB) plus the id/occupancy rings per CTA;
// variant 16: a 1-stage row ring (more L1 left for the occupancy bitmap)
template <typename TV>
void* pick_cq(uint32_t nsec, int nl, int variant, int* smem) {
#define ARA_CQ_V(NLB)                                                         \
    if (variant == 17) return pick_pk<TV, NLB, 10, false>(smem);              \
    if (variant == 18) return pick_pk<TV, NLB, 10, true>(smem);               \
    if (variant == 19) return pick_pk<TV, NLB, 40, false>(smem);              \
    if (variant == 20) return pick_pk<TV, NLB, 10, false, 256>(smem);         \
    if (variant == 21) return pick_pk<TV, NLB, 10, false, 128, true>(smem);   \
    if (variant == 16) return pick_nsec_cq<TV, NLB, 40, 2>(nsec, smem);       \
    return pick_nsec_cq<TV, NLB, 66, 2>(nsec, smem);
    if (nl <= 1) { ARA_CQ_V(1) }
    if (nl <= 2) { ARA_CQ_V(2) }
    ARA_CQ_V(4)
#undef ARA_CQ_V
}

// multi-window compacted rounds: up to 4 disjoint windows of equal width
template <typename TV>
void* pick_cqm(uint32_t nsec, int* smem) {
    if (nsec <= 1) { *smem = CqGeo<TV, 1, 66, 2>::BYTES; return (void*)trial_kernel_cq<TV, 1, 4, 66, 2, 4>; }
    if (nsec <= 2) { *smem = CqGeo<TV, 2, 66, 2>::BYTES; return (void*)trial_kernel_cq<TV, 2, 4, 66, 2, 4>; }
    *smem = CqGeo<TV, 4, 66, 2>::BYTES;
    return (void*)trial_kernel_cq<TV, 4, 4, 66, 2, 4>;
}

// variant: 0 = register-pipelined, 1 = shared-memory staged (cp.async ring),
// 2-4 = register + L2 prefetch, 5-7 = register at higher occupancy,
// 8 = TMA gather4 ring (needs p.tmap; windows of <= 4 sectors in one block),
// 10-13 = cooperative cp.async ring (whole rows per instruction) at 1/2/3 CTAs/SM,
// 14 = compacted rounds over the cooperative ring (skips zero rows' arithmetic),
// 15 = the same over up to 4 disjoint layer windows in one launch (host-selected),
// 16 = 14 with a 1-stage row ring, 17 = compacted rounds over packed rows (p.pk),
// 18 = 17 with the occupancy words by L1-cached loads into registers,
// 19 = 17 with a 4-stage row ring, 20 = 17 with 256-event scan steps,
// 21 = 17 with rounds packed across trial boundaries.
void* pick_kernel(int fp32, uint32_t nsec, int nl, int variant, int* smem) {
    *smem = 0;
    if (variant == 8 && nsec <= 4)
        return fp32 ? pick_tma<float>(nsec, nl, smem) : pick_tma<double>(nsec, nl, smem);
    if (nsec > (uint32_t)kMaxSec) return fp32 ? (void*)trial_kernel_wide<float> : (void*)trial_kernel_wide<double>;
    if (variant == 1) return fp32 ? pick_sm<float>(nsec, nl, smem) : pick_sm<double>(nsec, nl, smem);
    if (variant >= 10 && variant <= 13 && nsec <= 4)
        return fp32 ? pick_co<float>(nsec, nl, variant, smem) : pick_co<double>(nsec, nl, variant, smem);
    if (((variant >= 16 && variant <= 21) || variant == 14) && nsec <= 4)
        return fp32 ? pick_cq<float>(nsec, nl, variant, smem) : pick_cq<double>(nsec, nl, variant, smem);
    if (variant == 15 && nsec <= 4) return fp32 ? pick_cqm<float>(nsec, smem) : pick_cqm<double>(nsec, smem);
    return fp32 ? pick<float>(nsec, nl, variant) : pick<double>(nsec, nl, variant);
}

}  // namespace

int trial_kernel_grid(int fp32, uint32_t max_nsec, int n_layers, int variant) {
    static int cache[32][2][kMaxSec + 2][kMaxLB + 1] = {};
    const uint32_t ns = max_nsec > (uint32_t)kMaxSec ? kMaxSec + 1 : max_nsec;
    int& c = cache[variant & 31][fp32 ? 1 : 0][ns][n_layers];
    if (c) return c;
    int dev = 0, nsm = 148, per_sm = 1, smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    void* fn = pick_kernel(fp32, max_nsec, n_layers, variant, &smem);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    c = nsm * per_sm;
    return c;
}

void set_ldg_carveout(int fp32, uint32_t nsec, int nl, int pct) {
    int smem = 0;
    cudaFuncSetAttribute(pick_kernel(fp32, nsec, nl, 5, &smem), cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();
}

cudaError_t launch_trials(const TrialParams& p, int fp32, uint32_t max_nsec, int grid, int variant, cudaStream_t s) {
    if (p.t_end <= p.t_begin) return cudaSuccess;
    const uint64_t need = ((p.t_end - p.t_begin) * 32 + kThreads - 1) / kThreads;
    const int g = (int)((uint64_t)grid < need ? (uint64_t)grid : need);
    int smem = 0;
    void* fn = pick_kernel(fp32, max_nsec, (int)p.n_layers, variant, &smem);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    if (const char* v = getenv("ARA_CARVEOUT")) {   // A/B: shared-memory carveout preference (percent)
        cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(v));
        cudaGetLastError();
    } else if (variant == 17 || variant == 21) {
        // the smallest shared-memory configuration that holds the 2 CTAs/SM
        // (2 x 37 KB -> the 100 KB split): the rest of the 256 KB is L1 for
        // the occupancy bitmap (measured 5.94 vs 5.98 ms at the driver's 132 KB)
        cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 34);
        cudaGetLastError();
    }
    void* args[] = {(void*)&p};
    return cudaLaunchKernel(fn, dim3(g), dim3(kThreads), args, (size_t)smem, s);
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
    // per-trial folded pass (default), or the scan-based one (ARA_FOLD_KERNEL=1, A/B:
    // measured slower, 5.1 vs 4.0 ms on the paper config -- the scan costs more
    // than the one-gather-per-event pass it replaces)
    // (a cross-trial register-pipelined pass with occupancy gating, 32 events
    // per step, measured 5.25 ms -- slower too: more instructions per event)
    static int legacy = -1;
    if (legacy < 0) {
        const char* v = getenv("ARA_FOLD_KERNEL");
        legacy = (v && atoi(v) == 1) ? 0 : 1;
    }
    void* fn;
    int smem = 0;
    if (!legacy) {
        fn = p.fold_stride <= 1 ? (void*)trial_fold_kernel_cq<1>
             : p.fold_stride <= 2 ? (void*)trial_fold_kernel_cq<2>
             : p.fold_stride <= 4 ? (void*)trial_fold_kernel_cq<4>
                                  : (void*)trial_fold_kernel_cq<8>;
        smem = p.fold_stride <= 1 ? FoldCqGeo<1>::BYTES
               : p.fold_stride <= 2 ? FoldCqGeo<2>::BYTES
               : p.fold_stride <= 4 ? FoldCqGeo<4>::BYTES
                                    : FoldCqGeo<8>::BYTES;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
        }
    } else {
        fn = p.fold_stride <= 1 ? (void*)trial_fold_kernel<1>
             : p.fold_stride <= 2 ? (void*)trial_fold_kernel<2>
             : p.fold_stride <= 4 ? (void*)trial_fold_kernel<4>
                                  : (void*)trial_fold_kernel<8>;
    }
    int dev = 0, nsm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        per_sm = 1;
    }
    uint64_t grid = (uint64_t)nsm * per_sm * grid_mult_x100 / 100;
    const uint64_t need = ((p.t_end - p.t_begin) * 32 + kThreads - 1) / kThreads;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    void* args[] = {(void*)&p};
    return cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(kThreads), args, (size_t)smem, s);
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

cudaError_t launch_trials_wide(const TrialParams& p, int fp32, const uint32_t* d_cols, const double2* d_cterm,
                               uint32_t ncol, int grid, cudaStream_t s) {
    if (p.t_end <= p.t_begin) return cudaSuccess;
    const uint64_t need = ((p.t_end - p.t_begin) * 32 + kThreads - 1) / kThreads;
    const int g = (int)((uint64_t)grid < need ? (uint64_t)grid : need);
    if (fp32)
        trial_kernel_wide<float><<<g, kThreads, 0, s>>>(p, d_cols, d_cterm, ncol);
    else
        trial_kernel_wide<double><<<g, kThreads, 0, s>>>(p, d_cols, d_cterm, ncol);
    return cudaGetLastError();
}

}  // namespace ara
