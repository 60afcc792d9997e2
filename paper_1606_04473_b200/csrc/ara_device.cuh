// ara_device.cuh -- device-side building blocks shared by the trial kernels
// (product path; nothing here is shared with oracle/).  Internal linkage: each
// kernel translation unit gets its own copy.
//
// The arithmetic follows PAPER.md Alg. 3 with P:371-377: per
// event and ELT of the layer a lookup and the per-ELT terms I
// (P:360), the sum across ELTs in ELT order, occurrence terms on the
// event's combined loss, accumulation over the trial, aggregate terms
// on the total.  Readings A1-A22: DESIGN.md section 2.
#pragma once
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

// Events per lane per pipeline step (~16-32 row registers per stage); windows
// wider than 32 registers run without the row double buffer (PIPE = false).
template <typename TV, int NSEC>
struct Batch {
    static constexpr int R = NSEC * SecT<TV>::N * (int)sizeof(TV) / 4;   // row registers per event
    static constexpr int QB = R >= 16 ? 1 : (R >= 8 ? 2 : 4);
    static constexpr bool PIPE = R <= 32;
};

// Warp-level static trial scheduler: trials gw, gw+nw, ... of the launch
// range.  Per-trial arithmetic does not depend on which warp takes a trial,
// so the YLT bits do not either.
struct TrialSched {
    uint64_t cur, stride;
    __device__ __forceinline__ void init(const TrialParams& p, uint64_t gw, uint64_t nw) {
        cur = p.t_begin + gw;
        stride = nw;
    }
    // next trial index for this warp, or ~0 when the range is exhausted
    __device__ __forceinline__ uint64_t next(const TrialParams& p) {
        const uint64_t t = cur;
        cur += stride;
        return t < p.t_end ? t : ~0ull;
    }
};

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

}  // namespace
}  // namespace ara
