// kernel_dense.cu -- the ARA trial kernels for dense direct-access tables
// (SURVEY.md 8a rows a2-a8 when most rows of the table are occupied), the
// generic kernel for layer windows wider than kMaxSec sectors, and the launch
// dispatcher.  Sparse column blocks (the paper's ELTs) go to
// trial_kernel_bc (kernel_sparse.cu).
//
// B200 mapping:
//   * one warp per trial (the paper used one thread per trial);
//   * event k of the trial -> lane k % 32, each lane in increasing k, then a
//     fixed 5-step xor tree: the summation order depends only on the trial's
//     own events;
//   * one lane reads one event's row window of the column-blocked table --
//     the layer's 32-B sectors -- and sums the ELT terms sequentially in ELT
//     order (bit-identical per-event loss to the sequential oracle, hence
//     exact lossy-occurrence counts);
//   * validation of YET ids / offsets is fused (error bits, no extra pass).
// This is a gather-and-reduce path: no tensor cores (not a contraction).
#include <cstdlib>

#include "ara_device.cuh"

namespace ara {
namespace {

// Register-pipelined kernel (dense fp32 windows; windows of 5-8 sectors): ids
// D + 1 steps ahead, rows one step ahead of the fp64 term arithmetic
// (instantiated with D = 1).
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
            }
#pragma unroll 1
            for (uint64_t k0 = 0; k0 < n; k0 += STEP) {
                uint32_t en[QB];
                load_ids(k0 + (D + 1) * STEP, en);
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
// Cooperative cp.async ring (dense fp64 windows).  The row windows of a step
// land in a per-warp shared-memory ring NS steps deep, so in-flight rows hold
// no registers and the ring runs across trial boundaries (no pipeline drain
// per trial).  Unlike a per-lane ring (each lane copying its own row in 16-B
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

template <typename TV, int NLB, int MINB>
void* pick_nsec(uint32_t nsec) {
    if (nsec <= 1) return (void*)trial_kernel<TV, 1, NLB, 1, MINB>;
    if (nsec <= 2) return (void*)trial_kernel<TV, 2, NLB, 1, MINB>;
    if (nsec <= 4) return (void*)trial_kernel<TV, 4, NLB, 1, MINB>;
    return (void*)trial_kernel<TV, 8, NLB, 1, MINB>;
}

// register pipeline: variant 5 = 3 CTAs/SM (single layers), otherwise 2 CTAs/SM
template <typename TV>
void* pick(uint32_t nsec, int nl, int variant) {
    if (nl <= 1) return variant == 5 ? pick_nsec<TV, 1, 3>(nsec) : pick_nsec<TV, 1, 2>(nsec);
    if (nl <= 2) return pick_nsec<TV, 2, 2>(nsec);
    return pick_nsec<TV, 4, 2>(nsec);
}

// cooperative cp.async ring at 3 CTAs/SM (~66 KB of ring each)
template <typename TV, int NLB>
void* pick_nsec_co(uint32_t nsec, int* smem) {
    if (nsec <= 1) { *smem = CoGeo<TV, 1, 66>::BYTES; return (void*)trial_kernel_co<TV, 1, NLB, 66, 3, false>; }
    if (nsec <= 2) { *smem = CoGeo<TV, 2, 66>::BYTES; return (void*)trial_kernel_co<TV, 2, NLB, 66, 3, false>; }
    *smem = CoGeo<TV, 4, 66>::BYTES;
    return (void*)trial_kernel_co<TV, 4, NLB, 66, 3, false>;
}

template <typename TV>
void* pick_co(uint32_t nsec, int nl, int* smem) {
    if (nl <= 1) return pick_nsec_co<TV, 1>(nsec, smem);
    if (nl <= 2) return pick_nsec_co<TV, 2>(nsec, smem);
    return pick_nsec_co<TV, 4>(nsec, smem);
}

// variant (ARA_KERNEL): 0 = register pipeline, 2 CTAs/SM; 5 = register
// pipeline, 3 CTAs/SM; 12 = cooperative cp.async ring (3 CTAs/SM, windows of
// <= 4 sectors); 30 = trial_kernel_bc (sparse blocks, kernel_sparse.cu)
void* pick_kernel(int fp32, uint32_t nsec, int nl, int variant, int* smem) {
    *smem = 0;
    if (nsec > (uint32_t)kMaxSec) return fp32 ? (void*)trial_kernel_wide<float> : (void*)trial_kernel_wide<double>;
    if (variant == 12 && nsec <= 4) return fp32 ? pick_co<float>(nsec, nl, smem) : pick_co<double>(nsec, nl, smem);
    return fp32 ? pick<float>(nsec, nl, variant) : pick<double>(nsec, nl, variant);
}

}  // namespace

int trial_kernel_grid(int fp32, uint32_t max_nsec, int n_layers, int variant) {
    if (variant == 30) {   // persistent: one CTA per SM
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        return nsm;
    }
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

cudaError_t launch_trials(const TrialParams& p, int fp32, uint32_t max_nsec, int grid, int variant, cudaStream_t s) {
    if (p.t_end <= p.t_begin) return cudaSuccess;
    if (variant == 30) return launch_trials_bc(p, fp32, grid, s);
    const uint64_t need = ((p.t_end - p.t_begin) * 32 + kThreads - 1) / kThreads;
    const int g = (int)((uint64_t)grid < need ? (uint64_t)grid : need);
    int smem = 0;
    void* fn = pick_kernel(fp32, max_nsec, (int)p.n_layers, variant, &smem);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    void* args[] = {(void*)&p};
    return cudaLaunchKernel(fn, dim3(g), dim3(kThreads), args, (size_t)smem, s);
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
