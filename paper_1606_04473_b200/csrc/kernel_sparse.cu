// kernel_sparse.cu -- trial_kernel_bc: ballot-compacted rounds over packed
// rows, the ARA trial kernel for sparse column blocks (SURVEY.md 8a rows
// a2-a8 on the paper's ELTs).
//
// The paper's ELTs hold 10k-30k losses over a catalogue of millions,
// so most events of a trial hit an all-zero row of the direct-access table,
// which adds an exact +0 (every deductible and retention is >= 0).  Per event
// the only work left is the occupancy test; the loss arithmetic (P:359-P:375)
// runs for the occupied events only, 32 at a time.
//
//  * persistent: one CTA of 24-32 warps per SM; each warp owns a contiguous range
//    of trials holding an equal share of the launch's events (a 32-ary search
//    over the CSR offsets), so its event ids are ONE contiguous stream;
//  * the stream is staged by the Tensor Memory Accelerator: one elected lane
//    issues cp.async.bulk copies of 512-B chunks (128 ids) into a 2-stage
//    per-warp ring, completion counted by an mbarrier per stage, with an
//    L2::evict_first policy (the 4 GB YET is read exactly once; the paper's
//    "chunking ... for the efficient use of shared memory");
//  * the block's row-occupancy bitmap is copied once per CTA into shared
//    memory (as much as fits next to the rings: ~72 % of a 2M-event
//    catalogue); probes of the rest go to L1/L2.  The ids and probe words of
//    batch c+1 are loaded while batch c is scanned;
//  * scan: 32 consecutive events per ballot; occupied events are appended,
//    in stream order, to a per-warp compaction ring in shared memory (the
//    popc of the ballot below the lane gives the slot);
//  * round: 32 queued events, queue entry i to lane i; each lane gathers its
//    event's 32-B packed slot (one sector: non-zero mask, id, first values)
//    and does a4-a7 for the layers of the launch.  A round's slot loads are
//    issued one round before its arithmetic, and a trial's last (partial)
//    round is finished -- with the trial's tree and stores -- when the next
//    round is issued, so gathers overlap the scan and no trial end stalls;
//  * the rounds of a trial start at an empty queue, so lane l adds the
//    trial's occupied events l, l+32, ... in stream order, then a fixed
//    5-step xor tree: an order that depends only on the trial's own events
//    (partition and alignment invariant; A18/A21) and exact on
//    integer-valued data (P10).
#include <cstdlib>
#include <mutex>

#include "ara_device.cuh"

namespace ara {
namespace {

#ifndef BC_NSTG
#define BC_NSTG 2
#endif
#ifndef BC_CHB
#define BC_CHB 512
#endif
// Warps per CTA (one CTA per SM) by layers per launch, measured
// (profiles/r02_ab_bc_warps.txt): the loop is latency-bound, so as many warps
// as the registers allow -- 32 for one layer (64 registers), 24 for towers.
template <int NLB> struct BcWarps { static constexpr int value = NLB <= 1 ? 32 : 24; };
// Compaction queue entries per warp: 128 for one layer (32 warps: the smaller
// queue leaves 16 KB more of the bitmap in shared memory), 256 for towers.
template <int NLB> struct BcQueue { static constexpr int value = NLB <= 1 ? 128 : 256; };
template <int W, int CB>
struct BcGeo {
    static constexpr int WARPS = W;                  // per CTA, one CTA per SM
    static constexpr int THREADS = WARPS * 32;
    static constexpr int CHB = BC_CHB;               // bytes per id chunk: 1 or 2 batches of 128 ids
    static constexpr int NSTG = BC_NSTG;             // chunks per warp ring (power of two)
    static constexpr int RING = NSTG * CHB;          // id ring bytes per warp
    // compaction queue entries per warp (power of two >= 64: a batch whose
    // last group would overflow it has that group appended after rounds)
    static constexpr int CBUF = CB;
    static constexpr int FIXED = WARPS * (RING + CBUF * 4);   // dynamic smem before the bitmap
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_nohint(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
// expect_tx + bulk copy issued by one lane chosen by elect.sync: the whole
// (converged) warp executes this with warp-uniform operands, so no branch
// around a single lane and no per-lane loop to make the operands uniform
__device__ __forceinline__ void bulk_g2s_elect(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                               uint64_t pol) {
    asm volatile(
        "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
        "@p mbarrier.arrive.expect_tx.shared::cta.b64 _, [%3], %2;\n\t"
        "@p cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        "\n\t}" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// a shared-memory address the compiler must keep in a register (instead of
// re-deriving it from the CTA's shared window at every use)
__device__ __forceinline__ uint32_t pin(uint32_t v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}
// occupancy word wi: shared memory for the first Ws words, else L1/L2
__device__ __forceinline__ uint32_t probe(uint32_t wi, uint32_t Ws, uint32_t s_bm, const uint32_t* bm) {
    uint32_t w;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.lt.u32 p, %1, %2;\n\t@p ld.shared.u32 %0, [%3];\n\t"
        "@!p ld.global.nc.u32 %0, [%4];\n\t}"
        : "=r"(w)
        : "r"(wi), "r"(Ws), "r"(s_bm + 4u * wi), "l"(bm + wi)
        : "memory");
    return w;
}

// One packed slot (kPackBytes) in registers: u32 mask, u32 id, then the row's
// first non-zero values in column order (3 fp64 / 6 fp32).
template <typename TV> struct Slot;
template <> struct Slot<double> {
    static constexpr int CAP = 3;
    uint64_t q[4];
    __device__ __forceinline__ uint32_t mask() const { return (uint32_t)q[0]; }
    __device__ __forceinline__ uint32_t id() const { return (uint32_t)(q[0] >> 32); }
    __device__ __forceinline__ double val(uint32_t v) const {
        return __longlong_as_double((long long)(v == 0 ? q[1] : (v == 1 ? q[2] : q[3])));
    }
};
template <> struct Slot<float> {
    static constexpr int CAP = 6;
    uint64_t q[4];
    __device__ __forceinline__ uint32_t mask() const { return (uint32_t)q[0]; }
    __device__ __forceinline__ uint32_t id() const { return (uint32_t)(q[0] >> 32); }
    __device__ __forceinline__ double val(uint32_t v) const {
        const uint64_t w = v < 2 ? q[1] : (v < 4 ? q[2] : q[3]);
        return (double)__int_as_float((int)(uint32_t)((v & 1u) ? (w >> 32) : w));
    }
};
__device__ __forceinline__ void ld_slot(const void* p, uint64_t (&q)[4]) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(q[0]), "=l"(q[1]), "=l"(q[2]), "=l"(q[3])
                 : "l"(p));
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}

// FOLD (catalogue-fold mode): the rounds gather o(e), the
// occurrence-net loss folded once per catalogue event (fold_kernel), for the
// NLB layers of the fold chunk instead of the packed slot, and accumulate it
// exactly as the direct rounds accumulate the o they compute: same events,
// same dealing, same order -- the YLT and the lossy counts equal the direct
// sparse kernel's bit for bit (reading A18).
template <typename TV, int NLB, bool FOLD = false, int W = BcWarps<NLB>::value>
__global__ void __launch_bounds__(W * 32, 1) trial_kernel_bc(const __grid_constant__ TrialParams p) {
    using Geo = BcGeo<W, BcQueue<NLB>::value>;
    constexpr int CAP = Slot<TV>::CAP;
    constexpr uint32_t CHE = 128;                  // ids per batch
    constexpr uint32_t BPC = Geo::CHB / 512;       // batches per chunk
    constexpr uint32_t NSTG = Geo::NSTG;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(16) double2 s_term[NLB][32];
    __shared__ __align__(8) uint64_t s_bar[Geo::WARPS * Geo::NSTG + 1];
    __shared__ __align__(16) uintptr_t s_stream[Geo::WARPS][2];   // per warp: the id stream's 16-B aligned byte range
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t sbase = pin((uint32_t)__cvta_generic_to_shared(smem));
    const uint32_t ring = sbase + wib * (uint32_t)Geo::RING;
    const uint32_t cbuf = sbase + (uint32_t)(Geo::WARPS * Geo::RING) + wib * (uint32_t)(Geo::CBUF * 4);
    const uint32_t s_bm = sbase + (uint32_t)Geo::FIXED;
    const uint32_t s_tm = pin((uint32_t)__cvta_generic_to_shared(&s_term[0][0]));
    const uint32_t bar0 = pin((uint32_t)__cvta_generic_to_shared(&s_bar[wib * Geo::NSTG]));
    const uint32_t bmbar = (uint32_t)__cvta_generic_to_shared(&s_bar[Geo::WARPS * Geo::NSTG]);
    const uint32_t Ws = p.bm_smem_words;
    const uint32_t* bm = p.bm;

    for (int i = threadIdx.x; i < NLB * 32; i += Geo::THREADS) s_term[i / 32][i % 32] = p.term[i / 32][i % 32];
    if (threadIdx.x == 0) {
        for (int s = 0; s < Geo::WARPS * Geo::NSTG + 1; ++s)
            mbar_init((uint32_t)__cvta_generic_to_shared(&s_bar[s]), 1u);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && Ws) {   // the shared-memory part of the occupancy bitmap (read by every CTA)
        mbar_expect_tx(bmbar, Ws * 4u);
        bulk_g2s_nohint(s_bm, bm, Ws * 4u, bmbar);
    }

    // ---- this warp's trials [tb, te): an equal share of the launch's events
    const uint64_t nw = (uint64_t)gridDim.x * Geo::WARPS, gw = (uint64_t)blockIdx.x * Geo::WARPS + wib;
    const uint64_t base = __ldg(p.off);
    const uint64_t o_b = __ldg(p.off + p.t_begin);
    uint64_t o_e = __ldg(p.off + p.t_end);
    uint32_t err = 0;
    if (o_b < base || o_e < o_b) { err |= ERRBIT_OFFSETS; o_e = o_b; }
    // first t in [t_begin, t_end] with off[t] >= target (32-ary search; the
    // offsets are non-decreasing when valid, and a violation is caught below)
    auto lower_bound = [&](uint64_t target) {
        uint64_t lo = p.t_begin, hi = p.t_end;
        while (hi > lo) {
            const uint64_t step = (hi - lo + 31) / 32;
            const uint64_t idx = lo + (uint64_t)lane * step;
            const bool ge = idx >= hi || __ldg(p.off + idx) >= target;
            const uint32_t m = __ballot_sync(0xffffffffu, ge);
            if (m == 0u) {
                lo = lo + 31 * step + 1;
            } else {
                const uint32_t f = (uint32_t)(__ffs(m) - 1);
                if (f == 0u) {
                    hi = lo;
                } else {
                    const uint64_t l0 = lo;
                    lo = l0 + (f - 1) * step + 1;
                    hi = l0 + f * step < hi ? l0 + f * step : hi;
                }
            }
        }
        return lo;
    };
    const uint64_t span_ev = o_e - o_b;
    const uint64_t tb = gw == 0 ? p.t_begin : lower_bound(o_b + span_ev * gw / nw);
    uint64_t te = gw + 1 == nw ? p.t_end : lower_bound(o_b + span_ev * (gw + 1) / nw);
    if (te < tb) { err |= ERRBIT_OFFSETS; te = tb; }
    int64_t S0 = 0, S1 = 0;   // the warp's event stream [S0, S1), indices into p.ids
    if (te > tb) {
        const uint64_t a = __ldg(p.off + tb), b = __ldg(p.off + te);
        if (a < o_b || b < a || b > o_e) { err |= ERRBIT_OFFSETS; te = tb; }
        else { S0 = (int64_t)(a - base); S1 = (int64_t)(b - base); }
    }

    // ---- the stream's chunks, 16-B aligned; chunk c = batch c.  Positions
    // are 32-bit offsets from P0, the stream index of the ring's first id.
    const uintptr_t a_s = reinterpret_cast<uintptr_t>(p.ids + S0);
    const uintptr_t a0 = a_s & ~(uintptr_t)15;
    const uintptr_t aend = (reinterpret_cast<uintptr_t>(p.ids + S1) + 15) & ~(uintptr_t)15;
    const int64_t P0 = S0 - (int64_t)((a_s - a0) >> 2);
    if (S1 - P0 > (int64_t)0x7fffff00) { err |= ERRBIT_OFFSETS; te = tb; S1 = S0; }   // > 2^31 events in one warp
    const uint32_t nchunks = S1 > S0 ? (uint32_t)((aend - a0 + Geo::CHB - 1) / Geo::CHB) : 0u;
    // the stream's byte range lives in shared memory (read when a stage is
    // refilled), not in registers
    if (lane == 0) { s_stream[wib][0] = a0; s_stream[wib][1] = aend; }
    const uint32_t s_str = pin((uint32_t)__cvta_generic_to_shared(&s_stream[wib][0]));
    // chunk c goes to stage c % NSTG; only the stream's last chunk is short
    auto issue_chunk = [&](uint32_t c) {   // lane 0
        const uintptr_t b0 = s_stream[wib][0], b1 = s_stream[wib][1];
        const uintptr_t src = b0 + (uintptr_t)c * Geo::CHB;
        const uint32_t bytes = c + 1 < nchunks ? (uint32_t)Geo::CHB : (uint32_t)(b1 - src);
        const uint32_t st = c & (NSTG - 1);
        mbar_expect_tx(bar0 + 8u * st, bytes);
        bulk_g2s(ring + st * Geo::CHB, reinterpret_cast<const void*>(src), bytes, bar0 + 8u * st,
                 policy_evict_first());
    };
    if (lane == 0)
        for (uint32_t c = 0; c < NSTG && c < nchunks; ++c) issue_chunk(c);
    if (Ws) mbar_wait(bmbar, 0u);   // the bitmap has landed

    // batch c: its ids (0 for an id outside [1, C], A14 -- row 0 is never
    // occupied) and their occupancy words; the chunk's stage is refilled as
    // soon as its ids are in registers.  A batch past the stream's end reads
    // stale ids: none of its positions is ever live.
    const uint32_t C = p.catalog;
    auto load_batch = [&](uint32_t c, uint32_t (&x)[4], uint32_t (&wd)[4]) {
        const uint32_t ch = c / BPC, half = c % BPC;   // chunk, batch inside it
        const uint32_t st = ch & (NSTG - 1);
        if (half == 0 && ch < nchunks) mbar_wait(bar0 + 8u * st, (ch / NSTG) & 1u);
        const uint32_t ra = ring + st * (uint32_t)Geo::CHB + half * 512u + lane * 4u;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t v = lds32(ra + 128u * j);
            const uint32_t xc = min(v, C + 1u);   // C + 1: a padding bit, never occupied; 0: the zero row
            x[j] = xc;
            wd[j] = probe(xc >> 5, Ws, s_bm, bm);
        }
        if (half == BPC - 1 && ch + NSTG < nchunks) {   // the chunk's last batch: refill its stage
            __syncwarp();
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // our reads precede the refill
            {
                const uint32_t c2 = ch + NSTG;
                uint64_t b0, b1;   // the stream's byte range (shared memory, pinned address)
                asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(b0), "=l"(b1) : "r"(s_str) : "memory");
                const uintptr_t src = b0 + (uintptr_t)c2 * Geo::CHB;
                const uint32_t bytes = c2 + 1 < nchunks ? (uint32_t)Geo::CHB : (uint32_t)(b1 - src);
                bulk_g2s_elect(ring + st * Geo::CHB, reinterpret_cast<const void*>(src), bytes, bar0 + 8u * st,
                               policy_evict_first());
            }
        }
    };

    uint32_t head = 0, tail = 0;   // compaction ring: queued entries [head, tail) (warp-uniform)
    double G[NLB];
    uint32_t m[NLB];
#pragma unroll
    for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }
    Slot<TV> sl;
    double fv[FOLD ? NLB : 1];   // FOLD: the lane's event's o(e) per layer of the chunk
    bool pend = false;       // a round's slots are in flight
    bool pend_fin = false;   // ... and it is the last round of trial tb + pend_i
    uint32_t pend_i = 0;

    // scan the current batch over its positions [dlo, dhi): append the
    // occupied events in stream order
    // (full: the whole batch belongs to the trial -- no position masks, and
    // invalid ids are caught by a running maximum of id - 1 instead of a per-event test)
    uint32_t idm1 = 0u;   // max of id - 1 over the ids of full batches (>= C: an id outside [1, C])
    uint32_t ltm;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(ltm));
    // append the occupied events of one group (ballot Mj; this lane's event is
    // occupied iff own != 0), in stream order: slot tail + popc(Mj below lane)
    auto append = [&](uint32_t Mj, uint32_t own, uint32_t xj) {
        const uint32_t slot = (tail + __popc(Mj & ltm)) & (uint32_t)(Geo::CBUF - 1);
        // predicated store (no branch around it)
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(
                         cbuf + slot * 4u),
                     "r"(xj), "r"(own)
                     : "memory");
        tail += __popc(Mj);
    };
    uint32_t M3 = 0;   // a deferred group 3 (its ballot), or 0
    // scan the current batch over its positions [dlo, dhi): append the
    // occupied events in stream order.  Groups 0-2 always fit the queue (it
    // holds < 32 entries when a batch starts); group 3 is appended only if it
    // fits, else its ballot is kept (M3) and it is appended after rounds have
    // drained the queue (densely occupied batches only).
    auto scan = [&](bool full, uint32_t dlo, uint32_t dhi, const uint32_t (&x)[4], const uint32_t (&wd)[4]) {
        const uint32_t span = dhi - dlo;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t k = 32u * j + lane;
            const bool live = full || k - dlo < span;
            if (full) idm1 = max(idm1, x[j] - 1u);   // x - 1 >= C (unsigned): an id outside [1, C]
            else err |= (live && x[j] - 1u >= C) ? (uint32_t)ERRBIT_EVENT_RANGE : 0u;
            if (j < 3) {
                // probe bit, ballot and stream-order append in one block (the
                // predicate feeds both the vote and the store)
                uint32_t M;
                asm volatile(
                    "{\n\t.reg .pred p;\n\t.reg .b32 r, a;\n\t"
                    "shf.r.wrap.b32 r, %1, %1, %2;\n\t"
                    "and.b32 r, r, %3;\n\t"
                    "setp.ne.u32 p, r, 0;\n\t"
                    "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
                    "and.b32 a, %0, %4;\n\t"
                    "popc.b32 a, a;\n\t"
                    "add.u32 a, a, %5;\n\t"
                    "and.b32 a, a, %6;\n\t"
                    "mad.lo.u32 a, a, 4, %7;\n\t"
                    "@p st.shared.u32 [a], %2;\n\t}"
                    : "=r"(M)
                    : "r"(wd[j]), "r"(x[j]), "r"(live ? 1u : 0u), "r"(ltm), "r"(tail), "n"(Geo::CBUF - 1), "r"(cbuf)
                    : "memory");
                tail += __popc(M);
                continue;
            }
            uint32_t r;
            asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(wd[j]), "r"(x[j]));
            const uint32_t own = live ? (r & 1u) : 0u;
            const uint32_t M = __ballot_sync(0xffffffffu, own != 0u);
            if (j == 3 && tail - head + __popc(M) > (uint32_t)Geo::CBUF) {
                M3 = M;
                break;
            }
            append(M, own, x[j]);
        }
    };
    // a7 tree + a8 stores of trial t (lane 0), accumulators reset
    auto finalize = [&](uint64_t t) {
#pragma unroll
        for (int l = 0; l < NLB; ++l) {
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) G[l] = __dadd_rn(G[l], __shfl_xor_sync(0xffffffffu, G[l], off));
            m[l] = __reduce_add_sync(0xffffffffu, m[l]);
        }
        if (lane == 0) store_trial(p, t, G, m);
#pragma unroll
        for (int l = 0; l < NLB; ++l) { G[l] = 0.0; m[l] = 0u; }
    };
    // a4-a7 for the lane's event of the pending round (a lane without one
    // adds +0); the trial's tree and stores when it was its last round
    auto consume = [&]() {
        pend = false;
        if constexpr (FOLD) {
#pragma unroll
            for (int l = 0; l < NLB; ++l) {
                if (l > 0 && l >= (int)p.n_layers) break;
                const double o = fv[l];   // a lane without an event holds +0
                G[l] = __dadd_rn(G[l], o);
                m[l] += (o > 0.0) ? 1u : 0u;
            }
            if (pend_fin) {
                pend_fin = false;
                finalize(tb + pend_i);
            }
            return;
        }
        const uint32_t mask = sl.mask();
        double le[NLB];
#pragma unroll
        for (int l = 0; l < NLB; ++l) le[l] = 0.0;
        auto add = [&](double xv, uint32_t j) {
            // a tower whose layers share the per-ELT terms (same ELT set): the
            // terms of a looked-up loss are evaluated once and added to every
            // layer's event loss -- identical inputs, identical f_j
            if (NLB > 1 && p.same_terms) {
                const double2 tc = lds_f64x2(s_tm + j * 16u);
                const double f = terms(xv, tc.x, tc.y);
#pragma unroll
                for (int l = 0; l < NLB; ++l)
                    if (l == 0 || l < (int)p.n_layers) le[l] = __dadd_rn(le[l], f);
                return;
            }
#pragma unroll
            for (int l = 0; l < NLB; ++l) {
                if (l == 0 || l < (int)p.n_layers) {
                    const double2 tc = lds_f64x2(s_tm + ((uint32_t)l * 32u + j) * 16u);
                    le[l] = __dadd_rn(le[l], terms(xv, tc.x, tc.y));
                }
            }
        };
        const bool fits = __popc(mask) <= CAP;
        // the round's longest row: one reduction decides both whether every row
        // fits its slot and how many walk steps the round needs (no vote per step)
        const uint32_t vmax = __reduce_max_sync(0xffffffffu, (uint32_t)__popc(mask));
        if (vmax <= (uint32_t)CAP) {
            // every lane's slot holds all of its row's non-zeros (the common
            // case): walk them in column order, the v-th from slot value v --
            // unrolled, so v is a register name, and branch-free: a lane whose
            // walk has ended (or whose column is outside the window) adds
            // terms(0) = +0, which leaves l_e unchanged (every deductible >= 0)
            uint32_t mm = mask;
#pragma unroll
            for (int v = 0; v < CAP; ++v) {
                if ((uint32_t)v >= vmax) break;   // (vmax >= 1: a round holds an occupied event)
                const uint32_t b = (uint32_t)(__ffs(mm) - 1);   // 0xffffffff when mm == 0
                mm &= mm - 1u;
                const uint32_t j = b - p.pk_col0;                // window element (wraps when b < col0)
                const bool in = j < 32u && ((p.pk_wmask >> j) & 1u);
                add(in ? sl.val((uint32_t)v) : 0.0, in ? j : 0u);
            }
        } else if (fits) {
            uint32_t mm = mask, v = 0;
            while (mm) {
                const uint32_t b = (uint32_t)(__ffs(mm) - 1);
                mm &= mm - 1u;
                const uint32_t j = b - p.pk_col0;
                if (j < 32u && ((p.pk_wmask >> j) & 1u)) add(sl.val(v), j);
                ++v;
            }
        } else {
            // more non-zeros than the slot holds: the rest from the dense table
            uint32_t mm = (mask >> p.pk_col0) & p.pk_wmask;
            while (mm) {
                const uint32_t j = (uint32_t)(__ffs(mm) - 1);
                mm &= mm - 1u;
                const uint32_t v = __popc(mask & ((1u << (j + p.pk_col0)) - 1u));
                const double xv = v < (uint32_t)CAP ? sl.val(v)
                                                    : (double)__ldg(static_cast<const TV*>(p.table) + p.sec_off[0] +
                                                                    (uint64_t)sl.id() * p.row_stride + j);
                add(xv, j);
            }
        }
#pragma unroll
        for (int l = 0; l < NLB; ++l) {
            if (l > 0 && l >= (int)p.n_layers) break;   // (a launch has >= 1 layer)
            const double o = terms(le[l], p.lw[l].occ_r, p.lw[l].occ_l);
            G[l] = __dadd_rn(G[l], o);
            m[l] += (o > 0.0) ? 1u : 0u;
        }
        if (pend_fin) {
            pend_fin = false;
            finalize(tb + pend_i);
        }
    };
    // issue a round of trial t: up to 32 queued events, entry head + i to lane i
    auto issue_round = [&](uint32_t i) {   // a round of trial tb + i
        __syncwarp();   // the scan's appends (other lanes' stores) are visible
        const uint32_t nr = tail - head < 32u ? tail - head : 32u;
        if constexpr (FOLD) {
            if (lane < nr) {
                const uint32_t e = lds32(cbuf + ((head + lane) & (uint32_t)(Geo::CBUF - 1)) * 4u);
                const double* src = p.fold + (uint64_t)e * NLB;   // fold row stride = NLB (host)
                if constexpr (NLB == 1) {
                    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(fv[0]) : "l"(src));
                } else if constexpr (NLB == 2) {
                    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];"
                                 : "=d"(fv[0]), "=d"(fv[1]) : "l"(src));
                } else {
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                                 : "=d"(fv[0]), "=d"(fv[1]), "=d"(fv[2]), "=d"(fv[3]) : "l"(src));
                }
            } else {
#pragma unroll
                for (int l = 0; l < NLB; ++l) fv[l] = 0.0;
            }
        } else {
            if (lane < nr) {
                const uint32_t e = lds32(cbuf + ((head + lane) & (uint32_t)(Geo::CBUF - 1)) * 4u);
                ld_slot(static_cast<const char*>(p.pk) + (uint64_t)e * kPackBytes, sl.q);
            } else {
                sl.q[0] = 0; sl.q[1] = 0; sl.q[2] = 0; sl.q[3] = 0;
            }
        }
        head += nr;
        pend = true;
        pend_i = i;
    };

    // two register sets, A and B, alternate between the current batch and the
    // next one (no copies): batch c lives in set (c & 1)
    uint32_t xa[4], wa[4], xb[4], wb[4];
    load_batch(0, xa, wa);
    load_batch(1, xb, wb);
    uint32_t c = 0;                                   // current batch
    uint32_t rlo = (uint32_t)(S0 - P0);               // next position of the stream
    const uint32_t rS1 = (uint32_t)(S1 - P0);
    const uint64_t B0 = base + (uint64_t)P0;          // offset value of stream position 0
    // trial tb + i ends at stream position rhi; the end of the next trial is
    // loaded one trial ahead (o_nx) and converted when that trial starts
    const uint32_t nt = te - tb < 0xffffffffull ? (uint32_t)(te - tb) : 0u;   // (a warp never holds 2^32 trials)
    auto to_pos = [&](uint64_t o) {   // offset value -> 32-bit stream position, validated
        const int64_t h = (int64_t)(o - B0);
        uint32_t r = (uint32_t)h;
        if (h < (int64_t)rlo) { err |= ERRBIT_OFFSETS; r = rlo; }
        if (r > rS1) { err |= ERRBIT_OFFSETS; r = rS1 > rlo ? rS1 : rlo; }
        return r;
    };
    uint64_t o_nx = nt ? __ldg(p.off + tb + 1) : 0;
#pragma unroll 1
    for (uint32_t i = 0; i < nt; ++i) {
        const uint32_t rhi = to_pos(o_nx);
        if (i + 1 < nt) o_nx = __ldg(p.off + tb + i + 2);   // the next trial's end, one trial ahead
#pragma unroll 1
        for (;;) {
            const uint32_t bs = c * CHE;
            if (rlo <= bs && rhi >= bs + CHE) {   // the whole batch belongs to the trial
                if (c & 1u) scan(true, 0u, CHE, xb, wb);
                else scan(true, 0u, CHE, xa, wa);
            } else {
                const uint32_t dlo = rlo > bs ? rlo - bs : 0u;            // <= CHE
                const uint32_t dhi = rhi - bs < CHE ? rhi - bs : CHE;
                if (dhi > dlo) {
                    if (c & 1u) scan(false, dlo, dhi, xb, wb);
                    else scan(false, dlo, dhi, xa, wa);
                }
            }
            const bool fin = rhi <= bs + CHE;   // the trial ends in this batch
#pragma unroll 1
            for (;;) {
                // full rounds; at the trial's end (no group deferred) every queued entry
                const uint32_t need = (fin && !M3) ? 1u : 32u;
#pragma unroll 1
                while (tail - head >= need) {
                    if (pend) consume();
                    issue_round(i);
                }
                if (!M3) break;
                append(M3, (M3 >> lane) & 1u, (c & 1u) ? xb[3] : xa[3]);   // the deferred group 3 now fits
                M3 = 0;
            }
            if (fin) break;
            // the finished batch's set receives batch c + 2
            if (c & 1u) load_batch(c + 2, xb, wb);
            else load_batch(c + 2, xa, wa);
            ++c;
        }
        if (pend && pend_i == i) {
            pend_fin = true;   // finished when the next round is issued (or at the end)
        } else {
            if (pend) consume();   // the previous trial's last round (finalises it)
            finalize(tb + i);      // no round of the trial in flight: its sum is complete
        }
        rlo = rhi;
    }
    if (pend) consume();
    // every issued chunk has landed before the CTA's shared memory is released
    // (batches 0 .. c+1 were loaded: chunks 0 .. (c+1)/BPC waited for; the
    // (c+2)/BPC chunks whose last batch was loaded each issued a refill)
    const uint32_t waited_ch = (c + 1) / BPC + 1;
    const uint32_t loaded = waited_ch < nchunks ? waited_ch : nchunks;
    const uint32_t issued = NSTG + (c + 2) / BPC < nchunks ? NSTG + (c + 2) / BPC : nchunks;
    for (uint32_t cc = loaded; cc < issued; ++cc) mbar_wait(bar0 + 8u * (cc & (NSTG - 1)), (cc / NSTG) & 1u);
    if (idm1 >= C) err |= ERRBIT_EVENT_RANGE;
    if (lane == 0 && p.n_gathered && tail) atomicAdd(p.n_gathered, (unsigned long long)tail);   // queue entries = gathers
    peer_fence(p);
    if (err) atomicOr(p.err, err);
}

template <typename TV, int NLB, bool FOLD = false>
void* pick_bc_nl(int* warps, int* fixed) {
    using Geo = BcGeo<BcWarps<NLB>::value, BcQueue<NLB>::value>;
    *warps = Geo::WARPS;
    *fixed = Geo::FIXED;
    return (void*)trial_kernel_bc<TV, NLB, FOLD>;
}
template <typename TV>
void* pick_bc(int nl, int* warps, int* fixed) {
    if (nl <= 1) return pick_bc_nl<TV, 1>(warps, fixed);
    if (nl <= 2) return pick_bc_nl<TV, 2>(warps, fixed);
    return pick_bc_nl<TV, 4>(warps, fixed);
}
// fold mode: the template's layer count is the fold row stride (1, 2 or 4)
void* pick_bc_fold(int stride, int* warps, int* fixed) {
    if (stride <= 1) return pick_bc_nl<double, 1, true>(warps, fixed);
    if (stride <= 2) return pick_bc_nl<double, 2, true>(warps, fixed);
    return pick_bc_nl<double, 4, true>(warps, fixed);
}

}  // namespace

// One CTA of 24-32 warps per SM; dynamic shared memory = the rings plus as much
// of the occupancy bitmap as the opt-in limit leaves (a 16-B multiple).
cudaError_t launch_trials_bc(const TrialParams& p, int fp32, int grid, cudaStream_t s) {
    if (p.t_end <= p.t_begin) return cudaSuccess;
    const bool fold = fp32 < 0;   // fp32 = -1: fold mode (rounds gather o(e) from p.fold)
    if (!p.bm || (!fold && !p.pk) || (fold && (!p.fold || (p.fold_stride != 1 && p.fold_stride != 2 &&
                                                             p.fold_stride != 4))))
        return cudaErrorInvalidValue;
    int warps = 16, fixed = 0;
    void* fn = fold ? pick_bc_fold((int)p.fold_stride, &warps, &fixed)
               : fp32 ? pick_bc<float>((int)p.n_layers, &warps, &fixed)
                      : pick_bc<double>((int)p.n_layers, &warps, &fixed);
    // the device's opt-in limit and the kernel's static shared memory, queried
    // once per kernel and device (host time between the calls of a step is GPU
    // idle time)
    struct AttrCache { void* fn; int dev, optin, stat, dyn_set; };
    static AttrCache cache[16] = {};
    static std::mutex mu;   // contexts may launch from several host threads
    std::lock_guard<std::mutex> lock(mu);
    int dev = 0;
    cudaGetDevice(&dev);
    AttrCache* ac = nullptr;
    for (auto& x : cache)
        if (x.fn == fn && x.dev == dev) { ac = &x; break; }
    if (!ac) {
        int optin = 0;
        cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cudaFuncAttributes fa{};
        cudaError_t e = cudaFuncGetAttributes(&fa, fn);
        if (e != cudaSuccess) return e;
        for (auto& x : cache)
            if (!x.fn) { x = AttrCache{fn, dev, optin, (int)fa.sharedSizeBytes, -1}; ac = &x; break; }
        if (!ac) { static AttrCache spill; spill = AttrCache{fn, dev, optin, (int)fa.sharedSizeBytes, -1}; ac = &spill; }
    }
    const int64_t avail = (int64_t)ac->optin - (int64_t)ac->stat - fixed;
    uint64_t ws = avail > 0 ? (uint64_t)avail / 16 * 4 : 0;   // words, 16-B multiple
    const uint64_t need = (((uint64_t)p.catalog + 1 + 31) / 32 + 3) / 4 * 4;   // within the padded bitmap
    if (ws > need) ws = need;
    if (const char* v = getenv("ARA_BC_SMEM_WORDS")) {   // A/B: cap the shared-memory part of the bitmap
        const uint64_t cap = strtoull(v, nullptr, 10) / 4 * 4;
        if (cap < ws) ws = cap;
    }
    TrialParams q = p;
    q.bm_smem_words = (uint32_t)ws;
    const size_t dyn = (size_t)fixed + ws * 4;
    if (ac->dyn_set < (int)dyn) {
        const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        if (e != cudaSuccess) return e;
        ac->dyn_set = (int)dyn;
    }
    void* args[] = {(void*)&q};
    return cudaLaunchKernel(fn, dim3(grid > 0 ? grid : 1), dim3(warps * 32), args, dyn, s);
}

}  // namespace ara
