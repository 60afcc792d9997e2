// metrics_fast.cu -- PML / TVaR (readings
// A9/A10) in four kernels instead of ten: two wide radix passes, one
// compaction, one exact finish.
//
//   k = ceil(T / R);  PML(R) = k-th largest Y;  TVaR(R) = mean of the k largest.
//
// Keys are the u64 bit patterns of the (non-negative, canonical +0) YLT
// values: for non-negative doubles the bit order is the value order.
//  A  histogram of bits 63..52 (sign + exponent: 4096 bins) of every key,
//     shared by all return periods; the last block picks each period's bin;
//  B  histogram of bits 51..40 of the keys inside each picked bin (one 4096-
//     bin histogram per distinct bin); the last block picks the next 12 bits
//     and lays out, per distinct 24-bit prefix, a segment of the candidate
//     buffer sized by that bin's exact count;
//  C  one sweep: keys ABOVE a period's 24-bit bin add to its tail sum and
//     count (a per-thread sequential sum in key-index order, then the blocks'
//     partials in block order -- deterministic); keys INSIDE a distinct bin are
//     copied to its segment (order irrelevant, see D);
//  D  one block per distinct bin: radix select of the remaining 40 bits over
//     its candidates (shared memory when they fit), then the sum of the
//     candidates above v -- they share the exponent, so it is an exact integer
//     sum of their significands (order-independent) scaled once:
//       TVaR = (tail_above + sum_gt + (k - cnt_above - cnt_gt) v) / k,
//     which is the mean of the k largest (ties included).  On integer-valued
//     YLTs every term is exact, as the oracle's sequential sum is.
// Only single-shard YLTs (one GPU, or every rank on the assembled global
// YLT); the distributed select stays in metrics.cu.
#include <cstdlib>

#include "ara_internal.cuh"

namespace ara {
namespace {

constexpr int kBins = 4096;          // 12-bit digits
constexpr int kRC = 10;              // return periods per tail sweep of kernel C
constexpr int kFinSmemKeys = 16384;  // candidates kernel D selects in shared memory
constexpr uint32_t kBSmem = 4;       // pass-B histograms in shared memory (the periods' distinct
                                     // exponent bins; more go straight to the global histogram)

struct FParams {
    const double* ylt;
    uint64_t T, ld;
    uint32_t rows, n_rp, nblk;
    uint32_t* hist;        // [rows][kBins]            pass A
    uint32_t* hist2;       // [rows][n_rp][kBins]      pass B, slot = the period's rep
    uint64_t* pre;         // [rows][n_rp]             selected prefix (bits 63..40 after B)
    uint64_t* krem;        // [rows][n_rp]             rank inside the selected bin
    uint32_t* rep;         // [rows][n_rp]             first period with the same prefix
    uint64_t* seg;         // [rows][n_rp][2]          candidate segment (offset, count) of a rep
    uint32_t* fill;        // [rows][n_rp]             appended so far
    uint64_t* cand;        // [rows][T]                candidate keys
    double* part_sum;      // [rows][n_rp][nblk]
    uint64_t* part_cnt;    // [rows][n_rp][nblk]
    double* above_sum;     // [rows][n_rp]
    uint64_t* above_cnt;   // [rows][n_rp]
    uint32_t* done;        // [rows][3] last-block counters of A, B, C
    double* out;           // [rows][n_rp][2]
    uint64_t k[ARA_MAX_RP];
};

__device__ __forceinline__ uint64_t fkey(double y) { return (uint64_t)__double_as_longlong(y + 0.0); }

// the digit d of a descending scan of `h` (kBins counts) where the kr-th
// largest falls: count(bins > d) < kr <= count(bins >= d); returns d and the
// count above it.  One warp; lane l owns bins 4095-128l .. 3968-128l.
__device__ void warp_pick(const uint32_t* h, uint64_t kr, uint32_t& d, uint64_t& above) {
    const uint32_t lane = threadIdx.x & 31u;
    uint64_t tot = 0;
    for (int q = 0; q < 128; ++q) tot += h[kBins - 1 - 128 * lane - q];
    uint64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += v;
    }
    const uint64_t excl = incl - tot;
    const unsigned hit = __ballot_sync(0xffffffffu, excl < kr && kr <= incl);
    const uint32_t src = hit ? (uint32_t)(__ffs(hit) - 1) : 31u;
    uint32_t dd = 0;
    uint64_t ab = 0;
    if (lane == src) {
        uint64_t cum = excl;
        dd = kBins - 1 - 128 * lane - 127;
        for (int q = 0; q < 128; ++q) {
            const uint32_t c = h[kBins - 1 - 128 * lane - q];
            if (kr <= cum + c) { dd = kBins - 1 - 128 * lane - q; break; }
            cum += c;
        }
        ab = cum;
    }
    d = __shfl_sync(0xffffffffu, dd, src);
    above = __shfl_sync(0xffffffffu, ab, src);
}

// warp_pick over a global histogram written by other blocks' atomics
__device__ void warp_pick_global(const uint32_t* gh, uint64_t kr, uint32_t& d, uint64_t& above) {
    const uint32_t lane = threadIdx.x & 31u;
    uint64_t tot = 0;
    for (int q = 0; q < 128; ++q) tot += __ldcg(gh + kBins - 1 - 128 * lane - q);
    uint64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += v;
    }
    const uint64_t excl = incl - tot;
    const unsigned hit = __ballot_sync(0xffffffffu, excl < kr && kr <= incl);
    const uint32_t src = hit ? (uint32_t)(__ffs(hit) - 1) : 31u;
    uint32_t dd = 0;
    uint64_t ab = 0;
    if (lane == src) {
        uint64_t cum = excl;
        dd = kBins - 1 - 128 * lane - 127;
        for (int q = 0; q < 128; ++q) {
            const uint32_t c = __ldcg(gh + kBins - 1 - 128 * lane - q);
            if (kr <= cum + c) { dd = kBins - 1 - 128 * lane - q; break; }
            cum += c;
        }
        ab = cum;
    }
    d = __shfl_sync(0xffffffffu, dd, src);
    above = __shfl_sync(0xffffffffu, ab, src);
}

// block-level "last block of this row" hand-off
__device__ bool last_block(uint32_t* counter, uint32_t n) {
    __shared__ uint32_t s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == n - 1) ? 1u : 0u;
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// add a block's shared histogram into the global one
__device__ void merge_hist(const uint32_t* sh, uint32_t* gh, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
        if (sh[i]) atomicAdd(gh + i, sh[i]);
}

__global__ void __launch_bounds__(256) fm_pass_a(const __grid_constant__ FParams P) {
    __shared__ uint32_t sh[kBins];
    const uint32_t row = blockIdx.y, lane = threadIdx.x & 31u;
    for (uint32_t i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    const double* y = P.ylt + (uint64_t)row * P.ld;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < P.T; i0 += stride) {   // warp-uniform trips
        const uint64_t i = i0 + threadIdx.x;
        const uint32_t d = i < P.T ? (uint32_t)(fkey(__ldcg(y + i)) >> 52) : 0xffffffffu;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        if (d != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&sh[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    merge_hist(sh, P.hist + (uint64_t)row * kBins, kBins);
    if (!last_block(P.done + row * 3 + 0, P.nblk)) return;
    // pick the bin of every return period (one warp each)
    const uint32_t* gh = P.hist + (uint64_t)row * kBins;
    for (uint32_t i = threadIdx.x; i < kBins; i += blockDim.x) sh[i] = __ldcg(gh + i);
    __syncthreads();
    for (uint32_t r = threadIdx.x >> 5; r < P.n_rp; r += blockDim.x >> 5) {
        uint32_t d;
        uint64_t above;
        warp_pick(sh, P.k[r], d, above);
        if (lane == 0) {
            P.pre[row * P.n_rp + r] = (uint64_t)d << 52;
            P.krem[row * P.n_rp + r] = P.k[r] - above;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (uint32_t r = 0; r < P.n_rp; ++r) {
            uint32_t rr = r;
            for (uint32_t q = 0; q < r; ++q)
                if (__ldcg(P.pre + row * P.n_rp + q) == __ldcg(P.pre + row * P.n_rp + r)) { rr = q; break; }
            P.rep[row * P.n_rp + r] = rr;
        }
    }
}

__global__ void __launch_bounds__(256) fm_pass_b(const __grid_constant__ FParams P) {
    extern __shared__ uint32_t sh2[];              // [n_rep][kBins]
    __shared__ uint8_t s_map[kBins];               // top 12 bits -> rep slot index + 1 (0: none)
    __shared__ uint32_t s_slot[ARA_MAX_RP];        // rep slot -> period index
    __shared__ uint32_t s_nu;
    const uint32_t row = blockIdx.y, lane = threadIdx.x & 31u, n_rp = P.n_rp;
    for (uint32_t i = threadIdx.x; i < kBins; i += blockDim.x) s_map[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t nu = 0;
        for (uint32_t r = 0; r < n_rp; ++r)
            if (P.rep[row * n_rp + r] == r) {
                s_slot[nu] = r;
                s_map[P.pre[row * n_rp + r] >> 52] = (uint8_t)(nu + 1);
                ++nu;
            }
        s_nu = nu;
    }
    __syncthreads();
    const uint32_t nu = s_nu;
    const uint32_t ns = nu < kBSmem ? nu : kBSmem;   // histograms kept in shared memory
    uint32_t* gh = P.hist2 + (uint64_t)row * n_rp * kBins;
    for (uint32_t i = threadIdx.x; i < ns * kBins; i += blockDim.x) sh2[i] = 0u;
    __syncthreads();
    const double* y = P.ylt + (uint64_t)row * P.ld;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < P.T; i0 += stride) {
        const uint64_t i = i0 + threadIdx.x;
        uint32_t tag = 0xffffffffu;
        if (i < P.T) {
            const uint64_t key = fkey(__ldcg(y + i));
            const uint32_t u = s_map[key >> 52];
            if (u) tag = (u - 1) * kBins + (uint32_t)((key >> 40) & (kBins - 1));
        }
        const unsigned peers = __match_any_sync(0xffffffffu, tag);
        if (tag != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1)) {
            const uint32_t u = tag / kBins;
            if (u < ns) atomicAdd(&sh2[tag], (uint32_t)__popc(peers));
            else atomicAdd(gh + (uint64_t)s_slot[u] * kBins + (tag % kBins), (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    for (uint32_t u = 0; u < ns; ++u) merge_hist(sh2 + u * kBins, gh + (uint64_t)s_slot[u] * kBins, kBins);
    if (!last_block(P.done + row * 3 + 1, P.nblk)) return;
    // pick the next 12 bits of every period inside its pass-A bin (the
    // histograms of the distinct bins, staged coherently in shared memory)
    for (uint32_t u = 0; u < ns; ++u)
        for (uint32_t i = threadIdx.x; i < kBins; i += blockDim.x)
            sh2[u * kBins + i] = __ldcg(gh + (uint64_t)s_slot[u] * kBins + i);
    __syncthreads();
    // (bins past kBSmem are read from the global histogram, coherently: __ldcg)
    auto hist_of = [&](uint32_t u) -> const uint32_t* { return u < ns ? sh2 + u * kBins : nullptr; };
    for (uint32_t r = threadIdx.x >> 5; r < n_rp; r += blockDim.x >> 5) {
        const uint32_t u = s_map[P.pre[row * n_rp + r] >> 52] - 1u;   // this period's pass-A bin
        uint32_t d;
        uint64_t above;
        if (hist_of(u)) warp_pick(hist_of(u), P.krem[row * n_rp + r], d, above);
        else warp_pick_global(gh + (uint64_t)s_slot[u] * kBins, P.krem[row * n_rp + r], d, above);
        if (lane == 0) {
            P.pre[row * n_rp + r] |= (uint64_t)d << 40;
            P.krem[row * n_rp + r] -= above;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // distinct 24-bit prefixes: candidate segments sized by their bins' exact counts
        uint64_t off = 0;
        for (uint32_t r = 0; r < n_rp; ++r) {
            const uint64_t pr = __ldcg(P.pre + row * n_rp + r);
            uint32_t rr = r;
            for (uint32_t q = 0; q < r; ++q)
                if (__ldcg(P.pre + row * n_rp + q) == pr) { rr = q; break; }
            if (rr == r) {
                const uint32_t u = s_map[pr >> 52] - 1u;
                const uint32_t dig = (uint32_t)((pr >> 40) & (kBins - 1));
                const uint64_t cnt = u < ns ? sh2[u * kBins + dig] : __ldcg(gh + (uint64_t)s_slot[u] * kBins + dig);
                P.seg[(row * n_rp + r) * 2 + 0] = off;
                P.seg[(row * n_rp + r) * 2 + 1] = cnt;
                off += cnt;
            }
            P.rep[row * n_rp + r] = rr;
            P.fill[row * n_rp + r] = 0;
        }
    }
}

// C: tail sums above each period's 24-bit bin + candidate copy
__global__ void __launch_bounds__(256) fm_pass_c(const __grid_constant__ FParams P) {
    __shared__ double s_sum[kRC][256];
    __shared__ uint64_t s_cnt[kRC][256];
    __shared__ uint64_t s_pre[ARA_MAX_RP];     // distinct 24-bit prefixes (bits 63..40) ...
    __shared__ uint32_t s_prr[ARA_MAX_RP];     // ... and their periods
    __shared__ uint32_t s_nu;
    const uint32_t row = blockIdx.y, lane = threadIdx.x & 31u, n_rp = P.n_rp;
    if (threadIdx.x == 0) {
        uint32_t nu = 0;
        for (uint32_t r = 0; r < n_rp; ++r)
            if (P.rep[row * n_rp + r] == r) { s_pre[nu] = P.pre[row * n_rp + r]; s_prr[nu] = r; ++nu; }
        s_nu = nu;
    }
    __syncthreads();
    const uint32_t nu = s_nu;
    const double* y = P.ylt + (uint64_t)row * P.ld;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    // candidate copy (once, with the first sweep)
    for (uint32_t r0 = 0; r0 < n_rp; r0 += kRC) {
        uint64_t hi[kRC];
        double sm[kRC];
        uint64_t cn[kRC];
#pragma unroll
        for (int j = 0; j < kRC; ++j) {
            // keys above the bin: key > prefix | (2^40 - 1); periods past n_rp: none
            hi[j] = r0 + j < n_rp ? (P.pre[row * n_rp + r0 + j] | ((1ull << 40) - 1)) : ~0ull;
            sm[j] = 0.0;
            cn[j] = 0;
        }
        for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < P.T; i0 += stride) {   // warp-uniform trips
            const uint64_t i = i0 + threadIdx.x;
            const bool ok = i < P.T;
            const double v = ok ? __ldcg(y + i) + 0.0 : 0.0;
            const uint64_t key = ok ? fkey(v) : 0ull;
#pragma unroll
            for (int j = 0; j < kRC; ++j)   // per-thread sequential, key-index order
                if (ok && key > hi[j]) { sm[j] = __dadd_rn(sm[j], v); ++cn[j]; }
            if (r0 == 0) {
                uint32_t which = 0xffffffffu;
                if (ok)
                    for (uint32_t u = 0; u < nu; ++u)
                        if ((key >> 40) == (s_pre[u] >> 40)) which = u;
                const unsigned peers = __match_any_sync(0xffffffffu, which);
                if (which != 0xffffffffu) {
                    const uint32_t leader = (uint32_t)(__ffs(peers) - 1);
                    const uint32_t r = s_prr[which];
                    uint32_t base = 0;
                    if (lane == leader) base = atomicAdd(P.fill + row * n_rp + r, (uint32_t)__popc(peers));
                    base = __shfl_sync(peers, base, leader);
                    const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
                    P.cand[(uint64_t)row * P.T + P.seg[(row * n_rp + r) * 2] + base + rank] = key;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kRC; ++j) { s_sum[j][threadIdx.x] = sm[j]; s_cnt[j][threadIdx.x] = cn[j]; }
        __syncthreads();
        for (int w = 128; w >= 1; w >>= 1) {   // fixed tree over the block's threads
            if ((int)threadIdx.x < w) {
#pragma unroll
                for (int j = 0; j < kRC; ++j) {
                    s_sum[j][threadIdx.x] = __dadd_rn(s_sum[j][threadIdx.x], s_sum[j][threadIdx.x + w]);
                    s_cnt[j][threadIdx.x] += s_cnt[j][threadIdx.x + w];
                }
            }
            __syncthreads();
        }
        if (threadIdx.x < kRC && r0 + threadIdx.x < n_rp) {
            const uint32_t r = r0 + threadIdx.x;
            P.part_sum[((uint64_t)row * n_rp + r) * P.nblk + blockIdx.x] = s_sum[threadIdx.x][0];
            P.part_cnt[((uint64_t)row * n_rp + r) * P.nblk + blockIdx.x] = s_cnt[threadIdx.x][0];
        }
        __syncthreads();
    }
    if (!last_block(P.done + row * 3 + 2, P.nblk)) return;
    // the blocks' partials in block order (one warp per period)
    const uint32_t wid = threadIdx.x >> 5;
    for (uint32_t r = wid; r < n_rp; r += blockDim.x >> 5) {
        const double* ps = P.part_sum + ((uint64_t)row * n_rp + r) * P.nblk;
        const uint64_t* pc = P.part_cnt + ((uint64_t)row * n_rp + r) * P.nblk;
        double sum = 0.0;
        uint64_t c = 0;
        for (uint32_t b0 = 0; b0 < P.nblk; b0 += 32) {
            const uint32_t b = b0 + lane;
            const double x = b < P.nblk ? __ldcg(ps + b) : 0.0;
            const uint64_t yc = b < P.nblk ? __ldcg(pc + b) : 0ull;
            for (uint32_t q = 0; q < 32 && b0 + q < P.nblk; ++q) {
                sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, x, q));
                c += __shfl_sync(0xffffffffu, yc, q);
            }
        }
        if (lane == 0) {
            P.above_sum[row * n_rp + r] = sum;
            P.above_cnt[row * n_rp + r] = c;
        }
    }
}

// D: per distinct 24-bit bin (blockIdx.x = its period slot), the remaining
// 40 bits by radix select over its candidates, then the exact sum of the
// candidates above the selected value
__global__ void __launch_bounds__(1024) fm_pass_d(const __grid_constant__ FParams P) {
    extern __shared__ __align__(16) unsigned char dsm[];
    uint64_t* sk = reinterpret_cast<uint64_t*>(dsm);                 // candidates (when they fit)
    __shared__ uint32_t sh[1024];                                    // 10-bit digit histogram
    __shared__ uint32_t sh0[1024];                                   // first-digit histogram (shared by the bin's periods)
    __shared__ uint32_t s_d;
    __shared__ uint64_t s_above;
    __shared__ unsigned long long s_lo[32], s_hi[32];
    __shared__ unsigned long long s_cgt[32];
    const uint32_t row = blockIdx.y, r0 = blockIdx.x, n_rp = P.n_rp;
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    if (r0 >= n_rp || P.rep[row * n_rp + r0] != r0) return;
    const uint64_t off = P.seg[(row * n_rp + r0) * 2], n = P.seg[(row * n_rp + r0) * 2 + 1];
    const uint64_t* gk = P.cand + (uint64_t)row * P.T + off;
    const bool in_smem = n <= (uint64_t)kFinSmemKeys;
    if (in_smem) {
        for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) sk[i] = __ldcg(gk + i);
        __syncthreads();
    }
    auto key_at = [&](uint64_t i) { return in_smem ? sk[i] : __ldcg(gk + i); };
    // histogram of digit (key >> shift) & 1023 over the candidates matching
    // `pre` on the bits above it: 4 keys per thread per step (independent
    // loads), lanes with equal digits merged (ties pile onto one bin)
    auto histogram = [&](uint32_t* h, int shift, uint64_t hmask, uint64_t pre) {
        for (uint32_t i = threadIdx.x; i < 1024; i += blockDim.x) h[i] = 0u;
        __syncthreads();
        for (uint64_t i0 = 0; i0 < n; i0 += 4ull * blockDim.x) {   // block-uniform trips
            uint64_t kk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = i0 + (uint64_t)u * blockDim.x + threadIdx.x;
                kk[u] = i < n ? key_at(i) : ~0ull;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool ok = kk[u] != ~0ull && (kk[u] & hmask) == (pre & hmask);
                const uint32_t tag = ok ? (uint32_t)((kk[u] >> shift) & 1023u) : 0xffffffffu;
                const unsigned peers = __match_any_sync(0xffffffffu, tag);
                if (tag != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&h[tag], (uint32_t)__popc(peers));
            }
        }
        __syncthreads();
    };
    histogram(sh0, 30, ~((1ull << 40) - 1), P.pre[row * n_rp + r0]);   // same for every period of the bin
    const uint64_t top = P.pre[row * n_rp + r0] >> 40;   // the 24-bit prefix every candidate shares
    for (uint32_t r = r0; r < n_rp; ++r) {               // every period of this bin
        if (P.rep[row * n_rp + r] != r0) continue;
        uint64_t pre = P.pre[row * n_rp + r], kr = P.krem[row * n_rp + r];
        // 4 passes of 10 bits: bits 39..30, 29..20, 19..10, 9..0
        for (int pass = 0; pass < 4; ++pass) {
            const int shift = 30 - 10 * pass;
            const uint64_t hmask = ~((1ull << (shift + 10)) - 1);   // bits already fixed
            const uint32_t* hh = sh0;
            if (pass > 0) {
                histogram(sh, shift, hmask, pre);
                hh = sh;
            }
            if (wid == 0) {   // descending scan: lane l owns digits 1023-32l .. 992-32l
                uint64_t tot = 0;
                for (int q = 0; q < 32; ++q) tot += hh[1023 - 32 * lane - q];
                uint64_t incl = tot;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= (uint32_t)o) incl += v;
                }
                const uint64_t excl = incl - tot;
                const unsigned hit = __ballot_sync(0xffffffffu, excl < kr && kr <= incl);
                const uint32_t src = hit ? (uint32_t)(__ffs(hit) - 1) : 31u;
                if (lane == src) {
                    uint64_t cum = excl;
                    uint32_t dd = 1023 - 32 * lane - 31;
                    for (int q = 0; q < 32; ++q) {
                        const uint32_t c = hh[1023 - 32 * lane - q];
                        if (kr <= cum + c) { dd = 1023 - 32 * lane - q; break; }
                        cum += c;
                    }
                    s_d = dd;
                    s_above = cum;
                }
            }
            __syncthreads();
            pre |= (uint64_t)s_d << shift;
            kr -= s_above;
            __syncthreads();
        }
        // v = the selected key; exact sum and count of the candidates above it:
        // they share sign and exponent, so value = significand * 2^(exp - 1075)
        const uint64_t v = pre;
        unsigned long long lo = 0, hi = 0, cgt = 0;
        for (uint64_t i0 = 0; i0 < n; i0 += 4ull * blockDim.x) {
            uint64_t kk[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t i = i0 + (uint64_t)u * blockDim.x + threadIdx.x;
                kk[u] = i < n ? key_at(i) : 0ull;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (kk[u] > v) {
                    const uint64_t key = kk[u];
                    const uint64_t sig = (key & ((1ull << 52) - 1)) | (((key >> 52) & 2047u) ? (1ull << 52) : 0ull);
                    const unsigned long long nlo = lo + sig;
                    hi += nlo < lo ? 1ull : 0ull;
                    lo = nlo;
                    ++cgt;
                }
            }
        }
        // exact 128-bit warp / block reduction (integer: order-independent)
        for (int o = 16; o >= 1; o >>= 1) {
            const unsigned long long olo = __shfl_xor_sync(0xffffffffu, lo, o);
            const unsigned long long ohi = __shfl_xor_sync(0xffffffffu, hi, o);
            const unsigned long long nlo = lo + olo;
            hi += ohi + (nlo < lo ? 1ull : 0ull);
            lo = nlo;
            cgt += __shfl_xor_sync(0xffffffffu, cgt, o);
        }
        if (lane == 0) { s_lo[wid] = lo; s_hi[wid] = hi; s_cgt[wid] = cgt; }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long L = 0, H = 0, CG = 0;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
                const unsigned long long nl = L + s_lo[w];
                H += s_hi[w] + (nl < L ? 1ull : 0ull);
                L = nl;
                CG += s_cgt[w];
            }
            const uint32_t ex = (uint32_t)((top >> 12) & 2047u);   // biased exponent of the bin
            const int sc = (ex ? (int)ex : 1) - 1075;               // value = significand * 2^sc
            // (H:L) * 2^sc, H and L each exactly representable when the true sum is
            const double sum_gt = ldexp((double)H, sc + 64) + ldexp((double)L, sc);
            const double vd = __longlong_as_double((long long)v);
            const uint64_t k = P.k[r];
            const uint64_t c_above = P.above_cnt[row * n_rp + r] + CG;
            const double tail = __dadd_rn(__dadd_rn(P.above_sum[row * n_rp + r], sum_gt),
                                          __dmul_rn((double)(k - c_above), vd));
            P.out[((uint64_t)row * n_rp + r) * 2 + 0] = vd;
            P.out[((uint64_t)row * n_rp + r) * 2 + 1] = __ddiv_rn(tail, (double)k);
        }
        __syncthreads();
    }
}

}  // namespace

// scratch: one allocation carved into FParams' arrays
size_t metrics_fast_bytes(uint32_t rows, uint32_t n_rp, uint64_t T, int nblk) {
    const size_t q = (size_t)rows * n_rp;
    return (size_t)rows * kBins * 4 + q * kBins * 4 + q * 8 * 2 + q * 4 + q * 16 + q * 4 + (size_t)rows * T * 8 +
           q * nblk * 16 + q * 16 + (size_t)rows * 3 * 4 + q * 16 + 1024;
}

cudaError_t launch_metrics_fast(const double* d_ylt, uint64_t T, uint64_t ld, uint32_t rows, uint32_t n_rp,
                                const uint64_t* h_k, void* scratch, int nblk, double* d_out, cudaStream_t s) {
    FParams P{};
    P.ylt = d_ylt;
    P.T = T;
    P.ld = ld;
    P.rows = rows;
    P.n_rp = n_rp;
    P.nblk = (uint32_t)nblk;
    for (uint32_t i = 0; i < n_rp; ++i) P.k[i] = h_k[i];
    const size_t q = (size_t)rows * n_rp;
    char* b = static_cast<char*>(scratch);
    auto take = [&](size_t bytes) { char* r = b; b += (bytes + 255) / 256 * 256; return r; };
    // zero-initialised part first (histograms, counters), one memset
    P.hist = reinterpret_cast<uint32_t*>(take((size_t)rows * kBins * 4));
    P.hist2 = reinterpret_cast<uint32_t*>(take(q * kBins * 4));
    P.done = reinterpret_cast<uint32_t*>(take((size_t)rows * 3 * 4));
    const size_t zero_bytes = (size_t)(b - static_cast<char*>(scratch));
    P.pre = reinterpret_cast<uint64_t*>(take(q * 8));
    P.krem = reinterpret_cast<uint64_t*>(take(q * 8));
    P.rep = reinterpret_cast<uint32_t*>(take(q * 4));
    P.seg = reinterpret_cast<uint64_t*>(take(q * 16));
    P.fill = reinterpret_cast<uint32_t*>(take(q * 4));
    P.part_sum = reinterpret_cast<double*>(take(q * nblk * 8));
    P.part_cnt = reinterpret_cast<uint64_t*>(take(q * nblk * 8));
    P.above_sum = reinterpret_cast<double*>(take(q * 8));
    P.above_cnt = reinterpret_cast<uint64_t*>(take(q * 8));
    P.cand = reinterpret_cast<uint64_t*>(take((size_t)rows * T * 8));
    P.out = d_out;
    cudaError_t e = cudaMemsetAsync(scratch, 0, zero_bytes, s);
    if (e != cudaSuccess) return e;
    const dim3 grid((unsigned)nblk, rows);
    fm_pass_a<<<grid, 256, 0, s>>>(P);
    const size_t smem_b = (size_t)(n_rp < kBSmem ? n_rp : kBSmem) * kBins * 4;
    e = cudaFuncSetAttribute(fm_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
    if (e != cudaSuccess) return e;
    fm_pass_b<<<grid, 256, smem_b, s>>>(P);
    fm_pass_c<<<grid, 256, 0, s>>>(P);
    const size_t smem_d = (size_t)kFinSmemKeys * 8;
    e = cudaFuncSetAttribute(fm_pass_d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
    if (e != cudaSuccess) return e;
    fm_pass_d<<<dim3(n_rp, rows), 1024, smem_d, s>>>(P);
    return cudaGetLastError();
}

}  // namespace ara
