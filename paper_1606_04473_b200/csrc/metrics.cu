// metrics.cu — device PML / TVaR over the YLT (§8a row a10).
//
// PAPER.md P:273 names PML and TVaR; readings A9/A10 fix them:
//   k = ceil(T / R);  PML(R) = k-th largest Y;  TVaR(R) = mean of the k largest.
// Method (hand-written, no library sort):
//   1. MSD radix select, 8 passes of 8 bits over the u64 bit patterns of the
//      (non-negative, canonical +0) fp64 YLT values — for non-negative doubles
//      the bit order is the value order.  All return periods of all rows
//      (layers + portfolio) are selected together; return periods whose
//      current prefixes coincide share one histogram.  The last block of each
//      row (threadfence + completion counter) picks the digit, so one launch
//      per pass.
//   2. One pass of masked tail sums with the selected value v:
//      TVaR = (sum_{Y > v} Y + (k - #{Y > v}) v) / k, which equals the mean of
//      the k largest exactly in real arithmetic (ties included); partial sums
//      are combined in a fixed block order, so the result is deterministic.
#include <cooperative_groups.h>
#include <cstdlib>

#include "ara_internal.cuh"

namespace cg = cooperative_groups;

namespace ara {
namespace {

struct MParams {
    const double* ylt;
    uint64_t T, ld;
    uint32_t n_rp, nblk;
    uint32_t* hist;      // [rows][n_rp][256]
    uint64_t* prefix;    // [rows][n_rp]
    uint64_t* krem;      // [rows][n_rp]
    uint32_t* rep;       // [rows][n_rp]
    double* part_sum;    // [rows][n_rp][nblk]
    uint64_t* part_cnt;  // [rows][n_rp][nblk]
    double* out;         // [rows][n_rp][2]
    uint32_t* done;      // [rows]
    double* dsum;        // distributed mode: this rank's tail sums [rows][n_rp] ...
    uint64_t* dcnt;      // ... and counts (all-reduced across ranks, then finished)
    int dist;            // 1: the YLT is this rank's shard; histograms and sums are all-reduced
    uint64_t k[ARA_MAX_RP];
};

__device__ __forceinline__ uint64_t key_of(double y) {
    return (uint64_t)__double_as_longlong(y + 0.0);   // canonical +0 (A16)
}

__global__ void init_kernel(const __grid_constant__ MParams P) {
    const uint32_t row = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < P.n_rp; i += blockDim.x) {
        P.prefix[row * P.n_rp + i] = 0;
        P.krem[row * P.n_rp + i] = P.k[i];
        P.rep[row * P.n_rp + i] = 0;   // all prefixes equal: share slot 0
    }
    for (uint32_t i = threadIdx.x; i < P.n_rp * 256u; i += blockDim.x) P.hist[(uint64_t)row * P.n_rp * 256 + i] = 0;
    if (threadIdx.x == 0) P.done[row] = 0;
}

// Pick the digit of every return period of `row` from the row's (complete)
// global histograms: stage them in shared memory, one warp per return period
// scans from the top digit down; update prefix / remaining rank / reps and
// clear the histograms.  (The last block of a pass, or select_kernel.)
__device__ void select_row(const MParams& P, uint32_t row, int shift, uint32_t* sh, uint64_t* s_prefix) {
    const uint32_t n_rp = P.n_rp;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t* gh = P.hist + (uint64_t)row * n_rp * 256;
    __shared__ uint32_t s_rep2[ARA_MAX_RP];
    for (uint32_t i = threadIdx.x; i < n_rp; i += blockDim.x) s_rep2[i] = P.rep[row * n_rp + i];
    __syncthreads();
    const uint32_t* s_rep = s_rep2;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x) sh[i] = (s_rep[i >> 8] == (i >> 8)) ? __ldcg(gh + i) : 0u;
    __syncthreads();
    const uint32_t wid = threadIdx.x >> 5;
    for (uint32_t r = wid; r < n_rp; r += blockDim.x >> 5) {
        const uint32_t* h = sh + s_rep[r] * 256;
        const uint64_t kr = P.krem[row * n_rp + r];
        // lane l owns digits 255-8l .. 248-8l (descending)
        uint32_t c[8];
        uint64_t tot = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { c[q] = h[255 - 8 * lane - q]; tot += c[q]; }
        uint64_t incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (uint32_t)o) incl += v;
        }
        const uint64_t excl = incl - tot;
        const unsigned hit = __ballot_sync(0xffffffffu, excl < kr && kr <= incl);
        const uint32_t src = (uint32_t)(__ffs(hit) - 1);
        if (lane == src) {
            uint64_t cum = excl;
            uint32_t d = 255 - 8 * lane;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (kr <= cum + c[q]) { d = 255 - 8 * lane - q; break; }
                cum += c[q];
            }
            const uint64_t pre = s_prefix[r] | ((uint64_t)d << shift);
            P.prefix[row * n_rp + r] = pre;
            P.krem[row * n_rp + r] = kr - cum;
            s_prefix[r] = pre;
        }
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < n_rp; r += blockDim.x) {
        uint32_t rr = r;
        for (uint32_t q = 0; q < r; ++q)
            if (s_prefix[q] == s_prefix[r]) { rr = q; break; }
        P.rep[row * n_rp + r] = rr;
    }
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x) gh[i] = 0;
}

__global__ void __launch_bounds__(256) radix_pass_kernel(const __grid_constant__ MParams P, int pass) {
    extern __shared__ uint32_t sh[];                      // [n_rp][256]
    __shared__ uint64_t s_prefix[ARA_MAX_RP];
    __shared__ uint32_t s_rep[ARA_MAX_RP];
    __shared__ uint32_t s_last;
    const uint32_t row = blockIdx.y, n_rp = P.n_rp;
    const uint32_t lane = threadIdx.x & 31u;
    const int shift = 56 - 8 * pass;
    for (uint32_t i = threadIdx.x; i < n_rp; i += blockDim.x) {
        s_prefix[i] = P.prefix[row * n_rp + i];
        s_rep[i] = P.rep[row * n_rp + i];
    }
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x) sh[i] = 0;
    __syncthreads();

    // Warp-uniform sweep.  Distinct current prefixes ("reps") are disjoint, so
    // a key belongs to at most one rep; lanes with the same (rep, digit) are
    // merged with match_any so each pair costs one shared atomic per warp
    // (YLT keys concentrate in a few top-byte bins).
    __shared__ uint32_t s_ulist[ARA_MAX_RP];
    __shared__ uint64_t s_upre[ARA_MAX_RP];
    __shared__ uint32_t s_nu;
    if (threadIdx.x == 0) {
        uint32_t nu = 0;
        for (uint32_t r = 0; r < n_rp; ++r)
            if (s_rep[r] == r) { s_ulist[nu] = r; s_upre[nu] = s_prefix[r]; ++nu; }
        s_nu = nu;
    }
    __syncthreads();
    const uint32_t nu = s_nu;
    const double* y = P.ylt + (uint64_t)row * P.ld;
    // Keys are loaded KB at a time per lane (independent loads in flight),
    // then binned.
    constexpr int KB = 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < P.T; i0 += stride * KB) {
        uint64_t keys[KB];
#pragma unroll
        for (int q = 0; q < KB; ++q) {
            const uint64_t i = i0 + q * stride + lane;
            keys[q] = i < P.T ? key_of(__ldcg(y + i)) : ~0ull;   // ~0: not a key (NaN pattern)
        }
#pragma unroll
        for (int q = 0; q < KB; ++q) {
            if (i0 + q * stride >= P.T) break;   // warp-uniform
            const uint64_t key = keys[q];
            const bool valid = key != ~0ull;
            const uint32_t d = (uint32_t)(key >> shift) & 255u;
            uint32_t which = 0xffffffffu;
            if (valid) {
                if (pass == 0) which = 0;
                else
                    for (uint32_t u = 0; u < nu; ++u)
                        if (((key ^ s_upre[u]) >> (shift + 8)) == 0) which = u;
            }
            const uint32_t tag = which == 0xffffffffu ? 0xffffffffu : (which << 8) | d;
            const unsigned peers = __match_any_sync(0xffffffffu, tag);
            if (tag != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1))
                atomicAdd(&sh[s_ulist[which] * 256 + d], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    uint32_t* gh = P.hist + (uint64_t)row * n_rp * 256;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
    if (P.dist) return;   // the histograms are all-reduced across ranks, then select_kernel
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&P.done[row], 1u) == P.nblk - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    select_row(P, row, shift, sh, s_prefix);
    if (threadIdx.x == 0) P.done[row] = 0;
}

// distributed mode: one block per row picks the digits from the all-reduced histograms
__global__ void __launch_bounds__(256) select_kernel(const __grid_constant__ MParams P, int pass) {
    extern __shared__ uint32_t sh[];
    __shared__ uint64_t s_prefix[ARA_MAX_RP];
    const uint32_t row = blockIdx.x;
    for (uint32_t i = threadIdx.x; i < P.n_rp; i += blockDim.x) s_prefix[i] = P.prefix[row * P.n_rp + i];
    __syncthreads();
    select_row(P, row, 56 - 8 * pass, sh, s_prefix);
}

// distributed mode: TVaR from the all-reduced tail sums and counts
__global__ void finish_kernel(const __grid_constant__ MParams P, uint32_t rows) {
    for (uint32_t q = threadIdx.x; q < rows * P.n_rp; q += blockDim.x) {
        const double v = __longlong_as_double((long long)P.prefix[q]);
        const uint64_t k = P.k[q % P.n_rp];
        const double tail = __dadd_rn(P.dsum[q], __dmul_rn((double)(k - P.dcnt[q]), v));
        P.out[(uint64_t)q * 2 + 0] = v;
        P.out[(uint64_t)q * 2 + 1] = __ddiv_rn(tail, (double)k);
    }
}

__global__ void __launch_bounds__(256) tail_kernel(const __grid_constant__ MParams P) {
    // RC return periods per sweep over the row (each accumulator is the same
    // per-thread sequential sum over the same keys as a one-period sweep).
    // RC = 10 covers the paper's 10 return periods in one sweep (40 KB of
    // static shared memory for the block reductions).
    constexpr int RC = 10;
    __shared__ double s_sum[RC][256];
    __shared__ uint64_t s_cnt[RC][256];
    __shared__ uint32_t s_last;
    const uint32_t row = blockIdx.y, n_rp = P.n_rp;
    const double* y = P.ylt + (uint64_t)row * P.ld;
    constexpr int KB = 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint32_t r0 = 0; r0 < n_rp; r0 += RC) {
        double v[RC], s[RC];
        uint64_t c[RC];
#pragma unroll
        for (int j = 0; j < RC; ++j) {
            // periods past n_rp compare against +inf: nothing is added
            v[j] = r0 + j < n_rp ? __longlong_as_double((long long)P.prefix[row * n_rp + r0 + j]) : INFINITY;
            s[j] = 0.0;
            c[j] = 0;
        }
        for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < P.T; i0 += stride * KB) {
            double xs[KB];
#pragma unroll
            for (int q = 0; q < KB; ++q) {
                const uint64_t i = i0 + q * stride;
                xs[q] = i < P.T ? __ldcg(y + i) + 0.0 : -1.0;
            }
#pragma unroll
            for (int q = 0; q < KB; ++q)   // fixed order per thread: deterministic
#pragma unroll
                for (int j = 0; j < RC; ++j)
                    if (xs[q] > v[j]) { s[j] = __dadd_rn(s[j], xs[q]); ++c[j]; }
        }
#pragma unroll
        for (int j = 0; j < RC; ++j) {
            s_sum[j][threadIdx.x] = s[j];
            s_cnt[j][threadIdx.x] = c[j];
        }
        __syncthreads();
        for (int w = 128; w >= 1; w >>= 1) {
            if ((int)threadIdx.x < w) {
#pragma unroll
                for (int j = 0; j < RC; ++j) {
                    s_sum[j][threadIdx.x] = __dadd_rn(s_sum[j][threadIdx.x], s_sum[j][threadIdx.x + w]);
                    s_cnt[j][threadIdx.x] += s_cnt[j][threadIdx.x + w];
                }
            }
            __syncthreads();
        }
        if (threadIdx.x < RC && r0 + threadIdx.x < n_rp) {
            const uint32_t r = r0 + threadIdx.x;
            P.part_sum[((uint64_t)row * n_rp + r) * P.nblk + blockIdx.x] = s_sum[threadIdx.x][0];
            P.part_cnt[((uint64_t)row * n_rp + r) * P.nblk + blockIdx.x] = s_cnt[threadIdx.x][0];
        }
        __syncthreads();
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&P.done[row], 1u) == P.nblk - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // Combine the per-block partials in block order (deterministic): one warp
    // per return period, partials staged through registers in fixed chunks.
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    for (uint32_t r = wid; r < n_rp; r += blockDim.x >> 5) {
        const double v = __longlong_as_double((long long)P.prefix[row * n_rp + r]);
        const double* ps = P.part_sum + ((uint64_t)row * n_rp + r) * P.nblk;
        const uint64_t* pc = P.part_cnt + ((uint64_t)row * n_rp + r) * P.nblk;
        double s = 0.0;
        uint64_t c = 0;
        for (uint32_t b0 = 0; b0 < P.nblk; b0 += 32) {
            const uint32_t b = b0 + lane;
            const double x = b < P.nblk ? __ldcg(ps + b) : 0.0;
            const uint64_t y = b < P.nblk ? __ldcg(pc + b) : 0ull;
            for (uint32_t q = 0; q < 32 && b0 + q < P.nblk; ++q) {   // sequential, block order
                s = __dadd_rn(s, __shfl_sync(0xffffffffu, x, q));
                c += __shfl_sync(0xffffffffu, y, q);
            }
        }
        if (lane == 0) {
            if (P.dist) {   // this rank's share; finish_kernel completes it after the all-reduce
                P.dsum[(uint64_t)row * n_rp + r] = s;
                P.dcnt[(uint64_t)row * n_rp + r] = c;
            } else {
                const uint64_t k = P.k[r];
                const double tail = __dadd_rn(s, __dmul_rn((double)(k - c), v));
                P.out[((uint64_t)row * n_rp + r) * 2 + 0] = v;
                P.out[((uint64_t)row * n_rp + r) * 2 + 1] = __ddiv_rn(tail, (double)k);
            }
        }
    }
    if (threadIdx.x == 0) P.done[row] = 0;
}

// ---------------------------------------------------------------------------
// The same method in ONE cooperative launch (the default when the grid fits):
// the 8 radix passes and the tail sums are separated by grid-wide barriers
// instead of kernel boundaries and "last block" hand-offs.  Every block keeps
// the per-(row, return period) prefixes in shared memory and selects the digit
// itself from the global histogram after each barrier (identical inputs,
// identical choices), so a pass costs one sweep + one barrier.  Global
// histograms rotate over three buffers: the one a pass accumulates into was
// zeroed two barriers earlier, after every block had finished reading it.
struct CoopLayout {
    uint32_t nq;          // rows * n_rp
    size_t hist_off, pre_off, krem_off, up_off, rep_off, uq_off, nu_off, bytes;
};
__host__ __device__ inline CoopLayout coop_layout(uint32_t rows, uint32_t n_rp) {
    CoopLayout L;
    L.nq = rows * n_rp;
    L.hist_off = 0;
    L.pre_off = (size_t)L.nq * 256 * 4;
    L.krem_off = L.pre_off + (size_t)L.nq * 8;
    L.up_off = L.krem_off + (size_t)L.nq * 8;     // per row: its distinct prefixes ...
    L.rep_off = L.up_off + (size_t)L.nq * 8;
    L.uq_off = L.rep_off + (size_t)L.nq * 4;      // ... and their slots
    L.nu_off = L.uq_off + (size_t)L.nq * 4;       // number of distinct prefixes per row
    L.bytes = L.nu_off + (size_t)rows * 4;
    return L;
}

__global__ void __launch_bounds__(256) metrics_coop_kernel(const __grid_constant__ MParams P, uint32_t rows,
                                                           uint32_t* __restrict__ ghist /*[3][nq][256]*/) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char dsm[];
    const uint32_t n_rp = P.n_rp;
    const CoopLayout Lo = coop_layout(rows, n_rp);
    const uint32_t nq = Lo.nq;
    uint32_t* sh = reinterpret_cast<uint32_t*>(dsm + Lo.hist_off);
    uint64_t* s_prefix = reinterpret_cast<uint64_t*>(dsm + Lo.pre_off);
    uint64_t* s_krem = reinterpret_cast<uint64_t*>(dsm + Lo.krem_off);
    uint32_t* s_rep = reinterpret_cast<uint32_t*>(dsm + Lo.rep_off);
    uint64_t* s_up = reinterpret_cast<uint64_t*>(dsm + Lo.up_off);
    uint32_t* s_uq = reinterpret_cast<uint32_t*>(dsm + Lo.uq_off);
    uint32_t* s_nu = reinterpret_cast<uint32_t*>(dsm + Lo.nu_off);
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {
        s_prefix[q] = 0;
        s_krem[q] = P.k[q % n_rp];
        s_rep[q] = q - q % n_rp;   // all prefixes of a row equal: share the row's first slot
        s_uq[q] = q - q % n_rp;
        s_up[q] = 0;
    }
    for (uint32_t row = threadIdx.x; row < rows; row += blockDim.x) s_nu[row] = 1;
    // this block's key range (the same for every row), staged once in shared
    // memory as sort keys: the 8 passes and the tail sums read it from there
    const uint64_t per = (P.T + gridDim.x - 1) / gridDim.x;
    const uint64_t i_lo = (uint64_t)blockIdx.x * per;
    const uint64_t i_hi = i_lo + per < P.T ? i_lo + per : P.T;
    const uint32_t nk = i_hi > i_lo ? (uint32_t)(i_hi - i_lo) : 0u;
    uint64_t* s_key = reinterpret_cast<uint64_t*>(dsm + Lo.bytes);   // [rows][per]
    for (uint32_t row = 0; row < rows; ++row) {
        const double* y = P.ylt + (uint64_t)row * P.ld + i_lo;
        for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) s_key[(uint64_t)row * per + i] = key_of(__ldcg(y + i));
    }
    __syncthreads();

    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        uint32_t* gh = ghist + (size_t)(pass % 3) * nq * 256;
        for (uint32_t i = threadIdx.x; i < nq * 256u; i += blockDim.x) sh[i] = 0;
        __syncthreads();
        for (uint32_t row = 0; row < rows; ++row) {
            const double* y = P.ylt + (uint64_t)row * P.ld;
            const uint32_t q0 = row * n_rp;
            // the row's distinct current prefixes (disjoint: a key extends at most one)
            const uint32_t nu = s_nu[row];
            const uint64_t* up = s_up + q0;
            const uint32_t* uq = s_uq + q0;
            // per-lane cache of the last (slot, digit) tag this lane added for:
            // YLT keys concentrate in a few bins, so most adds stay in a register
            uint32_t ctag = 0xffffffffu, ccnt = 0;
            const uint64_t* kr = s_key + (uint64_t)row * per;
            for (uint32_t i0 = threadIdx.x & ~31u; i0 < nk; i0 += blockDim.x) {   // warp-uniform trip count
                const uint32_t i = i0 + lane;
                const uint64_t key = i < nk ? kr[i] : ~0ull;
                uint32_t which = 0xffffffffu;
                if (key != ~0ull) {
                    if (pass == 0) which = q0;
                    else
                        for (uint32_t u = 0; u < nu; ++u)
                            if (((key ^ up[u]) >> (shift + 8)) == 0) { which = uq[u]; break; }
                }
                const uint32_t tag = which == 0xffffffffu ? 0xffffffffu : (which << 8) | ((uint32_t)(key >> shift) & 255u);
                const unsigned peers = __match_any_sync(0xffffffffu, tag);
                if (tag != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1)) {
                    if (tag != ctag) {
                        if (ccnt) atomicAdd(&sh[(ctag >> 8) * 256 + (ctag & 255u)], ccnt);
                        ctag = tag;
                        ccnt = 0;
                    }
                    ccnt += (uint32_t)__popc(peers);
                }
            }
            if (ccnt) atomicAdd(&sh[(ctag >> 8) * 256 + (ctag & 255u)], ccnt);
        }
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < nq * 256u; i += blockDim.x)
            if (sh[i]) atomicAdd(&gh[i], sh[i]);
        grid.sync();
        // every block: pick the digit of every (row, return period) from the global histogram
        for (uint32_t q = wid; q < nq; q += blockDim.x >> 5) {
            const uint32_t* h = gh + (size_t)s_rep[q] * 256;
            const uint64_t kr = s_krem[q];
            uint32_t c[8];
            uint64_t tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = __ldcg(h + 255 - 8 * lane - j); tot += c[j]; }
            uint64_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= (uint32_t)o) incl += v;
            }
            const uint64_t excl = incl - tot;
            const unsigned hit = __ballot_sync(0xffffffffu, excl < kr && kr <= incl);
            const uint32_t src = (uint32_t)(__ffs(hit) - 1);
            uint64_t pre = 0, krn = 0;
            if (lane == src) {
                uint64_t cum = excl;
                uint32_t dd = 255 - 8 * lane;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (kr <= cum + c[j]) { dd = 255 - 8 * lane - j; break; }
                    cum += c[j];
                }
                pre = s_prefix[q] | ((uint64_t)dd << shift);
                krn = kr - cum;
            }
            pre = __shfl_sync(0xffffffffu, pre, src);
            krn = __shfl_sync(0xffffffffu, krn, src);
            __syncwarp();
            if (lane == 0) { s_prefix[q] = pre; s_krem[q] = krn; }
        }
        // the buffer pass + 2 will use was last read before this barrier: clear it
        if (blockIdx.x == 0) {
            uint32_t* gz = ghist + (size_t)((pass + 2) % 3) * nq * 256;
            for (uint32_t i = threadIdx.x; i < nq * 256u; i += blockDim.x) gz[i] = 0;
        }
        __syncthreads();
        for (uint32_t q = threadIdx.x; q < nq; q += blockDim.x) {   // dedupe equal prefixes per row
            const uint32_t q0 = q - q % n_rp;
            uint32_t rr = q;
            for (uint32_t j = q0; j < q; ++j)
                if (s_prefix[j] == s_prefix[q]) { rr = j; break; }
            s_rep[q] = rr;
        }
        __syncthreads();
        for (uint32_t row = threadIdx.x; row < rows; row += blockDim.x) {   // per-row list of distinct prefixes
            uint32_t nu = 0;
            for (uint32_t q = row * n_rp; q < (row + 1) * n_rp; ++q)
                if (s_rep[q] == q) { s_uq[row * n_rp + nu] = q; s_up[row * n_rp + nu] = s_prefix[q]; ++nu; }
            s_nu[row] = nu;
        }
        __syncthreads();
    }

    // tail sums over this block's keys, then block 0 combines in block order
    __shared__ double s_sum[256];
    __shared__ uint64_t s_cnt[256];
    for (uint32_t q = 0; q < nq; ++q) {
        const uint32_t row = q / n_rp;
        const uint64_t* kr = s_key + (uint64_t)row * per;
        const uint64_t vk = s_prefix[q];
        double sm = 0.0;
        uint64_t c = 0;
        for (uint32_t i = threadIdx.x; i < nk; i += blockDim.x) {   // fixed order: deterministic
            const uint64_t key = kr[i];   // key order = value order (non-negative doubles)
            if (key > vk) { sm = __dadd_rn(sm, __longlong_as_double((long long)key)); ++c; }
        }
        s_sum[threadIdx.x] = sm;
        s_cnt[threadIdx.x] = c;
        __syncthreads();
        for (int w = 128; w >= 1; w >>= 1) {
            if ((int)threadIdx.x < w) {
                s_sum[threadIdx.x] = __dadd_rn(s_sum[threadIdx.x], s_sum[threadIdx.x + w]);
                s_cnt[threadIdx.x] += s_cnt[threadIdx.x + w];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            P.part_sum[(uint64_t)q * gridDim.x + blockIdx.x] = s_sum[0];
            P.part_cnt[(uint64_t)q * gridDim.x + blockIdx.x] = s_cnt[0];
        }
        __syncthreads();
    }
    grid.sync();
    if (blockIdx.x != 0) return;
    for (uint32_t q = wid; q < nq; q += blockDim.x >> 5) {
        const double v = __longlong_as_double((long long)s_prefix[q]);
        const double* ps = P.part_sum + (uint64_t)q * gridDim.x;
        const uint64_t* pc = P.part_cnt + (uint64_t)q * gridDim.x;
        double sm = 0.0;
        uint64_t c = 0;
        for (uint32_t b0 = 0; b0 < gridDim.x; b0 += 32) {
            const uint32_t b = b0 + lane;
            const double x = b < gridDim.x ? __ldcg(ps + b) : 0.0;
            const uint64_t yy = b < gridDim.x ? __ldcg(pc + b) : 0ull;
            for (uint32_t j = 0; j < 32 && b0 + j < gridDim.x; ++j) {   // sequential, block order
                sm = __dadd_rn(sm, __shfl_sync(0xffffffffu, x, j));
                c += __shfl_sync(0xffffffffu, yy, j);
            }
        }
        if (lane == 0) {
            const uint64_t k = P.k[q % n_rp];
            const double tail = __dadd_rn(sm, __dmul_rn((double)(k - c), v));
            P.out[(uint64_t)q * 2 + 0] = v;
            P.out[(uint64_t)q * 2 + 1] = __ddiv_rn(tail, (double)k);
        }
    }
}

}  // namespace

cudaError_t launch_metrics_dist(const double* d_ylt, uint64_t T_local, uint64_t ld, uint32_t rows, uint32_t n_rp,
                                const uint64_t* h_k, MetricsScratch& m, int nblk, ncclComm_t comm,
                                cudaStream_t s, int* nccl_err) {
    MParams P{};
    P.ylt = d_ylt;
    P.T = T_local;
    P.ld = ld;
    P.n_rp = n_rp;
    P.nblk = (uint32_t)nblk;
    P.hist = m.hist;
    P.prefix = m.prefix;
    P.krem = m.krem;
    P.part_sum = m.part_sum;
    P.part_cnt = m.part_cnt;
    P.out = m.out;
    P.done = m.done;
    P.rep = m.done + rows;
    P.dsum = m.dsum;
    P.dcnt = m.dcnt;
    P.dist = 1;
    for (uint32_t i = 0; i < n_rp; ++i) P.k[i] = h_k[i];
    const size_t smem = (size_t)n_rp * 256 * sizeof(uint32_t);
    if (smem > 32 * 1024) {   // leaves room for the kernels' static shared memory under the 48 KB default
        cudaError_t e = cudaFuncSetAttribute(radix_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    *nccl_err = 0;
    init_kernel<<<rows, 256, 0, s>>>(P);
    const size_t nh = (size_t)rows * n_rp * 256;
    for (int pass = 0; pass < 8; ++pass) {
        radix_pass_kernel<<<dim3(P.nblk, rows), 256, smem, s>>>(P, pass);
        // comm == null: a single shard (world 1, ARA_METRICS_DIST / loopback): the reduce is the identity
        if (comm && ncclAllReduce(P.hist, P.hist, nh, ncclUint32, ncclSum, comm, s) != ncclSuccess) { *nccl_err = 1; break; }
        select_kernel<<<rows, 256, smem, s>>>(P, pass);
    }
    if (*nccl_err) return cudaGetLastError();
    tail_kernel<<<dim3(P.nblk, rows), 256, 0, s>>>(P);
    const size_t nq = (size_t)rows * n_rp;
    if (comm && (ncclGroupStart() != ncclSuccess || ncclAllReduce(P.dsum, P.dsum, nq, ncclDouble, ncclSum, comm, s) != ncclSuccess ||
        ncclAllReduce(P.dcnt, P.dcnt, nq, ncclUint64, ncclSum, comm, s) != ncclSuccess || ncclGroupEnd() != ncclSuccess)) {
        *nccl_err = 1;
        return cudaGetLastError();
    }
    finish_kernel<<<1, 256, 0, s>>>(P, rows);
    return cudaGetLastError();
}

cudaError_t metrics_alloc(MetricsScratch& m, uint32_t rows, uint32_t n_rp, int nblk) {
    const size_t need = (size_t)rows * n_rp;
    if (m.cap_rows_rp >= need && m.nblk >= nblk && m.cap_rows >= rows) return cudaSuccess;
    metrics_free(m);
    const size_t rr = need;
    cudaError_t e;
    if ((e = cudaMalloc(&m.hist, rr * 256 * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.prefix, rr * sizeof(uint64_t) * 2 + rr * sizeof(uint32_t))) != cudaSuccess) return e;
    m.krem = m.prefix + rr;
    if ((e = cudaMalloc(&m.part_sum, rr * nblk * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.part_cnt, rr * nblk * sizeof(uint64_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.out, rr * 2 * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.done, rows * sizeof(uint32_t) + rr * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.coop_hist, 3 * rr * 256 * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.dsum, rr * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.dcnt, rr * sizeof(uint64_t))) != cudaSuccess) return e;
    m.cap_rows_rp = need;
    m.cap_rows = rows;
    m.nblk = nblk;
    return cudaSuccess;
}

void metrics_free(MetricsScratch& m) {
    cudaFree(m.hist);
    cudaFree(m.prefix);
    cudaFree(m.part_sum);
    cudaFree(m.part_cnt);
    cudaFree(m.out);
    cudaFree(m.done);
    cudaFree(m.coop_hist);
    cudaFree(m.dsum);
    cudaFree(m.dcnt);
    m = MetricsScratch{};
}

cudaError_t launch_metrics(const double* d_ylt, uint64_t T, uint64_t ld, uint32_t rows,
                           uint32_t n_rp, const uint64_t* h_k, MetricsScratch& m, int nblk, cudaStream_t s) {
    MParams P{};
    P.ylt = d_ylt;
    P.T = T;
    P.ld = ld;
    P.n_rp = n_rp;
    P.nblk = (uint32_t)nblk;
    P.hist = m.hist;
    P.prefix = m.prefix;
    P.krem = m.krem;
    P.part_sum = m.part_sum;
    P.part_cnt = m.part_cnt;
    P.out = m.out;
    P.done = m.done;
    P.rep = m.done + rows;
    for (uint32_t i = 0; i < n_rp; ++i) P.k[i] = h_k[i];
    const size_t smem = (size_t)n_rp * 256 * sizeof(uint32_t);
    if (smem > 32 * 1024) {   // leaves room for the kernels' static shared memory under the 48 KB default
        cudaError_t e = cudaFuncSetAttribute(radix_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    // One cooperative launch (ARA_METRICS_COOP=1, when the per-block state
    // fits in shared memory); otherwise 10 plain launches (default).
    const CoopLayout Lo = coop_layout(rows, n_rp);
    static int coop_ok = -1, n_sm = 0, per_sm = 0;
    if (coop_ok < 0) {   // measured slower than the multi-launch path on B200 (0.34 vs 0.23 ms at
                         // 2 x 1M keys): opt-in with ARA_METRICS_COOP=1 for A/B runs
        int dev = 0, attr = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&attr, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        coop_ok = attr ? 1 : 0;
    }
    const char* coop_env = getenv("ARA_METRICS_COOP");
    const bool coop_on = coop_ok && coop_env && atoi(coop_env) != 0;
    // Grid: two blocks per SM; each block stages rows x ceil(T / grid) keys.
    int grid = 2 * n_sm;
    if (grid > m.nblk) grid = m.nblk;   // partial-sum capacity
    const uint64_t want = (T + 255) / 256;
    if ((uint64_t)grid > want) grid = (int)want;
    const uint64_t per = grid > 0 ? (T + grid - 1) / grid : 0;
    const size_t cbytes = Lo.bytes + (size_t)rows * per * sizeof(uint64_t);
    if (coop_on && grid >= 1 && cbytes <= 110 * 1024 && m.coop_hist && (size_t)rows * n_rp <= m.cap_rows_rp) {
        cudaFuncSetAttribute(metrics_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cbytes);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, metrics_coop_kernel, 256, cbytes) != cudaSuccess)
            per_sm = 0;
        cudaGetLastError();
        if ((int64_t)per_sm * n_sm >= grid) {
            cudaError_t e = cudaMemsetAsync(m.coop_hist, 0, (size_t)3 * Lo.nq * 256 * sizeof(uint32_t), s);
            if (e != cudaSuccess) return e;
            uint32_t* gh = m.coop_hist;
            void* args[] = {(void*)&P, (void*)&rows, (void*)&gh};
            e = cudaLaunchCooperativeKernel((void*)metrics_coop_kernel, dim3(grid), dim3(256), args, cbytes, s);
            if (e == cudaSuccess) return cudaSuccess;
            cudaGetLastError();   // fall through to the multi-launch path
        }
    }
    init_kernel<<<rows, 256, 0, s>>>(P);
    for (int pass = 0; pass < 8; ++pass)
        radix_pass_kernel<<<dim3(P.nblk, rows), 256, smem, s>>>(P, pass);
    tail_kernel<<<dim3(P.nblk, rows), 256, 0, s>>>(P);
    return cudaGetLastError();
}

}  // namespace ara
