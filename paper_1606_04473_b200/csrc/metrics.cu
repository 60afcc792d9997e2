// metrics.cu — device PML / TVaR over the YLT (§8a row a10).
//
// PAPER.md P:273 names PML and TVaR; readings A9/A10 fix them:
//   k = ceil(T / R);  PML(R) = k-th largest Y;  TVaR(R) = mean of the k largest.
// Method (hand-written, no library sort): an MSD radix select over the u64
// bit patterns of the (non-negative, canonical +0) fp64 YLT values — for
// non-negative doubles the bit order is the value order — with all return
// periods of all rows (layers + portfolio) selected together (periods whose
// current prefixes coincide share one histogram), then
//   TVaR = (sum_{Y > v} Y + (k - #{Y > v}) v) / k,
// which equals the mean of the k largest exactly in real arithmetic (ties
// included).  Every sum is taken in a fixed order, so results are
// deterministic.  Two launch sequences (below): the fast path (n_rp <= 11:
// three full sweeps, then only the candidates that share the 16-bit prefix of
// a selected value) and the general one (8 full sweeps + tail), both also in a
// distributed form whose histograms and sums are all-reduced between launches.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ara_internal.cuh"

namespace ara {
namespace {

__device__ __forceinline__ uint64_t key_of(double y) {
    return (uint64_t)__double_as_longlong(y + 0.0);   // canonical +0 (A16)
}

// lane l's 8 histogram words 248-8l .. 255-8l as two 16-B loads (coalesced; every
// block reads the same global histogram right after a pass, so sector count matters)
__device__ __forceinline__ void hist_words(const uint32_t* h, uint32_t lane, uint32_t (&w)[8]) {
    const uint4 a = __ldcg(reinterpret_cast<const uint4*>(h + 248 - 8 * lane));
    const uint4 b = __ldcg(reinterpret_cast<const uint4*>(h + 252 - 8 * lane));
    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w; w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
}

// ---------------------------------------------------------------------------
// Default path (round 2): the same MSD radix select and tail sums, organised
// for throughput instead of latency chains.
//  * No "last block" hand-off between passes: every block of pass p first
//    derives the digits of pass p-1 itself from the (complete) global
//    histogram of pass p-1 — identical inputs, identical choices — and block 0
//    of each row records the state for the next pass (double-buffered).
//  * No warp-synchronous match_any per key: each thread keeps its last
//    (prefix slot, digit) bin and its count in registers (YLT keys fall into a
//    few bins), flushing to the block's shared histogram only when the bin
//    changes.
//  * Consecutive launches use programmatic dependent launch: pass p+1's blocks
//    are resident and waiting (griddepcontrol.wait) when pass p ends.
//  * Tail sums: per-thread fixed-order sums, fixed shuffle trees within a warp
//    and across warps, block partials combined in block order by a fixed
//    per-lane split + shuffle tree: deterministic for a given device and size.
// Histogram zeroing: pass 0 clears the buffers of passes 1..7, the tail kernel
// clears pass 0's buffer for the next call (metrics_alloc zeroes all of them
// once).
#ifndef M3_THREADS_V
#define M3_THREADS_V 512
#endif
#ifndef M3_KB_V
#define M3_KB_V 16
#endif
constexpr int M3_THREADS = M3_THREADS_V;
constexpr int M3_KB = M3_KB_V;
constexpr int M3_RC = 10;

struct M3Params {
    const double* ylt;
    uint64_t T, ld;
    uint32_t n_rp, nblk, rows;
    uint32_t* hist;      // [8][rows][n_rp][256]
    uint64_t* st;        // [2][rows][n_rp][2]: prefix, remaining rank
    uint32_t* strep;     // [2][rows][n_rp]: histogram slot (first period with the same prefix)
    double* part_sum;    // [rows][n_rp][nblk]
    uint64_t* part_cnt;
    uint32_t* done;      // [rows]
    double* out;         // [rows][n_rp][2]
    double* dsum;        // distributed: this rank's tail sums / counts
    uint64_t* dcnt;
    int dist;
    uint64_t k[ARA_MAX_RP];
};

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

struct M3Smem {   // per block, for its row
    uint64_t pre[ARA_MAX_RP];
    uint64_t krem[ARA_MAX_RP];
    uint32_t rep[ARA_MAX_RP];
    uint64_t up[ARA_MAX_RP];   // distinct current prefixes ...
    uint32_t uq[ARA_MAX_RP];   // ... and their slots
    uint32_t nu;
};

// S_p into shared memory: p == 0 the initial state, else the state recorded in st[p & 1].
__device__ void m3_load(const M3Params& P, uint32_t row, int p, M3Smem& S) {
    const uint32_t n_rp = P.n_rp;
    const size_t q0 = (size_t)row * n_rp;
    for (uint32_t r = threadIdx.x; r < n_rp; r += blockDim.x) {
        if (p == 0) { S.pre[r] = 0; S.krem[r] = P.k[r]; S.rep[r] = 0; }
        else {
            const size_t b = (size_t)(p & 1) * P.rows * n_rp + q0 + r;
            S.pre[r] = __ldcg(P.st + 2 * b);
            S.krem[r] = __ldcg(P.st + 2 * b + 1);
            S.rep[r] = __ldcg(P.strep + b);
        }
    }
    __syncthreads();
}

// the distinct prefixes (up) and their histogram slots (uq)
__device__ void m3_ulist(const M3Params& P, M3Smem& S) {
    if (threadIdx.x == 0) {
        uint32_t nu = 0;
        for (uint32_t r = 0; r < P.n_rp; ++r)
            if (S.rep[r] == r) { S.up[nu] = S.pre[r]; S.uq[nu] = r; ++nu; }
        S.nu = nu;
    }
    __syncthreads();
}

// S_{p+1} from S_p (in shared memory) and the complete histogram of pass p
// (row-local); record it in st[(p + 1) & 1] when `record`.
__device__ void m3_select(const M3Params& P, uint32_t row, int p, M3Smem& S, bool record) {
    const uint32_t n_rp = P.n_rp, lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    const size_t q0 = (size_t)row * n_rp;
    const int shift = 56 - 8 * p;
    const uint32_t* gh = P.hist + ((size_t)p * P.rows * n_rp + q0) * 256;
    for (uint32_t r = wid; r < n_rp; r += blockDim.x >> 5) {
        const uint32_t* h = gh + (size_t)S.rep[r] * 256;
        const uint64_t kr = S.krem[r];
        uint32_t c[8];
        uint64_t tot = 0;
        uint32_t hw[8];
        hist_words(h, lane, hw);
#pragma unroll
        for (int j = 0; j < 8; ++j) { c[j] = hw[7 - j]; tot += c[j]; }
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
            for (int j = 0; j < 8; ++j) {
                if (kr <= cum + c[j]) { d = 255 - 8 * lane - j; break; }
                cum += c[j];
            }
            S.pre[r] |= (uint64_t)d << shift;
            S.krem[r] = kr - cum;
        }
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < n_rp; r += blockDim.x) {
        uint32_t rr = r;
        for (uint32_t q = 0; q < r; ++q)
            if (S.pre[q] == S.pre[r]) { rr = q; break; }
        S.rep[r] = rr;
    }
    __syncthreads();
    m3_ulist(P, S);
    if (record) {
        for (uint32_t r = threadIdx.x; r < n_rp; r += blockDim.x) {
            const size_t b = (size_t)((p + 1) & 1) * P.rows * n_rp + q0 + r;
            P.st[2 * b] = S.pre[r];
            P.st[2 * b + 1] = S.krem[r];
            P.strep[b] = S.rep[r];
        }
    }
    __syncthreads();
}

// S_{p+1} from the recorded S_p and the complete histogram of pass p; block 0
// records it (p < 7) for the next pass.
__device__ void m3_advance(const M3Params& P, uint32_t row, int p, M3Smem& S) {
    m3_load(P, row, p, S);
    m3_select(P, row, p, S, blockIdx.x == 0 && p < 7);
}


__global__ void __launch_bounds__(M3_THREADS) m3_pass_kernel(const __grid_constant__ M3Params P, int pass) {
    extern __shared__ uint32_t sh[];   // [n_rp][256]
    __shared__ M3Smem S;
    const uint32_t row = blockIdx.y, n_rp = P.n_rp;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x) sh[i] = 0;
    pdl_wait();
    pdl_trigger();
    if (pass == 0) {
        // clear the histograms of passes 1..7 (not touched before pass 1 starts)
        const size_t per = (size_t)P.rows * n_rp * 256;
        const size_t n = 7 * per, stride = (size_t)gridDim.x * gridDim.y * blockDim.x;
        for (size_t i = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
            P.hist[per + i] = 0;
        if (threadIdx.x == 0) S.nu = 1;
        if (threadIdx.x == 0) { S.up[0] = 0; S.uq[0] = 0; }
        __syncthreads();
    } else {
        m3_advance(P, row, pass - 1, S);
    }
    const int shift = 56 - 8 * pass;
    const uint32_t nu = S.nu;
    const double* y = P.ylt + (size_t)row * P.ld;
    const uint64_t stride = (uint64_t)gridDim.x * M3_THREADS;
    uint32_t cbin = 0xffffffffu, ccnt = 0;
    for (uint64_t i0 = (uint64_t)blockIdx.x * M3_THREADS + threadIdx.x; i0 < P.T; i0 += stride * M3_KB) {
        uint64_t keys[M3_KB];
#pragma unroll
        for (int q = 0; q < M3_KB; ++q) {
            const uint64_t i = i0 + q * stride;
            keys[q] = i < P.T ? key_of(__ldcg(y + i)) : ~0ull;
        }
#pragma unroll
        for (int q = 0; q < M3_KB; ++q) {
            const uint64_t key = keys[q];
            uint32_t slot = 0xffffffffu;
            if (key != ~0ull) {
                if (pass == 0) slot = 0;
                else
                    for (uint32_t u = 0; u < nu; ++u)
                        if (((key ^ S.up[u]) >> (shift + 8)) == 0) slot = S.uq[u];
            }
            if (slot != 0xffffffffu) {
                const uint32_t bin = slot * 256 + ((uint32_t)(key >> shift) & 255u);
                if (bin != cbin) {
                    if (ccnt) atomicAdd(&sh[cbin], ccnt);
                    cbin = bin;
                    ccnt = 0;
                }
                ++ccnt;
            }
        }
    }
    if (ccnt) atomicAdd(&sh[cbin], ccnt);
    __syncthreads();
    uint32_t* gh = P.hist + ((size_t)pass * P.rows * n_rp + (size_t)row * n_rp) * 256;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

__device__ __forceinline__ double warp_sum_tree(double v) {   // fixed butterfly: lane 0's result is deterministic
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint64_t warp_cnt_tree(uint64_t v) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(M3_THREADS) m3_tail_kernel(const __grid_constant__ M3Params P) {
    __shared__ M3Smem S;
    __shared__ double s_ws[M3_RC][M3_THREADS / 32];
    __shared__ uint64_t s_wc[M3_RC][M3_THREADS / 32];
    __shared__ uint32_t s_last;
    const uint32_t row = blockIdx.y, n_rp = P.n_rp;
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    constexpr uint32_t NW = M3_THREADS / 32;
    pdl_wait();
    pdl_trigger();
    m3_advance(P, row, 7, S);   // S_8: the selected keys
    if (blockIdx.x == 0 && P.dist) {   // the distributed finish reads the values from st[0]
        for (uint32_t r = threadIdx.x; r < n_rp; r += blockDim.x) P.st[2 * ((size_t)row * n_rp + r)] = S.pre[r];
    }
    {   // clear this row's pass-0 histogram for the next call
        uint32_t* h0 = P.hist + (size_t)row * n_rp * 256;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rp * 256u; i += gridDim.x * blockDim.x) h0[i] = 0;
    }
    const double* y = P.ylt + (size_t)row * P.ld;
    const uint64_t stride = (uint64_t)gridDim.x * M3_THREADS;
    for (uint32_t r0 = 0; r0 < n_rp; r0 += M3_RC) {
        uint64_t v[M3_RC];
        double s[M3_RC];
        uint64_t c[M3_RC];
#pragma unroll
        for (int j = 0; j < M3_RC; ++j) {
            v[j] = r0 + j < n_rp ? S.pre[r0 + j] : ~0ull;   // past n_rp: nothing is above
            s[j] = 0.0;
            c[j] = 0;
        }
        for (uint64_t i0 = (uint64_t)blockIdx.x * M3_THREADS + threadIdx.x; i0 < P.T; i0 += stride * M3_KB) {
            double xs[M3_KB];
#pragma unroll
            for (int q = 0; q < M3_KB; ++q) {
                const uint64_t i = i0 + q * stride;
                xs[q] = i < P.T ? __ldcg(y + i) + 0.0 : 0.0;
            }
#pragma unroll
            for (int q = 0; q < M3_KB; ++q) {   // fixed order per thread: deterministic
                const uint64_t key = (uint64_t)__double_as_longlong(xs[q]);
#pragma unroll
                for (int j = 0; j < M3_RC; ++j)
                    if (key > v[j]) { s[j] = __dadd_rn(s[j], xs[q]); ++c[j]; }
            }
        }
#pragma unroll
        for (int j = 0; j < M3_RC; ++j) {
            const double ws = warp_sum_tree(s[j]);
            const uint64_t wc = warp_cnt_tree(c[j]);
            if (lane == 0) { s_ws[j][wid] = ws; s_wc[j][wid] = wc; }
        }
        __syncthreads();
        for (uint32_t j = wid; j < (uint32_t)M3_RC && r0 + j < n_rp; j += NW) {
            double x = lane < NW ? s_ws[j][lane] : 0.0;
            uint64_t cc = lane < NW ? s_wc[j][lane] : 0;
            x = warp_sum_tree(x);
            cc = warp_cnt_tree(cc);
            if (lane == 0) {
                const size_t q = (size_t)row * n_rp + r0 + j;
                P.part_sum[q * P.nblk + blockIdx.x] = x;
                P.part_cnt[q * P.nblk + blockIdx.x] = cc;
            }
        }
        __syncthreads();
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&P.done[row], 1u) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // block partials in a fixed per-lane split, then a fixed tree
    for (uint32_t r = wid; r < n_rp; r += NW) {
        const size_t q = (size_t)row * n_rp + r;
        double sm = 0.0;
        uint64_t cn = 0;
        for (uint32_t b = lane; b < gridDim.x; b += 32) {
            sm = __dadd_rn(sm, __ldcg(P.part_sum + q * P.nblk + b));
            cn += __ldcg(P.part_cnt + q * P.nblk + b);
        }
        sm = warp_sum_tree(sm);
        cn = warp_cnt_tree(cn);
        if (lane == 0) {
            if (P.dist) {
                P.dsum[q] = sm;
                P.dcnt[q] = cn;
            } else {
                const double vv = __longlong_as_double((long long)S.pre[r]);
                const uint64_t k = P.k[r];
                const double tail = __dadd_rn(sm, __dmul_rn((double)(k - cn), vv));
                P.out[q * 2 + 0] = vv;
                P.out[q * 2 + 1] = __ddiv_rn(tail, (double)k);
            }
        }
    }
    if (threadIdx.x == 0) P.done[row] = 0;
}

// distributed: TVaR from the all-reduced tail sums and counts
__global__ void m3_finish_kernel(const __grid_constant__ M3Params P) {
    for (uint32_t q = threadIdx.x; q < P.rows * P.n_rp; q += blockDim.x) {
        const double v = __longlong_as_double((long long)P.st[2 * (size_t)q]);
        const uint64_t k = P.k[q % P.n_rp];
        const double tail = __dadd_rn(P.dsum[q], __dmul_rn((double)(k - P.dcnt[q]), v));
        P.out[(uint64_t)q * 2 + 0] = v;
        P.out[(uint64_t)q * 2 + 1] = __ddiv_rn(tail, (double)k);
    }
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, bool pdl,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ---------------------------------------------------------------------------
// Fast path for n_rp <= 11 (the paper's 10 return periods): three full sweeps,
// then only the candidates.
//  pass 0, 1: full sweeps (digits 0 and 1; pass 1 finds a key's prefix slot by
//             a 256-entry table instead of comparing with every prefix).
//  pass 2:    full sweep.  With the 16-bit prefixes P16_r of all periods known,
//             the distinct ones sorted u_0 < .. < u_{m-1}, a key with 16-bit
//             prefix pk (found by binary search) is
//               - a candidate of u_j if pk == u_j: appended to its warp's
//                 candidate region (ballot order: deterministic), counted
//                 in the digit-2 histogram and added to slot 2j;
//               - in slot 2j+1 if u_j < pk < u_{j+1};
//               - below every period otherwise.
//             Slot sums are thread-private (fixed order).  Every key of a slot
//             above 2 idx(r) has a larger 16-bit prefix than v_r, so
//               sum_{Y > v_r} Y = sum_{slots > 2 idx(r)} B + sum of r's candidates > v_r.
//  pass 3..7: digits 3..7 over the candidate regions only.
//  tail:      the candidates > v_r of each period, block partials, then the
//             last block combines buckets (suffix, fixed order) + candidates.
constexpr int M4_MAXU = 16;      // sorted-prefix search array (padded)
constexpr int M4_MAXM = 11;      // distinct 16-bit prefixes (n_rp <= 11)
constexpr int M4_SLOTS = 2 * M4_MAXM;

struct M4Params {
    M3Params b;
    uint64_t* cand;        // [rows][nblk * warps][cap_w] candidate keys per warp region
    uint32_t* cand_n;      // [rows][nblk * warps]
    uint64_t cap_w;
    double* bsum;          // [rows][M4_SLOTS][nblk] slot sums per block
    uint64_t* bcnt;
};

__device__ __forceinline__ uint64_t m4_region(const M4Params& Q, uint32_t row, uint32_t blk, uint32_t w) {
    return ((uint64_t)row * Q.b.nblk * (M3_THREADS / 32) + (uint64_t)blk * (M3_THREADS / 32) + w);
}

// distinct 16-bit prefixes of the row's periods, sorted ascending, padded with 0xffffffff
__device__ void m4_ulist(const M3Params& P, const M3Smem& S, uint32_t* s_u, uint32_t* s_uslot, uint32_t* s_m) {
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        for (uint32_t r = 0; r < P.n_rp; ++r) {
            const uint32_t v = (uint32_t)(S.pre[r] >> 48);
            bool seen = false;
            for (uint32_t j = 0; j < m; ++j) seen |= s_u[j] == v;
            if (seen) continue;
            uint32_t j = m++;
            while (j > 0 && s_u[j - 1] > v) { s_u[j] = s_u[j - 1]; s_uslot[j] = s_uslot[j - 1]; --j; }
            s_u[j] = v;
            s_uslot[j] = S.rep[r];
        }
        for (uint32_t j = m; j < M4_MAXU; ++j) s_u[j] = 0xffffffffu;
        *s_m = m;
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t m4_rank(const uint32_t* s_u, uint32_t pk) {   // #{j : u_j <= pk}
    uint32_t pos = 0;
#pragma unroll
    for (uint32_t st = M4_MAXU / 2; st >= 1; st >>= 1)
        if (s_u[pos + st - 1] <= pk) pos += st;
    return pos;
}

__global__ void __launch_bounds__(M3_THREADS) m4_pass01_kernel(const __grid_constant__ M4Params Q, int pass) {
    const M3Params& P = Q.b;
    extern __shared__ uint32_t sh[];   // [n_rp][256]
    __shared__ M3Smem S;
    __shared__ uint8_t t1[256];
    const uint32_t row = blockIdx.y, n_rp = P.n_rp;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x) sh[i] = 0;
    for (uint32_t i = threadIdx.x; i < 256u; i += blockDim.x) t1[i] = 0xff;
    pdl_wait();
    pdl_trigger();
    if (pass == 0) {
        const size_t per = (size_t)P.rows * n_rp * 256;
        const size_t n = 7 * per, stride = (size_t)gridDim.x * gridDim.y * blockDim.x;
        for (size_t i = ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
            P.hist[per + i] = 0;
        m3_load(P, row, 0, S);
    } else {
        m3_advance(P, row, 0, S);
        for (uint32_t u = threadIdx.x; u < S.nu; u += blockDim.x) t1[(uint32_t)(S.up[u] >> 56)] = (uint8_t)S.uq[u];
        __syncthreads();
    }
    const int shift = 56 - 8 * pass;
    const double* y = P.ylt + (size_t)row * P.ld;
    const uint64_t stride = (uint64_t)gridDim.x * M3_THREADS;
    uint32_t cbin = 0xffffffffu, ccnt = 0;
    for (uint64_t i0 = (uint64_t)blockIdx.x * M3_THREADS + threadIdx.x; i0 < P.T; i0 += stride * M3_KB) {
        uint64_t keys[M3_KB];
#pragma unroll
        for (int q = 0; q < M3_KB; ++q) {
            const uint64_t i = i0 + q * stride;
            keys[q] = i < P.T ? key_of(__ldcg(y + i)) : ~0ull;
        }
#pragma unroll
        for (int q = 0; q < M3_KB; ++q) {
            const uint64_t key = keys[q];
            if (key == ~0ull) continue;
            const uint32_t slot = pass == 0 ? 0u : (uint32_t)t1[(uint32_t)(key >> 56)];
            if (slot == 0xffu) continue;
            const uint32_t bin = slot * 256 + ((uint32_t)(key >> shift) & 255u);
            if (bin != cbin) {
                if (ccnt) atomicAdd(&sh[cbin], ccnt);
                cbin = bin;
                ccnt = 0;
            }
            ++ccnt;
        }
    }
    if (ccnt) atomicAdd(&sh[cbin], ccnt);
    __syncthreads();
    uint32_t* gh = P.hist + ((size_t)pass * P.rows * n_rp + (size_t)row * n_rp) * 256;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

__global__ void __launch_bounds__(M3_THREADS) m4_pass2_kernel(const __grid_constant__ M4Params Q) {
    const M3Params& P = Q.b;
    extern __shared__ __align__(16) unsigned char dsm2[];
    const uint32_t n_rp = P.n_rp;
    uint32_t* sh = reinterpret_cast<uint32_t*>(dsm2);                                     // [n_rp][256]
    double* s_bs = reinterpret_cast<double*>(dsm2 + (size_t)n_rp * 256 * 4);              // [M4_SLOTS][THREADS]
    uint32_t* s_bc = reinterpret_cast<uint32_t*>(s_bs + (size_t)M4_SLOTS * M3_THREADS);   // [M4_SLOTS][THREADS]
    __shared__ M3Smem S;
    __shared__ uint32_t s_u[M4_MAXU], s_uslot[M4_MAXU], s_m;
    const uint32_t row = blockIdx.y, tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    for (uint32_t i = tid; i < n_rp * 256u; i += blockDim.x) sh[i] = 0;
    for (uint32_t i = tid; i < M4_SLOTS * M3_THREADS; i += blockDim.x) { s_bs[i] = 0.0; s_bc[i] = 0; }
    pdl_wait();
    pdl_trigger();
    m3_advance(P, row, 1, S);   // S_2: the 16-bit prefixes
    m4_ulist(P, S, s_u, s_uslot, &s_m);
    const uint32_t m = s_m;
    const double* y = P.ylt + (size_t)row * P.ld;
    const uint64_t stride = (uint64_t)gridDim.x * M3_THREADS;
    uint64_t* cr = Q.cand + m4_region(Q, row, blockIdx.x, wid) * Q.cap_w;
    uint32_t ncand = 0;   // warp-uniform
    const unsigned lt = (1u << lane) - 1u;
    uint32_t cbin = 0xffffffffu, ccnt = 0;
    // the loop trip count is warp-uniform (i0 - lane is the same for the warp)
    for (uint64_t i0 = (uint64_t)blockIdx.x * M3_THREADS + tid; i0 - lane < P.T; i0 += stride * M3_KB) {
        uint64_t keys[M3_KB];
#pragma unroll
        for (int q = 0; q < M3_KB; ++q) {
            const uint64_t i = i0 + q * stride;
            keys[q] = i < P.T ? key_of(__ldcg(y + i)) : ~0ull;
        }
#pragma unroll
        for (int q = 0; q < M3_KB; ++q) {
            const uint64_t key = keys[q];
            const bool valid = key != ~0ull;
            const uint32_t pk = (uint32_t)(key >> 48);
            const uint32_t pos = valid ? m4_rank(s_u, pk) : 0u;
            const bool is_c = pos > 0 && s_u[pos - 1] == pk;
            const unsigned cm = __ballot_sync(0xffffffffu, is_c);
            if (is_c) {
                cr[ncand + __popc(cm & lt)] = key;
                const uint32_t bin = s_uslot[pos - 1] * 256 + ((uint32_t)(key >> 40) & 255u);
                if (bin != cbin) {
                    if (ccnt) atomicAdd(&sh[cbin], ccnt);
                    cbin = bin;
                    ccnt = 0;
                }
                ++ccnt;
            }
            if (pos > 0) {   // slot 2(pos-1) (== u_{pos-1}) or 2(pos-1)+1 (strictly between u_{pos-1} and u_pos)
                const uint32_t bi = (2 * (pos - 1) + (is_c ? 0u : 1u)) * M3_THREADS + tid;
                s_bs[bi] = __dadd_rn(s_bs[bi], __longlong_as_double((long long)key));
                s_bc[bi] += 1;
            }
            ncand += __popc(cm);
        }
    }
    if (ccnt) atomicAdd(&sh[cbin], ccnt);
    if (lane == 0) Q.cand_n[m4_region(Q, row, blockIdx.x, wid)] = ncand;
    __syncthreads();
    uint32_t* gh = P.hist + ((size_t)2 * P.rows * n_rp + (size_t)row * n_rp) * 256;
    for (uint32_t i = tid; i < n_rp * 256u; i += blockDim.x)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
    // slot partials: fixed tree over the block's threads
    const uint32_t ns = 2 * m;
    for (uint32_t w = M3_THREADS / 2; w >= 1; w >>= 1) {
        for (uint32_t idx = tid; idx < ns * w; idx += blockDim.x) {
            const uint32_t j = idx / w, t = idx % w;
            s_bs[j * M3_THREADS + t] = __dadd_rn(s_bs[j * M3_THREADS + t], s_bs[j * M3_THREADS + t + w]);
            s_bc[j * M3_THREADS + t] += s_bc[j * M3_THREADS + t + w];
        }
        __syncthreads();
    }
    for (uint32_t j = tid; j < ns; j += blockDim.x) {
        Q.bsum[((size_t)row * M4_SLOTS + j) * P.nblk + blockIdx.x] = s_bs[j * M3_THREADS];
        Q.bcnt[((size_t)row * M4_SLOTS + j) * P.nblk + blockIdx.x] = s_bc[j * M3_THREADS];
    }
}

__global__ void __launch_bounds__(M3_THREADS) m4_cand_pass_kernel(const __grid_constant__ M4Params Q, int pass) {
    const M3Params& P = Q.b;
    extern __shared__ uint32_t sh[];
    __shared__ M3Smem S;
    const uint32_t row = blockIdx.y, n_rp = P.n_rp, lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x) sh[i] = 0;
    pdl_wait();
    pdl_trigger();
    m3_advance(P, row, pass - 1, S);
    const int shift = 56 - 8 * pass;
    const uint32_t nu = S.nu;
    const uint64_t reg = m4_region(Q, row, blockIdx.x, wid);
    const uint64_t* cr = Q.cand + reg * Q.cap_w;
    const uint32_t n = __ldcg(Q.cand_n + reg);
    uint32_t cbin = 0xffffffffu, ccnt = 0;
    for (uint32_t i = lane; i < n; i += 32) {
        const uint64_t key = __ldcg(cr + i);
        uint32_t slot = 0xffffffffu;
        for (uint32_t u = 0; u < nu; ++u)
            if (((key ^ S.up[u]) >> (shift + 8)) == 0) slot = S.uq[u];
        if (slot == 0xffffffffu) continue;
        const uint32_t bin = slot * 256 + ((uint32_t)(key >> shift) & 255u);
        if (bin != cbin) {
            if (ccnt) atomicAdd(&sh[cbin], ccnt);
            cbin = bin;
            ccnt = 0;
        }
        ++ccnt;
    }
    if (ccnt) atomicAdd(&sh[cbin], ccnt);
    __syncthreads();
    uint32_t* gh = P.hist + ((size_t)pass * P.rows * n_rp + (size_t)row * n_rp) * 256;
    for (uint32_t i = threadIdx.x; i < n_rp * 256u; i += blockDim.x)
        if (sh[i]) atomicAdd(&gh[i], sh[i]);
}

__global__ void __launch_bounds__(M3_THREADS) m4_tail_kernel(const __grid_constant__ M4Params Q) {
    const M3Params& P = Q.b;
    __shared__ M3Smem S;
    __shared__ uint32_t s_u[M4_MAXU], s_uslot[M4_MAXU], s_m;
    __shared__ double s_ws[M3_RC][M3_THREADS / 32];
    __shared__ uint64_t s_wc[M3_RC][M3_THREADS / 32];
    __shared__ double s_B[M4_SLOTS];
    __shared__ uint64_t s_Bc[M4_SLOTS];
    __shared__ uint32_t s_last;
    const uint32_t row = blockIdx.y, n_rp = P.n_rp;
    const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
    constexpr uint32_t NW = M3_THREADS / 32;
    pdl_wait();
    pdl_trigger();
    m3_advance(P, row, 7, S);   // S_8: the selected keys
    if (blockIdx.x == 0 && P.dist)   // the distributed finish reads the values from st[0]
        for (uint32_t r = threadIdx.x; r < n_rp; r += blockDim.x) P.st[2 * ((size_t)row * n_rp + r)] = S.pre[r];
    {   // clear this row's pass-0 histogram for the next call
        uint32_t* h0 = P.hist + (size_t)row * n_rp * 256;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_rp * 256u; i += gridDim.x * blockDim.x) h0[i] = 0;
    }
    const uint64_t reg = m4_region(Q, row, blockIdx.x, wid);
    const uint64_t* cr = Q.cand + reg * Q.cap_w;
    const uint32_t n = __ldcg(Q.cand_n + reg);
    for (uint32_t r0 = 0; r0 < n_rp; r0 += M3_RC) {
        uint64_t v[M3_RC];
        double s[M3_RC];
        uint64_t c[M3_RC];
#pragma unroll
        for (int j = 0; j < M3_RC; ++j) {
            v[j] = r0 + j < n_rp ? S.pre[r0 + j] : ~0ull;
            s[j] = 0.0;
            c[j] = 0;
        }
        for (uint32_t i = lane; i < n; i += 32) {   // fixed order: deterministic
            const uint64_t key = __ldcg(cr + i);
#pragma unroll
            for (int j = 0; j < M3_RC; ++j)
                if (key > v[j] && ((key ^ v[j]) >> 48) == 0) { s[j] = __dadd_rn(s[j], __longlong_as_double((long long)key)); ++c[j]; }
        }
#pragma unroll
        for (int j = 0; j < M3_RC; ++j) {
            const double ws = warp_sum_tree(s[j]);
            const uint64_t wc = warp_cnt_tree(c[j]);
            if (lane == 0) { s_ws[j][wid] = ws; s_wc[j][wid] = wc; }
        }
        __syncthreads();
        for (uint32_t j = wid; j < (uint32_t)M3_RC && r0 + j < n_rp; j += NW) {
            double x = lane < NW ? s_ws[j][lane] : 0.0;
            uint64_t cc = lane < NW ? s_wc[j][lane] : 0;
            x = warp_sum_tree(x);
            cc = warp_cnt_tree(cc);
            if (lane == 0) {
                const size_t q = (size_t)row * n_rp + r0 + j;
                P.part_sum[q * P.nblk + blockIdx.x] = x;
                P.part_cnt[q * P.nblk + blockIdx.x] = cc;
            }
        }
        __syncthreads();
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&P.done[row], 1u) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // S_8 has the same 16-bit prefixes as S_2: the same sorted list
    m4_ulist(P, S, s_u, s_uslot, &s_m);
    const uint32_t m = s_m;
    for (uint32_t j = wid; j < 2 * m; j += NW) {   // slot totals: fixed per-lane split + tree
        double sm = 0.0;
        uint64_t cn = 0;
        for (uint32_t b = lane; b < gridDim.x; b += 32) {
            sm = __dadd_rn(sm, __ldcg(Q.bsum + ((size_t)row * M4_SLOTS + j) * P.nblk + b));
            cn += __ldcg(Q.bcnt + ((size_t)row * M4_SLOTS + j) * P.nblk + b);
        }
        sm = warp_sum_tree(sm);
        cn = warp_cnt_tree(cn);
        if (lane == 0) { s_B[j] = sm; s_Bc[j] = cn; }
    }
    __syncthreads();
    for (uint32_t r = wid; r < n_rp; r += NW) {
        const size_t q = (size_t)row * n_rp + r;
        double sm = 0.0;
        uint64_t cn = 0;
        for (uint32_t b = lane; b < gridDim.x; b += 32) {
            sm = __dadd_rn(sm, __ldcg(P.part_sum + q * P.nblk + b));
            cn += __ldcg(P.part_cnt + q * P.nblk + b);
        }
        sm = warp_sum_tree(sm);
        cn = warp_cnt_tree(cn);
        if (lane == 0) {
            const uint32_t idx = m4_rank(s_u, (uint32_t)(S.pre[r] >> 48)) - 1;   // u_idx == P16_r
            double bs = 0.0;
            uint64_t bc = 0;
            for (int j = 2 * (int)m - 1; j > 2 * (int)idx; --j) { bs = __dadd_rn(bs, s_B[j]); bc += s_Bc[j]; }
            sm = __dadd_rn(bs, sm);
            cn += bc;
            if (P.dist) {
                P.dsum[q] = sm;
                P.dcnt[q] = cn;
            } else {
                const double vv = __longlong_as_double((long long)S.pre[r]);
                const uint64_t k = P.k[r];
                const double tail = __dadd_rn(sm, __dmul_rn((double)(k - cn), vv));
                P.out[q * 2 + 0] = vv;
                P.out[q * 2 + 1] = __ddiv_rn(tail, (double)k);
            }
        }
    }
    if (threadIdx.x == 0) P.done[row] = 0;
}

cudaError_t launch_m4(const M3Params& P, MetricsScratch& m, bool dist, ncclComm_t comm, cudaStream_t s,
                      int* nccl_err) {
    M4Params Q{};
    Q.b = P;
    const uint32_t rows = P.rows, n_rp = P.n_rp, nblk = P.nblk;
    const uint64_t stride = (uint64_t)nblk * M3_THREADS;
    Q.cap_w = 32 * ((P.T + stride - 1) / stride) * 1;
    const uint64_t nreg = (uint64_t)rows * nblk * (M3_THREADS / 32);
    const uint64_t need = nreg * Q.cap_w;
    cudaError_t e;
    if (m.cand_cap < need) {
        cudaFree(m.cand);
        m.cand = nullptr;
        m.cand_cap = 0;
        if ((e = cudaMalloc(&m.cand, need * sizeof(uint64_t))) != cudaSuccess) return e;
        m.cand_cap = need;
    }
    if (m.cand_n_cap < nreg) {
        cudaFree(m.cand_n);
        m.cand_n = nullptr;
        m.cand_n_cap = 0;
        if ((e = cudaMalloc(&m.cand_n, nreg * sizeof(uint32_t))) != cudaSuccess) return e;
        m.cand_n_cap = nreg;
    }
    const uint64_t nb = (uint64_t)rows * M4_SLOTS * nblk;
    if (m.bpart_cap < nb) {
        cudaFree(m.bsum);
        cudaFree(m.bcnt);
        m.bsum = nullptr;
        m.bcnt = nullptr;
        m.bpart_cap = 0;
        if ((e = cudaMalloc(&m.bsum, nb * sizeof(double))) != cudaSuccess) return e;
        if ((e = cudaMalloc(&m.bcnt, nb * sizeof(uint64_t))) != cudaSuccess) return e;
        m.bpart_cap = nb;
    }
    Q.cand = m.cand;
    Q.cand_n = m.cand_n;
    Q.bsum = m.bsum;
    Q.bcnt = m.bcnt;
    const size_t smem = (size_t)n_rp * 256 * sizeof(uint32_t);
    const size_t smem2 = smem + (size_t)M4_SLOTS * M3_THREADS * (sizeof(double) + sizeof(uint32_t));
    static size_t set01 = 0, set2 = 0, setc = 0;
    if (smem > 32 * 1024 && smem > set01) {
        if ((e = cudaFuncSetAttribute(m4_pass01_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
        set01 = smem;
    }
    if (smem > 32 * 1024 && smem > setc) {
        if ((e = cudaFuncSetAttribute(m4_cand_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess) return e;
        setc = smem;
    }
    if (smem2 > set2) {
        if ((e = cudaFuncSetAttribute(m4_pass2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2)) != cudaSuccess) return e;
        set2 = smem2;
    }
    if (nccl_err) *nccl_err = 0;
    const size_t nh = (size_t)rows * n_rp * 256;
    const bool pdl = !comm;
    const dim3 grid(nblk, rows), blk(M3_THREADS);
    // ARA_METRICS_TRACE=1: events between the launches (breaks the PDL overlap), per-kernel times on stderr
    static const bool trace = [] { const char* v = getenv("ARA_METRICS_TRACE"); return v && atoi(v); }();
    static cudaEvent_t tev[12];
    static bool tev_init = false;
    int nt = 0;
    if (trace && !tev_init) {
        for (auto& x : tev) cudaEventCreate(&x);
        tev_init = true;
    }
    auto mark = [&] { if (trace) cudaEventRecord(tev[nt++], s); };
    auto red = [&](int pass) {
        mark();
        if (comm && ncclAllReduce(P.hist + pass * nh, P.hist + pass * nh, nh, ncclUint32, ncclSum, comm, s) != ncclSuccess)
            *nccl_err = 1;
    };
    auto enqueue = [&]() -> cudaError_t {
        cudaError_t r = launch_pdl(m4_pass01_kernel, grid, blk, smem, s, false, Q, 0);
        if (r == cudaSuccess) red(0);
        if (r == cudaSuccess && !(nccl_err && *nccl_err)) r = launch_pdl(m4_pass01_kernel, grid, blk, smem, s, pdl, Q, 1);
        if (r == cudaSuccess && !(nccl_err && *nccl_err)) red(1);
        if (r == cudaSuccess && !(nccl_err && *nccl_err)) r = launch_pdl(m4_pass2_kernel, grid, blk, smem2, s, pdl, Q);
        if (r == cudaSuccess && !(nccl_err && *nccl_err)) red(2);
        for (int pass = 3; pass < 8 && r == cudaSuccess && !(nccl_err && *nccl_err); ++pass) {
            r = launch_pdl(m4_cand_pass_kernel, grid, blk, smem, s, pdl, Q, pass);
            if (r == cudaSuccess) red(pass);
        }
        if (r == cudaSuccess && !(nccl_err && *nccl_err)) r = launch_pdl(m4_tail_kernel, grid, blk, 0, s, pdl, Q);
        if (r == cudaSuccess && !(nccl_err && *nccl_err) && dist) {   // the all-reduced tail sums -> TVaR
            const size_t nq = (size_t)rows * n_rp;
            if (comm && (ncclGroupStart() != ncclSuccess ||
                         ncclAllReduce(P.dsum, P.dsum, nq, ncclDouble, ncclSum, comm, s) != ncclSuccess ||
                         ncclAllReduce(P.dcnt, P.dcnt, nq, ncclUint64, ncclSum, comm, s) != ncclSuccess ||
                         ncclGroupEnd() != ncclSuccess))
                *nccl_err = 1;
            else
                m3_finish_kernel<<<1, 256, 0, s>>>(P);
            r = cudaGetLastError();
        }
        return r;
    };
    // Launches without NCCL go through a CUDA graph of the kernels (with their
    // programmatic-launch edges), kept in a two-entry cache keyed by every
    // argument (consecutive multi-GPU runs alternate two global-YLT buffers).
    // The distributed select with NCCL all-reduces between the passes is
    // launched eagerly: captured into a graph it hung at N = 4 (DESIGN.md
    // section 7).
    const char* g_env = getenv("ARA_METRICS_GRAPH");
    const bool use_graph = !g_env || atoi(g_env);
    static_assert(sizeof(M4Params) + sizeof(cudaStream_t) + sizeof(ncclComm_t) + 1 <= sizeof(m.m4_key[0]),
                  "graph key buffer");
    if (!comm && !trace && use_graph) {
        unsigned char key[sizeof(m.m4_key[0])] = {};
        std::memcpy(key, &Q, sizeof(Q));
        std::memcpy(key + sizeof(Q), &s, sizeof(s));
        std::memcpy(key + sizeof(Q) + sizeof(s), &comm, sizeof(comm));
        key[sizeof(Q) + sizeof(s) + sizeof(comm)] = dist ? 1 : 0;
        int hit = -1;
        for (int q = 0; q < 2; ++q)
            if (m.m4_exec[q] && std::memcmp(key, m.m4_key[q], sizeof(key)) == 0) hit = q;
        if (hit < 0) {
            const int q = m.m4_next;
            m.m4_next ^= 1;
            if (m.m4_exec[q]) cudaGraphExecDestroy(m.m4_exec[q]);
            m.m4_exec[q] = nullptr;
            cudaGraph_t g = nullptr;
            if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
                const cudaError_t r = enqueue();
                const cudaError_t r2 = cudaStreamEndCapture(s, &g);
                if (nccl_err && *nccl_err) *nccl_err = 0;   // retried below without the graph
                if (r == cudaSuccess && r2 == cudaSuccess && g &&
                    cudaGraphInstantiate(&m.m4_exec[q], g, 0) == cudaSuccess) {
                    std::memcpy(m.m4_key[q], key, sizeof(key));
                    hit = q;
                } else {
                    m.m4_exec[q] = nullptr;
                }
                if (g) cudaGraphDestroy(g);
            }
            cudaGetLastError();   // a stream that cannot be captured: plain launches below
        }
        if (hit >= 0) e = cudaGraphLaunch(m.m4_exec[hit], s);
        else e = enqueue();
    } else {
        mark();
        e = enqueue();
        mark();
    }
    if (trace && e == cudaSuccess) {
        cudaEventSynchronize(tev[nt - 1]);
        fprintf(stderr, "m4 trace us:");
        for (int i = 1; i < nt; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tev[i - 1], tev[i]);
            fprintf(stderr, " %.1f", ms * 1e3f);
        }
        fprintf(stderr, "\n");
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess || (nccl_err && *nccl_err)) {
        cudaGetLastError();
        cudaMemsetAsync(m.hist8, 0, 8 * nh * sizeof(uint32_t), s);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    return e;
}



// The 8 passes + tail (+ the all-reduces when comm != null in distributed mode).
cudaError_t launch_m3(const double* d_ylt, uint64_t T, uint64_t ld, uint32_t rows, uint32_t n_rp,
                      const uint64_t* h_k, MetricsScratch& m, int nblk, bool dist, ncclComm_t comm,
                      cudaStream_t s, int* nccl_err) {
    M3Params P{};
    P.ylt = d_ylt;
    P.T = T;
    P.ld = ld;
    P.n_rp = n_rp;
    P.nblk = (uint32_t)nblk;
    P.rows = rows;
    P.hist = m.hist8;
    P.st = m.st;
    P.strep = m.strep;
    P.part_sum = m.part_sum;
    P.part_cnt = m.part_cnt;
    P.done = m.done;
    P.out = m.out;
    P.dsum = m.dsum;
    P.dcnt = m.dcnt;
    P.dist = dist ? 1 : 0;
    for (uint32_t i = 0; i < n_rp; ++i) P.k[i] = h_k[i];
    const char* m3_env = getenv("ARA_METRICS_M3");   // A/B and tests: the general path for any n_rp
    const int m4_off = m3_env ? atoi(m3_env) : 0;
    if (n_rp <= M4_MAXM && !m4_off) return launch_m4(P, m, dist, comm, s, nccl_err);
    const size_t smem = (size_t)n_rp * 256 * sizeof(uint32_t);
    static size_t smem_set = 0;
    if (smem > 32 * 1024 && smem > smem_set) {
        cudaError_t e = cudaFuncSetAttribute(m3_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        smem_set = smem;
    }
    if (nccl_err) *nccl_err = 0;
    const size_t nh = (size_t)rows * n_rp * 256;
    cudaError_t e = cudaSuccess;
    for (int pass = 0; pass < 8 && e == cudaSuccess; ++pass) {
        // PDL between our own consecutive kernels only (not after NCCL or the caller's work)
        e = launch_pdl(m3_pass_kernel, dim3(nblk, rows), dim3(M3_THREADS), smem, s, pass > 0 && !comm, P, pass);
        if (e == cudaSuccess && comm &&
            ncclAllReduce(P.hist + pass * nh, P.hist + pass * nh, nh, ncclUint32, ncclSum, comm, s) != ncclSuccess) {
            *nccl_err = 1;
            break;
        }
    }
    if (e == cudaSuccess && !(nccl_err && *nccl_err))
        e = launch_pdl(m3_tail_kernel, dim3(nblk, rows), dim3(M3_THREADS), 0, s, !comm, P);
    if (e == cudaSuccess && !(nccl_err && *nccl_err) && dist) {
        const size_t nq = (size_t)rows * n_rp;
        if (comm && (ncclGroupStart() != ncclSuccess || ncclAllReduce(P.dsum, P.dsum, nq, ncclDouble, ncclSum, comm, s) != ncclSuccess ||
                     ncclAllReduce(P.dcnt, P.dcnt, nq, ncclUint64, ncclSum, comm, s) != ncclSuccess ||
                     ncclGroupEnd() != ncclSuccess))
            *nccl_err = 1;
        else
            m3_finish_kernel<<<1, 256, 0, s>>>(P);
    }
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess || (nccl_err && *nccl_err)) {
        // a partial sequence may leave histograms dirty: clear them for the next call
        cudaGetLastError();
        cudaMemsetAsync(m.hist8, 0, 8 * nh * sizeof(uint32_t), s);
        if (e == cudaSuccess) e = cudaGetLastError();
    }
    return e;
}


}  // namespace

cudaError_t launch_metrics_dist(const double* d_ylt, uint64_t T_local, uint64_t ld, uint32_t rows, uint32_t n_rp,
                                const uint64_t* h_k, MetricsScratch& m, int nblk, ncclComm_t comm,
                                cudaStream_t s, int* nccl_err) {
    return launch_m3(d_ylt, T_local, ld, rows, n_rp, h_k, m, nblk, true, comm, s, nccl_err);
}

cudaError_t metrics_alloc(MetricsScratch& m, uint32_t rows, uint32_t n_rp, int nblk) {
    const size_t need = (size_t)rows * n_rp;
    if (m.cap_rows_rp >= need && m.nblk >= nblk && m.cap_rows >= rows) return cudaSuccess;
    metrics_free(m);
    const size_t rr = need;
    cudaError_t e;
    if ((e = cudaMalloc(&m.part_sum, rr * nblk * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.part_cnt, rr * nblk * sizeof(uint64_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.out, rr * 2 * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.done, rows * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.dsum, rr * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.dcnt, rr * sizeof(uint64_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.hist8, 8 * rr * 256 * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMemset(m.hist8, 0, 8 * rr * 256 * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.st, 2 * rr * 2 * sizeof(uint64_t))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&m.strep, 2 * rr * sizeof(uint32_t))) != cudaSuccess) return e;
    if ((e = cudaMemset(m.done, 0, rows * sizeof(uint32_t))) != cudaSuccess) return e;
    m.cap_rows_rp = need;
    m.cap_rows = rows;
    m.nblk = nblk;
    return cudaSuccess;
}

void metrics_free(MetricsScratch& m) {
    cudaFree(m.part_sum);
    cudaFree(m.part_cnt);
    cudaFree(m.out);
    cudaFree(m.done);
    cudaFree(m.dsum);
    cudaFree(m.dcnt);
    cudaFree(m.hist8);
    cudaFree(m.st);
    cudaFree(m.strep);
    cudaFree(m.cand);
    cudaFree(m.cand_n);
    cudaFree(m.bsum);
    cudaFree(m.bcnt);
    for (auto& x : m.m4_exec)
        if (x) cudaGraphExecDestroy(x);
    m = MetricsScratch{};
}

cudaError_t launch_metrics(const double* d_ylt, uint64_t T, uint64_t ld, uint32_t rows,
                           uint32_t n_rp, const uint64_t* h_k, MetricsScratch& m, int nblk, cudaStream_t s) {
    return launch_m3(d_ylt, T, ld, rows, n_rp, h_k, m, nblk, false, nullptr, s, nullptr);
}

}  // namespace ara
