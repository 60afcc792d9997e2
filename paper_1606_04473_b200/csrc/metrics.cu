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
#include "ara_internal.cuh"

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
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(&P.done[row], 1u) == P.nblk - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    // Last block of this row: stage the row's histograms in shared memory
    // (coalesced), then one warp per return period finds the digit with a
    // warp-wide scan from the top digit down.
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
    if (threadIdx.x == 0) P.done[row] = 0;
}

__global__ void __launch_bounds__(256) tail_kernel(const __grid_constant__ MParams P) {
    __shared__ double s_sum[256];
    __shared__ uint64_t s_cnt[256];
    __shared__ uint32_t s_last;
    const uint32_t row = blockIdx.y, n_rp = P.n_rp;
    const double* y = P.ylt + (uint64_t)row * P.ld;
    constexpr int KB = 8;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint32_t r = 0; r < n_rp; ++r) {
        const double v = __longlong_as_double((long long)P.prefix[row * n_rp + r]);
        double s = 0.0;
        uint64_t c = 0;
        for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < P.T; i0 += stride * KB) {
            double xs[KB];
#pragma unroll
            for (int q = 0; q < KB; ++q) {
                const uint64_t i = i0 + q * stride;
                xs[q] = i < P.T ? __ldcg(y + i) + 0.0 : -1.0;
            }
#pragma unroll
            for (int q = 0; q < KB; ++q)   // fixed order per thread: deterministic
                if (xs[q] > v) { s = __dadd_rn(s, xs[q]); ++c; }
        }
        s_sum[threadIdx.x] = s;
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
            P.part_sum[((uint64_t)row * n_rp + r) * P.nblk + blockIdx.x] = s_sum[0];
            P.part_cnt[((uint64_t)row * n_rp + r) * P.nblk + blockIdx.x] = s_cnt[0];
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
            const uint64_t k = P.k[r];
            const double tail = __dadd_rn(s, __dmul_rn((double)(k - c), v));
            P.out[((uint64_t)row * n_rp + r) * 2 + 0] = v;
            P.out[((uint64_t)row * n_rp + r) * 2 + 1] = __ddiv_rn(tail, (double)k);
        }
    }
    if (threadIdx.x == 0) P.done[row] = 0;
}

}  // namespace

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
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(radix_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    init_kernel<<<rows, 256, 0, s>>>(P);
    for (int pass = 0; pass < 8; ++pass)
        radix_pass_kernel<<<dim3(P.nblk, rows), 256, smem, s>>>(P, pass);
    tail_kernel<<<dim3(P.nblk, rows), 256, 0, s>>>(P);
    return cudaGetLastError();
}

}  // namespace ara
