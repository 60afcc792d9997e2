// ep_curve.cu -- aggregate exceedance-probability (EP) curve of the YLT rows
// (SURVEY.md 8f F4 "full EP curve"; reading A23 in DESIGN.md section 2):
//   counts[row][i] = #{t : Y[row][t] > x_i},   EP(x_i) = counts / T.
// The loss at an exceedance probability p is PML(1/p) (ara_metrics); this is
// the other direction of the curve, at any number of loss thresholds.
//
// One sweep: each YLT value finds b = #{i : x_i < y} by binary search over
// the (non-decreasing) thresholds staged in shared memory and adds one to bin
// b of a block histogram (lanes with the same bin merged by match_any, one
// shared atomic per group); block histograms are added into a global one;
// then counts[i] = sum_{b > i} hist[b] (a suffix sum).  Integer counts: exact
// and independent of the order of the adds, so the multi-GPU curve is the
// sum of the shards' curves (one all-reduce).
#include "ara_internal.cuh"

namespace ara {
namespace {

__global__ void __launch_bounds__(256) ep_hist_kernel(const double* __restrict__ ylt, uint64_t T, uint64_t ld,
                                                      const double* __restrict__ x, uint32_t n,
                                                      unsigned long long* __restrict__ hist /*[rows][n+1]*/) {
    extern __shared__ __align__(16) unsigned char dsm[];
    double* sx = reinterpret_cast<double*>(dsm);
    uint32_t* sh = reinterpret_cast<uint32_t*>(dsm + (size_t)n * sizeof(double));
    const uint32_t row = blockIdx.y;
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sx[i] = x[i];
    for (uint32_t i = threadIdx.x; i <= n; i += blockDim.x) sh[i] = 0u;
    __syncthreads();
    const double* y = ylt + (uint64_t)row * ld;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < T; i0 += stride) {   // warp-uniform trip count
        const uint64_t i = i0 + threadIdx.x;
        uint32_t b = 0xffffffffu;
        if (i < T) {
            const double v = __ldcg(y + i);
            uint32_t lo = 0, hi = n;   // b = #{x_j < v}: first j with !(x_j < v)
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (sx[mid] < v) lo = mid + 1;
                else hi = mid;
            }
            b = lo;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        if (b != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&sh[b], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i <= n; i += blockDim.x)
        if (sh[i]) atomicAdd(hist + (uint64_t)row * (n + 1) + i, (unsigned long long)sh[i]);
}

// counts[row][i] = sum of hist[row][b] over b > i (one block per row)
__global__ void __launch_bounds__(256) ep_suffix_kernel(const unsigned long long* __restrict__ hist, uint32_t n,
                                                        uint64_t* __restrict__ counts) {
    if (threadIdx.x != 0) return;
    const uint32_t row = blockIdx.x;
    const unsigned long long* h = hist + (uint64_t)row * (n + 1);
    uint64_t acc = 0;
    for (uint32_t i = n; i-- > 0;) {
        acc += h[i + 1];
        counts[(uint64_t)row * n + i] = acc;
    }
}

}  // namespace

cudaError_t launch_ep_curve(const double* d_ylt, uint64_t T, uint64_t ld, uint32_t rows, const double* d_x,
                            uint32_t n, unsigned long long* d_hist, uint64_t* d_counts, int n_sm, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(d_hist, 0, (size_t)rows * (n + 1) * sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    const size_t smem = (size_t)n * sizeof(double) + (size_t)(n + 1) * sizeof(uint32_t);
    if (smem > 32 * 1024) {
        e = cudaFuncSetAttribute(ep_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    uint64_t blocks = (T + 255) / 256;
    const uint64_t cap = (uint64_t)(n_sm > 0 ? n_sm : 148) * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    ep_hist_kernel<<<dim3((unsigned)blocks, rows), 256, smem, s>>>(d_ylt, T, ld, d_x, n, d_hist);
    ep_suffix_kernel<<<rows, 32, 0, s>>>(d_hist, n, d_counts);
    return cudaGetLastError();
}

}  // namespace ara
