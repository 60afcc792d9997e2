// microbench.cu — measured ceilings for the ARA gather:
//   mb_stream_read  : streaming 256-bit read of a large buffer (HBM read BW)
//   mb_gather       : random row gathers of `row_bytes` from a `table_bytes`
//                     table (HBM-sized -> DRAM random-access ceiling; 32 MB ->
//                     L2 gather ceiling), ids hashed on the fly
// Separate library (libara_mb.so); not on the product path.  Each call
// allocates, times `iters` launches with CUDA events, and returns ms/launch.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

namespace {

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return (uint32_t)x;
}

__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

__global__ void stream_read(const double* __restrict__ p, uint64_t n4, double* out) {
    double s = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
        double a, b, c, d;
        ld256(p + 4 * i, a, b, c, d);
        s += a + b + c + d;
    }
    if (s == 123.456) out[0] = s;
}

template <int SEC>
__global__ void gather(const double* __restrict__ tab, uint32_t n_rows, uint64_t row_elems, uint64_t n, uint32_t seed,
                       double* out) {
    double s = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t r = hash32(i * 0x9E3779B97F4A7C15ULL + seed) % n_rows;
        const double* row = tab + (uint64_t)r * row_elems;
#pragma unroll
        for (int k = 0; k < SEC; ++k) {
            double a, b, c, d;
            ld256(row + 4 * k, a, b, c, d);
            s += a + b + c + d;
        }
    }
    if (s == 123.456) out[0] = s;
}

float time_it(void (*launch)(void*), void* arg, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch(arg);   // warm-up
    cudaEventRecord(a);
    for (int i = 0; i < iters; ++i) launch(arg);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / iters;
}

struct SArg { const double* p; uint64_t n4; double* out; int grid; };
void launch_stream(void* v) {
    SArg* a = (SArg*)v;
    stream_read<<<a->grid, 256>>>(a->p, a->n4, a->out);
}

struct GArg { const double* tab; uint32_t n_rows; uint64_t row_elems; uint64_t n; uint32_t seed; double* out; int grid; int sec; };
void launch_gather(void* v) {
    GArg* a = (GArg*)v;
    a->seed += 0x1234567;
    switch (a->sec) {
        case 1: gather<1><<<a->grid, 256>>>(a->tab, a->n_rows, a->row_elems, a->n, a->seed, a->out); break;
        case 2: gather<2><<<a->grid, 256>>>(a->tab, a->n_rows, a->row_elems, a->n, a->seed, a->out); break;
        case 4: gather<4><<<a->grid, 256>>>(a->tab, a->n_rows, a->row_elems, a->n, a->seed, a->out); break;
        default: gather<8><<<a->grid, 256>>>(a->tab, a->n_rows, a->row_elems, a->n, a->seed, a->out); break;
    }
}

}  // namespace

extern "C" double mb_stream_read(uint64_t bytes, int iters) {
    double *p = nullptr, *out = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess || cudaMalloc(&out, 64) != cudaSuccess) return -1;
    cudaMemset(p, 0, bytes);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    SArg a{p, bytes / 32, out, nsm * 8};
    float ms = time_it(launch_stream, &a, iters);
    cudaFree(p);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? ms : -1;
}

extern "C" double mb_gather(uint64_t table_bytes, uint32_t row_bytes, uint64_t n_gathers, int iters) {
    double *tab = nullptr, *out = nullptr;
    if (cudaMalloc(&tab, table_bytes + 4096) != cudaSuccess || cudaMalloc(&out, 64) != cudaSuccess) return -1;
    cudaMemset(tab, 0, table_bytes);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    GArg a{tab, (uint32_t)(table_bytes / row_bytes), row_bytes / 8, n_gathers, 1u, out, nsm * 8, (int)(row_bytes / 32)};
    float ms = time_it(launch_gather, &a, iters);
    cudaFree(tab);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? ms : -1;
}

// ---------------------------------------------------------------------------
// TMA tile::gather4 gather ceiling: each warp owns NSTG smem stages of 32 rows;
// lanes 0..7 each issue one gather4 (4 hashed rows) per stage; completion via
// one mbarrier per stage (complete_tx).  Measures rows/s the TMA engine can
// gather from a `table_bytes` table with `row_bytes` rows.
#include <cuda.h>

namespace {
constexpr int MB_WARPS = 8, MB_NSTG = 6;

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

__global__ void __launch_bounds__(MB_WARPS * 32, 1) tma_gather_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                       uint32_t n_rows, uint32_t row_bytes,
                                                                       uint64_t steps_per_warp, uint32_t seed,
                                                                       double* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bars[MB_WARPS][MB_NSTG];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t stage_bytes = 32 * row_bytes;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + w * MB_NSTG * stage_bytes;
    if (lane == 0)
        for (int s = 0; s < MB_NSTG; ++s) mbar_init((uint32_t)__cvta_generic_to_shared(&bars[w][s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    double acc = 0;
    const uint64_t gwarp = (uint64_t)blockIdx.x * MB_WARPS + w;
    auto issue = [&](uint64_t step, int s) {
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&bars[w][s]);
        uint32_t r = hash32((gwarp * steps_per_warp + step) * 32 + lane + seed) % n_rows;
        uint32_t r0 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4 + 0);
        uint32_t r1 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4 + 1);
        uint32_t r2 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4 + 2);
        uint32_t r3 = __shfl_sync(0xffffffffu, r, (lane & 7) * 4 + 3);
        if (lane == 0) mbar_expect_tx(bar, stage_bytes);
        __syncwarp();
        if (lane < 8) {
            const uint32_t dst = base + s * stage_bytes + lane * 4 * row_bytes;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst), "l"(&tmap), "r"(bar), "r"(0), "r"(r0),
                "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
    };
    for (int s = 0; s < MB_NSTG - 1 && s < (int)steps_per_warp; ++s) issue(s, s);
    for (uint64_t step = 0; step < steps_per_warp; ++step) {
        const int s = (int)(step % MB_NSTG);
        if (step + MB_NSTG - 1 < steps_per_warp) issue(step + MB_NSTG - 1, (int)((step + MB_NSTG - 1) % MB_NSTG));
        mbar_wait((uint32_t)__cvta_generic_to_shared(&bars[w][s]), (uint32_t)((step / MB_NSTG) & 1));
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(base + s * stage_bytes + lane * row_bytes));
        acc += v;
        __syncwarp();
    }
    if (acc == 123.456) out[0] = acc;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
struct TArg { CUtensorMap tm; uint32_t n_rows, row_bytes; uint64_t spw; uint32_t seed; double* out; int grid; int smem; };
void launch_tma(void* v) {
    TArg* a = (TArg*)v;
    a->seed += 0x9e3779;
    tma_gather_kernel<<<a->grid, MB_WARPS * 32, a->smem>>>(a->tm, a->n_rows, a->row_bytes, a->spw, a->seed, a->out);
}
}  // namespace

extern "C" double mb_tma_gather(uint64_t table_bytes, uint32_t row_bytes, uint64_t n_gathers, int iters) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return -2;
    double *tab = nullptr, *out = nullptr;
    if (cudaMalloc(&tab, table_bytes + 4096) != cudaSuccess || cudaMalloc(&out, 64) != cudaSuccess) return -1;
    cudaMemset(tab, 0, table_bytes);
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    TArg a{};
    a.n_rows = (uint32_t)(table_bytes / row_bytes);
    a.row_bytes = row_bytes;
    cuuint64_t gdim[2] = {row_bytes / 8, a.n_rows};
    cuuint64_t gstr[1] = {row_bytes};
    cuuint32_t box[2] = {row_bytes / 8, 1};
    cuuint32_t est[2] = {1, 1};
    CUresult r = ((EncodeTiledFn)fn)(&a.tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, tab, gdim, gstr, box, est,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return -3 - (double)r;
    a.grid = nsm;
    a.spw = n_gathers / 32 / ((uint64_t)nsm * MB_WARPS);
    a.smem = MB_WARPS * MB_NSTG * 32 * row_bytes;
    a.seed = 7;
    a.out = out;
    cudaFuncSetAttribute(tma_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem);
    float ms = time_it(launch_tma, &a, iters);
    cudaError_t e = cudaGetLastError();
    cudaFree(tab);
    cudaFree(out);
    if (e != cudaSuccess) return -100 - (double)e;
    // report ms scaled to n_gathers rows
    return ms * (double)n_gathers / (double)(a.spw * 32 * (uint64_t)nsm * MB_WARPS);
}

// ---------------------------------------------------------------------------
// Random 4-B lookups into a 256 KB bit table (the row-occupancy bitmap of a
// 2M-event catalogue): (a) global memory (L1/L2 gather path, what the ARA
// kernel does per event), (b) a CTA-local shared-memory table (ceiling), (c)
// the table split over the shared memory of a thread-block cluster of K CTAs,
// remote parts read through distributed shared memory.
namespace {
__global__ void lookup_global(const uint32_t* __restrict__ tab, uint32_t words, uint64_t n, uint32_t seed,
                              uint32_t* out) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += 8ull * gridDim.x * blockDim.x) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t w = hash32((i + (uint64_t)k * gridDim.x * blockDim.x) * 0x9E3779B97F4A7C15ULL + seed) % words;
            v[k] = __ldg(tab + w);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void lookup_smem(uint32_t words, uint64_t n, uint32_t seed, uint32_t* out) {
    extern __shared__ uint32_t st[];
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) st[i] = hash32(i);
    __syncthreads();
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += 8ull * gridDim.x * blockDim.x) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t w = hash32((i + (uint64_t)k * gridDim.x * blockDim.x) * 0x9E3779B97F4A7C15ULL + seed) % words;
            v[k] = st[w];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k];
    }
    if (acc == 0x12345678u) out[0] = acc;
}

__global__ void lookup_dsmem(uint32_t words_per_cta, uint64_t n, uint32_t seed, uint32_t* out) {
    extern __shared__ uint32_t st[];
    cg::cluster_group cluster = cg::this_cluster();
    const uint32_t K = cluster.num_blocks();
    for (uint32_t i = threadIdx.x; i < words_per_cta; i += blockDim.x) st[i] = hash32(i + cluster.block_rank());
    cluster.sync();
    uint32_t acc = 0;
    const uint32_t words = words_per_cta * K;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += 8ull * gridDim.x * blockDim.x) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t w = hash32((i + (uint64_t)k * gridDim.x * blockDim.x) * 0x9E3779B97F4A7C15ULL + seed) % words;
            const uint32_t* rp = cluster.map_shared_rank(st, w / words_per_cta);
            v[k] = rp[w % words_per_cta];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc ^= v[k];
    }
    cluster.sync();   // no CTA leaves while others still read its table
    if (acc == 0x12345678u) out[0] = acc;
}
}  // namespace

extern "C" double mb_lookup(int mode, uint32_t table_bytes, int cluster, uint64_t n, int iters) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    uint32_t* out = nullptr;
    uint32_t* tab = nullptr;
    cudaMalloc(&out, 4);
    const uint32_t words = table_bytes / 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = -1.f;
    if (mode == 0) {
        cudaMalloc(&tab, table_bytes);
        cudaMemset(tab, 1, table_bytes);
        lookup_global<<<nsm * 4, 512>>>(tab, words, n, 1, out);
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) lookup_global<<<nsm * 4, 512>>>(tab, words, n, 2 + i, out);
        cudaEventRecord(b);
    } else if (mode == 1) {
        cudaFuncSetAttribute(lookup_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)table_bytes);
        lookup_smem<<<nsm, 1024, table_bytes>>>(words, n, 1, out);
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) lookup_smem<<<nsm, 1024, table_bytes>>>(words, n, 2 + i, out);
        cudaEventRecord(b);
    } else {
        const uint32_t per = table_bytes / cluster;
        cudaFuncSetAttribute(lookup_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)per);
        cudaFuncSetAttribute(lookup_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((nsm / cluster) * cluster);
        cfg.blockDim = dim3(1024);
        cfg.dynamicSmemBytes = per;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cluster;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, lookup_dsmem, per / 4, n, 1u, out);
        cudaEventRecord(a);
        for (int i = 0; i < iters; ++i) cudaLaunchKernelEx(&cfg, lookup_dsmem, per / 4, n, (uint32_t)(2 + i), out);
        cudaEventRecord(b);
    }
    if (cudaEventSynchronize(b) == cudaSuccess) cudaEventElapsedTime(&ms, a, b);
    if (cudaGetLastError() != cudaSuccess) ms = -1.f;
    cudaFree(out);
    cudaFree(tab);
    return ms < 0 ? -1.0 : ms / iters;
}
