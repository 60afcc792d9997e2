// microbench.cu — measured ceilings for the ARA gather:
//   mb_stream_read  : streaming 256-bit read of a large buffer (HBM read BW)
//   mb_gather       : random row gathers of `row_bytes` from a `table_bytes`
//                     table (HBM-sized -> DRAM random-access ceiling; 32 MB ->
//                     L2 gather ceiling), ids hashed on the fly
// Separate library (libara_mb.so); not on the product path.  Each call
// allocates, times `iters` launches with CUDA events, and returns ms/launch.
#include <cuda_runtime.h>
#include <stdint.h>

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
