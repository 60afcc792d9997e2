// densify.cu — ELT ingest into the interleaved direct-access table (§8a row a0).
//
// "ELTs corresponding to a Layer were implemented as direct
// access tables ... Each ELT is implemented as an independent table".  On B200
// the tables are interleaved instead: within a column block tab[e][j] holds
// ELT j's loss for event e, so the E losses one event needs are one
// contiguous row (one 128-B line for 16 fp64 ELTs) rather than E scattered
// sectors (geometry: ara::TableGeo).  Row 0 stays zero (event
// ids are 1-based, reading A14); a missing (event, ELT) pair reads 0 (A4).
//
// The table (and its row-occupancy bitmaps) was zero-filled by
// cudaMemsetAsync; this kernel scatters the sparse records, marks their rows in
// the bitmap of their column block, and validates them (fused, error bits).
#include <cfloat>
#include <cstring>
#include <type_traits>

#include "ara_internal.cuh"

namespace ara {
namespace {

template <typename TV>
__global__ void __launch_bounds__(256) densify_kernel(const uint64_t* __restrict__ eoff,
                                                      const uint32_t* __restrict__ ev,
                                                      const double* __restrict__ loss,
                                                      uint32_t catalog, TV* __restrict__ tab,
                                                      uint32_t epb, uint64_t block_elems, uint32_t* __restrict__ bm,
                                                      uint64_t bm_words, uint32_t* __restrict__ occ, uint32_t* err) {
    const uint32_t j = blockIdx.y;
    const uint64_t lo = eoff[j], hi = eoff[j + 1];
    uint32_t bad = 0;
    for (uint64_t k = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < hi;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t e = ev[k];
        const double x = loss[k];
        bool newrow = false;
        if (e == 0u || e > catalog) {
            bad |= ERRBIT_ELT_RANGE;
        } else {
            if (k > lo && ev[k - 1] >= e) bad |= ERRBIT_ELT_ORDER;
            if (!(x >= 0.0) || !(x <= DBL_MAX) || (sizeof(TV) == 4 && x > (double)FLT_MAX)) {
                bad |= ERRBIT_ELT_LOSS;
            } else {
                tab[(uint64_t)(j / epb) * block_elems + (uint64_t)e * epb + j % epb] = (TV)(x + 0.0);   // canonical +0 (A16)
                const uint32_t bit = 1u << (e & 31u);   // row e of column block j / epb is occupied
                newrow = !(atomicOr(bm + (uint64_t)(j / epb) * bm_words + (e >> 5), bit) & bit);
            }
        }
        // the block's occupied-row counter: one atomic per warp (j is uniform in the block)
        const uint32_t am = __activemask();
        const uint32_t nm = __ballot_sync(am, newrow);
        if (nm && (threadIdx.x & 31u) == (uint32_t)(__ffs(am) - 1)) atomicAdd(occ + j / epb, (uint32_t)__popc(nm));
    }
    if (bad) atomicOr(err, bad);
}

// Reload without the full-table memset: every non-zero element of the table
// lies in a row whose occupancy bit is set (densify sets the bit with every
// store), so zeroing exactly those rows -- ~15 % of the rows at the paper's ELT
// density, 38 MB instead of 256 MB -- restores an all-zero table.  One warp per
// 8 bitmap words, one lane per row; the caller then clears the bitmaps and counters.
__global__ void __launch_bounds__(256) clear_rows_kernel(unsigned char* __restrict__ tab, const uint32_t* __restrict__ bm,
                                                         uint64_t bm_words, uint32_t n_blocks, uint32_t catalog,
                                                         uint32_t row_bytes, uint64_t block_bytes) {
    // one warp per 8 consecutive bitmap words (loaded first, independently),
    // lane l clears row 32 * word + l of each word when its bit is set
    constexpr int WPW = 8;
    const uint64_t n = (uint64_t)n_blocks * bm_words;
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t i0 = ((uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5)) * WPW; i0 < n; i0 += nw * WPW) {
        uint32_t w[WPW];
#pragma unroll
        for (int k = 0; k < WPW; ++k) w[k] = i0 + k < n ? __ldg(bm + i0 + k) : 0u;
#pragma unroll
        for (int k = 0; k < WPW; ++k) {
            const uint64_t i = i0 + k;
            const uint64_t b = i / bm_words, e = (i % bm_words) * 32 + lane;
            if (!((w[k] >> lane) & 1u) || e > catalog) continue;
            uint4* row = reinterpret_cast<uint4*>(tab + b * block_bytes + e * row_bytes);
            for (uint32_t c = 0; c < row_bytes / 16; ++c) row[c] = make_uint4(0, 0, 0, 0);
        }
    }
}

// Packed rows of the sparse column blocks.  On the paper's ELTs an occupied
// row of a 16-ELT block holds one non-zero loss in ~93 % of cases (rho = 0.01,
// P:237), yet a full-row gather moves 4 sectors; the packed slot moves 1.
// Slot e: u32 mask (bit c = column c of the block is non-zero, bitwise, the
// test the sparse arithmetic uses), u32 e, then the first 24 / esz non-zero
// values in column order; a row with more non-zeros keeps the rest in the
// dense table, where the kernel reads them.  Written for the occupied rows
// only (the kernels read slot e only when bit e of the bitmap is set).  One
// thread per bitmap word; blockIdx.y = column block, skipped when dense.
template <typename TV>
__global__ void __launch_bounds__(256) pack_rows_kernel(const unsigned char* __restrict__ tab,
                                                        const uint32_t* __restrict__ bm, uint64_t bm_words,
                                                        const uint32_t* __restrict__ occ, uint32_t n_blocks,
                                                        uint32_t catalog, uint32_t epb,
                                                        uint64_t block_bytes, unsigned char* __restrict__ pk) {
    // one thread per row: the bitmap word is a warp broadcast, an occupied
    // row is read with independent 16-B loads
    constexpr int CAP = (kPackBytes - 8) / (int)sizeof(TV);
    constexpr int EPC = 16 / (int)sizeof(TV);   // elements per 16-B chunk
    using UT = typename std::conditional<sizeof(TV) == 8, unsigned long long, uint32_t>::type;
    const uint32_t nchunk = epb * (uint32_t)sizeof(TV) / 16u;   // 2 .. 8 (rows are 32-B multiples)
    for (uint32_t b = blockIdx.y; b < n_blocks; b += gridDim.y) {
        if (2ull * occ[b] > (uint64_t)catalog + 1) continue;   // dense block: not packed (host rule, ara_run)
        for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e <= catalog;
             e += (uint64_t)gridDim.x * blockDim.x) {
            if (!((__ldg(bm + b * bm_words + (e >> 5)) >> (e & 31u)) & 1u)) continue;
            const uint4* row = reinterpret_cast<const uint4*>(tab + b * block_bytes + e * epb * sizeof(TV));
            uint4 ch[kBlockBytes / 16];
#pragma unroll
            for (int q = 0; q < kBlockBytes / 16; ++q) ch[q] = (uint32_t)q < nchunk ? __ldg(row + q) : make_uint4(0, 0, 0, 0);
            uint32_t mask = 0, n = 0;
            UT v[CAP];
#pragma unroll
            for (int k = 0; k < CAP; ++k) v[k] = 0;
#pragma unroll
            for (int q = 0; q < kBlockBytes / 16; ++q) {
                UT x[EPC];
                memcpy(x, &ch[q], 16);
#pragma unroll
                for (int h = 0; h < EPC; ++h) {
                    if (x[h] == 0) continue;
                    mask |= 1u << (q * EPC + h);
#pragma unroll
                    for (int k = 0; k < CAP; ++k) v[k] = (n == (uint32_t)k) ? x[h] : v[k];
                    ++n;
                }
            }
            uint32_t out[kPackBytes / 4];
            out[0] = mask;
            out[1] = (uint32_t)e;
            memcpy(&out[2], v, sizeof(v));
            uint4* dst = reinterpret_cast<uint4*>(pk + ((uint64_t)b * ((uint64_t)catalog + 1) + e) * kPackBytes);
            dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
            dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
        }
    }
}

// Packed YET ids (F3): id i at bit offset i*bits of a u32 word stream.
__global__ void __launch_bounds__(256) unpack_kernel(const uint32_t* __restrict__ packed, uint32_t bits,
                                                     uint64_t e0, uint64_t e1, uint32_t* __restrict__ ids) {
    const uint64_t mask = bits >= 32 ? 0xffffffffull : ((1ull << bits) - 1);
    for (uint64_t i = e0 + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < e1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = i * bits;
        const uint64_t w = b >> 5;
        const uint64_t v = (uint64_t)__ldg(packed + w) | ((uint64_t)__ldg(packed + w + 1) << 32);
        ids[i] = (uint32_t)((v >> (b & 31)) & mask);
    }
}

}  // namespace

cudaError_t launch_pack_rows(void* d_table, const TableGeo& geo, uint32_t catalog, int fp32, cudaStream_t s) {
    if (!geo.n_blocks) return cudaSuccess;
    unsigned char* t = static_cast<unsigned char*>(d_table);
    const uint32_t* bm = reinterpret_cast<const uint32_t*>(t + geo.bm_off);
    const uint32_t* occ = reinterpret_cast<const uint32_t*>(t + geo.occ_off);
    uint64_t bx = ((uint64_t)catalog + 1 + 255) / 256;   // one thread per row (latency-bound row reads)
    if (bx > 65535) bx = 65535;
    const dim3 grid((unsigned)bx, geo.n_blocks < 65535u ? geo.n_blocks : 65535u);
    const uint64_t block_bytes = geo.block_elems * geo.esz;
    if (fp32)
        pack_rows_kernel<float><<<grid, 256, 0, s>>>(t, bm, geo.bm_words, occ, geo.n_blocks, catalog, geo.epb, block_bytes, t + geo.pk_off);
    else
        pack_rows_kernel<double><<<grid, 256, 0, s>>>(t, bm, geo.bm_words, occ, geo.n_blocks, catalog, geo.epb, block_bytes, t + geo.pk_off);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const uint32_t* packed, uint32_t bits, uint64_t e0, uint64_t e1, uint32_t* ids,
                          cudaStream_t s) {
    if (e1 <= e0) return cudaSuccess;
    uint64_t blocks = (e1 - e0 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    unpack_kernel<<<(unsigned)blocks, 256, 0, s>>>(packed, bits, e0, e1, ids);
    return cudaGetLastError();
}

cudaError_t launch_clear_rows(void* d_table, const TableGeo& geo, uint32_t catalog, cudaStream_t s) {
    const uint64_t n = (uint64_t)geo.n_blocks * geo.bm_words;   // 8 bitmap words per warp
    uint64_t blocks = (n + 63) / 64;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    clear_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(static_cast<unsigned char*>(d_table),
                                                       reinterpret_cast<const uint32_t*>(static_cast<char*>(d_table) + geo.bm_off),
                                                       geo.bm_words, geo.n_blocks, catalog, geo.epb * geo.esz,
                                                       geo.block_elems * geo.esz);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // bitmaps and occupied-row counters (not the packed slots: written before they are read)
    return cudaMemsetAsync(static_cast<char*>(d_table) + geo.bm_off, 0, geo.pk_off - geo.bm_off, s);
}

cudaError_t launch_densify(const uint64_t* d_eoff, const uint32_t* d_ev, const double* d_loss,
                           uint32_t n_elts, uint64_t n_records, uint32_t catalog, void* d_table,
                           const TableGeo& geo, int fp32, uint32_t* d_err, cudaStream_t s) {
    if (n_records == 0) return cudaSuccess;
    uint64_t per = (n_records + n_elts - 1) / n_elts;
    uint64_t bx = (per + 255) / 256;
    if (bx > 1024) bx = 1024;
    if (bx < 1) bx = 1;
    dim3 grid((unsigned)bx, n_elts);
    uint32_t* bm = reinterpret_cast<uint32_t*>(static_cast<char*>(d_table) + geo.bm_off);
    uint32_t* occ = reinterpret_cast<uint32_t*>(static_cast<char*>(d_table) + geo.occ_off);
    if (fp32)
        densify_kernel<float><<<grid, 256, 0, s>>>(d_eoff, d_ev, d_loss, catalog, static_cast<float*>(d_table),
                                                   geo.epb, geo.block_elems, bm, geo.bm_words, occ, d_err);
    else
        densify_kernel<double><<<grid, 256, 0, s>>>(d_eoff, d_ev, d_loss, catalog, static_cast<double*>(d_table),
                                                    geo.epb, geo.block_elems, bm, geo.bm_words, occ, d_err);
    return cudaGetLastError();
}

}  // namespace ara
