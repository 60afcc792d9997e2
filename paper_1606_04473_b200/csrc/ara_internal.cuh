// ara_internal.cuh — shared declarations of the B200 ARA library (product path).
// Nothing here is shared with oracle/ (the CPU oracle is independent test
// infrastructure); this header is private to paper_1606_04473_b200/csrc.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "ara.h"

namespace ara {

// ---- device error bits (fused validation, reported by the host after sync)
enum : uint32_t {
    ERRBIT_EVENT_RANGE = 1u << 0,   // YET event id outside [1, C]
    ERRBIT_OFFSETS = 1u << 1,       // YET trial offsets decreasing
    ERRBIT_ELT_RANGE = 1u << 2,     // ELT event id outside [1, C]
    ERRBIT_ELT_ORDER = 1u << 3,     // ELT ids not strictly ascending (duplicate)
    ERRBIT_ELT_LOSS = 1u << 4,      // ELT loss negative / non-finite / fp32-unrepresentable
};

constexpr int kSectorBytes = 32;     // one L2 sector; windows are sector-granular
constexpr int kBlockBytes = 128;     // column-block width of the direct-access table
constexpr int kMaxSec = 8;           // widest per-layer window handled by the fast kernel (256 B)
constexpr int kMaxLB = 4;            // layers sharing one window per launch
constexpr int kMaxFoldL = 8;         // layers per folded trial launch (fold mode)
constexpr int kMaxWin = kMaxSec * kSectorBytes / 4;   // 64 columns (fp32) per window
constexpr int kThreads = 256;        // 8 warps per CTA
constexpr int kTablePadBytes = kMaxSec * kSectorBytes;  // over-read slack after the last row
constexpr int kPackBytes = 32;       // packed row: u32 mask, u32 event id, 24 B of values
constexpr int kMaxPeers = 8;         // ranks whose global YLT a kernel epilogue writes over NVLink

// Direct-access table geometry: ELT columns are cut
// into blocks of `epb` elements (<= 128 B); block b is a dense [C+1][epb]
// array, so element (event e, ELT j) lives at
//   (j / epb) * block_elems + e * epb + j % epb.
// A layer of <= 16 fp64 ELTs therefore reads one contiguous 32..128-B row
// window per event, and each block spans at most (C+1) * 128 B (256 MB at the
// paper's 2M-event catalogue), inside the GPU TLB's reach.
struct TableGeo {
    uint32_t esz = 8;            // element bytes (8 fp64, 4 fp32-storage)
    uint32_t epb = 0;            // elements per block row
    uint32_t n_blocks = 0;
    uint64_t block_elems = 0;    // (C+1) * epb
    uint64_t bm_words = 0;       // row-occupancy bitmap words per block (ceil((C+2)/32), padded)
    size_t bm_off = 0;           // byte offset of the bitmaps in the allocation
    size_t occ_off = 0;          // byte offset of the per-block occupied-row counters (u32)
    size_t pk_off = 0;           // byte offset of the packed-row slots (kPackBytes per event per block)
    size_t bytes = 0;            // allocation incl. pad, bitmaps and packed slots
};
inline TableGeo table_geometry(uint32_t n_elts, uint32_t catalog, int fp32) {
    TableGeo g;
    g.esz = fp32 ? 4 : 8;
    uint64_t row = (uint64_t)n_elts * g.esz;
    row = (row + kSectorBytes - 1) / kSectorBytes * kSectorBytes;
    if (row > (uint64_t)kBlockBytes) row = kBlockBytes;
    g.epb = (uint32_t)(row / g.esz);
    g.n_blocks = (n_elts + g.epb - 1) / g.epb;
    g.block_elems = ((uint64_t)catalog + 1) * g.epb;
    // Row-occupancy bitmap per column block: bit e of block b is set when ELT
    // record (e, j) exists for some column j of the block.  A clear bit means
    // the row is all zeros, so its lookup can be skipped (a zero row adds an
    // exact +0 to every sum: every deductible and retention is >= 0).
    // bits 0 .. C + 1: bit C + 1 is padding that is never set (the sparse
    // trial kernel clamps out-of-range ids to C + 1)
    g.bm_words = (((uint64_t)catalog + 2 + 31) / 32 + 63) / 64 * 64;
    g.bm_off = ((size_t)g.n_blocks * g.block_elems * g.esz + kTablePadBytes + 255) / 256 * 256;
    g.occ_off = g.bm_off + (size_t)g.n_blocks * g.bm_words * 4;
    // Packed rows of the sparse blocks (one 32-B sector per event, written for
    // the occupied rows only, never zero-filled): the row's non-zero mask, its
    // event id and its first non-zero values in column order (PackedRow below).
    g.pk_off = g.occ_off + ((size_t)g.n_blocks * 4 + 255) / 256 * 256;
    g.bytes = g.pk_off + (size_t)g.n_blocks * ((size_t)catalog + 1) * kPackBytes;
    return g;
}

// Layer terms of one launch (P:373 occurrence, P:375 aggregate).
struct LayerWin {
    double occ_r, occ_l, agg_r, agg_l;
};

// All layers of one launch share one sector window: sec_off[s] is the element
// offset of window sector s for event 0 (event e adds e * row_stride).  Window
// columns outside a layer carry deductible +inf, so they contribute an exact
// +0 and need no predicate.  Passed by value (constant bank).
struct TrialParams {
    const uint64_t* off;        // local CSR offsets [n_local + 1]
    const uint32_t* ids;        // events of off[0] ...
    uint64_t t_begin, t_end;    // trial range of this launch (local indices)
    uint32_t catalog;
    uint32_t n_layers;          // layers in this launch (<= kMaxLB)
    const void* table;          // column-blocked direct-access table (+ pad)
    const uint32_t* bm;         // row-occupancy bitmap of the window's (sparse) column block, or null
    uint64_t row_stride;        // elements per block row (= epb)
    uint64_t block_stride;      // elements per column block (= (C+1) * epb)
    uint64_t sec_off[kMaxSec];  // window sector offsets (elements, event 0)
    double* ylt;                // [.. rows][ld] : row ylt_row0 + l
    uint64_t ld;                // row stride of ylt (= n_local)
    uint32_t ylt_row0;          // first YLT row written by this launch
    int portfolio_mode;         // 0: write portfolio row, 1: add to it, -1: none
    uint32_t portfolio_row;
    uint32_t* lossy;            // [.. rows][ld] or null
    uint32_t* err;              // device error word
    unsigned long long* n_gathered;   // trial_kernel_bc: packed slots gathered (added per warp), or null
    double* fold;               // fold mode: per-event occurrence-net losses, [C+1][fold_stride] per chunk
    uint32_t fold_stride;       // doubles per fold row (layers of one chunk, power of two <= 8)
    uint32_t fold_col0;         // fold column of the launch's first layer
    LayerWin lw[kMaxFoldL];
    double2 term[kMaxLB][kMaxWin];   // (deductible, limit) per window column
    // fused YLT assembly (world > 1): every rank's global YLT [rows][peer_ld],
    // mapped into this process (CUDA IPC over NVLink); 0 peers = not used
    double* peer_ylt[kMaxPeers];
    uint32_t n_peers;
    // packed rows of the window's (sparse) column block, or null: slot e holds
    // row e's non-zero mask over the block's columns, e, and its first
    // 24 / esz non-zero values in column order; the window is block columns
    // pk_col0 .. (pk_wmask's bits), i.e. window element j = block column pk_col0 + j
    const void* pk;
    uint32_t pk_col0, pk_wmask;
    uint32_t same_terms;        // every layer of the launch has layer 0's per-ELT terms (a tower over one ELT set)
    uint64_t peer_ld;           // = T_global
    uint64_t peer_t0;           // global index of local trial 0 (this rank's first trial)
    uint32_t bm_smem_words;     // trial_kernel_bc: leading bitmap words staged in shared memory (set by the launcher)
};

// ---- launchers (defined in the .cu files; all enqueue on `s`)
cudaError_t launch_densify(const uint64_t* d_eoff, const uint32_t* d_ev, const double* d_loss,
                           uint32_t n_elts, uint64_t n_records, uint32_t catalog, void* d_table,
                           const TableGeo& geo, int fp32, uint32_t* d_err, cudaStream_t s);

// packed rows (TrialParams::pk) of every sparse column block (<= half its rows occupied)
cudaError_t launch_pack_rows(void* d_table, const TableGeo& geo, uint32_t catalog, int fp32, cudaStream_t s);
// zero exactly the rows the occupancy bitmaps mark, then the bitmaps and counters
cudaError_t launch_clear_rows(void* d_table, const TableGeo& geo, uint32_t catalog, cudaStream_t s);
cudaError_t launch_trials(const TrialParams& p, int fp32, uint32_t max_nsec, int grid, int variant, cudaStream_t s);
// trial_kernel_bc (kernel_sparse.cu): needs p.bm and p.pk; grid = one CTA per SM
cudaError_t launch_trials_bc(const TrialParams& p, int fp32, int grid, cudaStream_t s);
int trial_kernel_grid(int fp32, uint32_t max_nsec, int n_layers, int variant);
cudaError_t launch_fold(const TrialParams& p, int fp32, uint32_t nsec, cudaStream_t s);
cudaError_t launch_unpack(const uint32_t* packed, uint32_t bits, uint64_t e0, uint64_t e1, uint32_t* ids,
                          cudaStream_t s);
cudaError_t launch_trials_folded(const TrialParams& p, int grid_mult_x100, cudaStream_t s);
cudaError_t launch_trials_wide(const TrialParams& p, int fp32, const uint32_t* d_cols, const double2* d_cterm,
                               uint32_t ncol, int grid, cudaStream_t s);
cudaError_t launch_program_sums(double* ylt, uint64_t ld, uint64_t t_local, uint32_t n_programs,
                                const uint32_t* d_program_layers, uint32_t n_layers, cudaStream_t s);

// EP curve (ep_curve.cu): counts[row][i] = #{t < T : ylt[row * ld + t] > x[i]}, x non-decreasing
cudaError_t launch_ep_curve(const double* d_ylt, uint64_t T, uint64_t ld, uint32_t rows, const double* d_x,
                            uint32_t n, unsigned long long* d_hist, uint64_t* d_counts, int n_sm, cudaStream_t s);

// metrics: radix select over the [rows][T] YLT (device), fixed-order tail sums
struct MetricsScratch {
    uint32_t* hist8 = nullptr;      // [8][rows * n_rp][256] per-pass histograms
    uint64_t* st = nullptr;         // [2][rows * n_rp][2] prefix / remaining rank, double-buffered
    uint32_t* strep = nullptr;      // [2][rows * n_rp] histogram slots
    double* part_sum = nullptr;     // [rows][n_rp][nblk] tail-sum partials per block
    uint64_t* part_cnt = nullptr;
    double* out = nullptr;          // [rows][n_rp][2] pml, tvar
    uint32_t* done = nullptr;       // [rows] block-completion counters
    double* dsum = nullptr;         // distributed select: tail sums / counts per (row, period)
    uint64_t* dcnt = nullptr;
    uint64_t* cand = nullptr;       // candidate keys per warp region (fast path)
    uint32_t* cand_n = nullptr;
    double* bsum = nullptr;         // slot partial sums / counts per block (fast path)
    uint64_t* bcnt = nullptr;
    uint64_t cand_cap = 0, cand_n_cap = 0, bpart_cap = 0;
    // the fast path's launch sequences, keyed by their arguments: two entries,
    // because consecutive multi-GPU runs alternate between two global-YLT buffers
    cudaGraphExec_t m4_exec[2] = {nullptr, nullptr};
    unsigned char m4_key[2][1024] = {};
    int m4_next = 0;                     // the entry a new capture replaces
    size_t cap_rows_rp = 0;
    uint32_t cap_rows = 0;
    int nblk = 0;                   // capacity in blocks
};
cudaError_t metrics_alloc(MetricsScratch& m, uint32_t rows, uint32_t n_rp, int nblk);
void metrics_free(MetricsScratch& m);
cudaError_t launch_metrics(const double* d_ylt, uint64_t T, uint64_t ld, uint32_t rows,
                           uint32_t n_rp, const uint64_t* h_k, MetricsScratch& m, int nblk, cudaStream_t s);
// Distributed select: each rank histograms its own YLT shard
// [rows][T_local] (row stride ld); the per-pass histograms and the tail sums are
// all-reduced over `comm`, so every rank derives the same global PML/TVaR
// without the global YLT.  *nccl_err is set when an NCCL call failed.
cudaError_t launch_metrics_dist(const double* d_ylt, uint64_t T_local, uint64_t ld, uint32_t rows, uint32_t n_rp,
                                const uint64_t* h_k, MetricsScratch& m, int nblk, ncclComm_t comm,
                                cudaStream_t s, int* nccl_err);

}  // namespace ara

// ---- the opaque context
struct ara_ctx {
    int device = 0, rank = 0, world = 1;
    ara_precision precision = ARA_F64;
    ara_load_mode load_mode = ARA_LOAD_ALL_AT_ONCE;
    uint64_t chunk_trials = 65536;
    int l2_persist = 0;
    cudaStream_t stream = nullptr, copy_stream = nullptr;
    bool own_stream = false;
    ncclComm_t comm = nullptr;
    int n_sm = 148;
    std::string last_error;

    uint32_t catalog = 0;

    // ELT direct-access table (column-blocked, ara::TableGeo), row 0 = zeros
    void* d_table = nullptr;
    size_t table_bytes = 0;
    ara::TableGeo geo;
    uint32_t n_elts = 0;
    uint64_t* d_sp_off = nullptr;      // sparse ELT staging (host uploads / NVLink broadcast)
    uint32_t* d_sp_ev = nullptr;
    double* d_sp_ls = nullptr;
    size_t sp_off_cap = 0, sp_ev_cap = 0, sp_ls_cap = 0;
    std::vector<ara_elt_terms> terms;

    // YET (local shard)
    bool yet_loaded = false;
    uint64_t T_global = 0, first = 0, T_local = 0;
    const uint64_t* d_off = nullptr;   // current device offsets (owned or borrowed)
    const uint32_t* d_ids = nullptr;
    uint64_t* d_off_own = nullptr;
    uint32_t* d_ids_own = nullptr;
    size_t own_off_cap = 0, own_ids_cap = 0;
    const uint64_t* h_off = nullptr;   // CHUNKED host source
    const uint32_t* h_ids = nullptr;
    void* h_registered = nullptr;      // host range we cudaHostRegister'ed
    bool chunked_pending = false;
    uint32_t pack_bits = 0;            // > 0: the YET ids arrive bit-packed (ara_load_yet_packed)
    const uint32_t* h_packed = nullptr;
    uint32_t* d_packed_own = nullptr;
    size_t packed_cap = 0;
    uint64_t n_events_host = 0;        // known when offsets were host memory
    bool tiling_checked = false;

    // YLT
    uint32_t last_layers = 0;          // layers of the last run (0 = none)
    uint32_t last_rows = 0;            // YLT rows of the last run (layers + programs + portfolio)
    double* d_ylt_local = nullptr;     // [(L+1)][T_local]
    size_t ylt_local_cap = 0;
    double* d_ylt_gather = nullptr;    // world>1: [(L+1)][world][Tpad]
    double* d_ylt_global = nullptr;    // world>1: [(L+1)][T_global]
    size_t ylt_global_cap = 0, ylt_gather_cap = 0;
    uint32_t* d_lossy = nullptr;
    size_t lossy_cap = 0;

    // status / small pinned block
    uint32_t* d_err = nullptr;
    uint64_t* h_small = nullptr;       // pinned: [0]=err, [1]=off0, [2]=offN, ...
    uint64_t* d_small = nullptr;

    ara::MetricsScratch ms;
    // fused YLT assembly over NVLink (world > 1): two global-YLT buffers used
    // alternately by consecutive runs (a run's peer stores cannot overwrite a
    // buffer another rank is still reading: the error all-reduce that closes
    // every run orders them), their IPC mappings on every rank
    double* d_p2p[2] = {nullptr, nullptr};
    double* peer_p2p[2][ara::kMaxPeers] = {};
    size_t p2p_cap = 0;               // doubles per buffer
    int p2p_state = 0;                // 0 unknown, 1 usable, -1 not usable (collective verdict)
    int p2p_next = 0;                 // buffer of the next run
    bool use_p2p = true;              // ARA_NO_P2P=1: assemble the YLT with ncclAllGather instead
    const double* d_last_full = nullptr;   // global YLT of the last run (metrics input)
    uint64_t last_ld_local = 1;       // row stride of d_ylt_local in the last run
    uint64_t run_T_global = 0;        // trials of the last run (global / this rank's): ara_metrics reads
    uint64_t run_T_local = 0;         //   the last run's YLT, whatever ara_load_yet happened since
    int metrics_dist = -1;            // ARA_METRICS_DIST: -1 auto (distributed when T >= 3M), 0 off, 1 on
    // ARA_LOOPBACK="W,r" (test knob, world == 1): this context holds rank r's
    // ara_partition shard of a W-rank job and runs the fused peer-store
    // epilogue into a local global-YLT buffer (peer_t0 = first trial,
    // peer_ld = T_global), so a9's indexing runs on one GPU; its metrics are
    // the distributed select over the shard with an identity reduce
    int lb_world = 0, lb_rank = 0;
    unsigned char* d_ep = nullptr;    // EP-curve scratch: thresholds, histograms, counts
    size_t ep_cap = 0;
    int run_mode = 0;                  // ARA_RUN_DIRECT / ARA_RUN_FOLD
    double* d_fold = nullptr;          // fold mode: per-event occurrence-net losses
    size_t fold_cap = 0;
    // tuning knobs (environment, read at ara_create; not part of the ABI)
    double grid_mult = 1.0;           // ARA_GRID_MULT
    int kernel_variant = -1;          // ARA_KERNEL (-1 auto; see pick_kernel in ara_kernel.cu)
    bool no_skip = false;             // ARA_NO_SKIP=1: never skip zero rows via the occupancy bitmap (A/B)
    bool fold_bc = true;              // fold mode on sparse blocks: the sparse kernel's rounds over o(e) (ARA_FOLD_BC=0: the dense fold pass)
    std::vector<uint32_t> occ_rows;   // occupied rows per column block (from densify)
    bool table_clean = false;         // table content is exactly described by its occupancy bitmaps
    cudaEvent_t ev[8] = {};
};
