/*
 * ara.h — C ABI of the B200-native Aggregate Risk Analysis (ARA) hot path.
 *
 * The calls follow the paper's problem statement (PAPER.md = P):
 *   inputs  YET (Eq. 1), ELTs (Eq. 2), layers (Eq. 3)
 *   output  YLT, one loss per trial (Alg. 1)
 *   metrics PML / TVaR at return periods (named P:273; defined DESIGN.md A9/A10)
 *
 *   ara_create     context on one GPU (Alg. 2 "Select device")
 *   ara_load_elts  ELT ingest + densify into a direct-access table   [§8a a0]
 *   ara_load_yet   YET ingest, all-at-once or chunked (Alg. 2)    [§8a a1]
 *   ara_run        Alg. 3 per trial + layer terms -> YLT;
 *                  multi-GPU YLT assembly (Alg. 1 l.9)                [§8a a2-a9]
 *   ara_metrics    PML / TVaR of every layer and of the portfolio            [§8a a10]
 *
 * Conventions shared by every call:
 *   - Every call returns ara_status; nothing throws across the ABI.  On error
 *     the context keeps its previous state and ara_last_error() describes it.
 *   - Pointers may be HOST or DEVICE memory unless stated otherwise; the
 *     library classifies each with cudaPointerGetAttributes.  Device pointers
 *     must live on the context's device.
 *   - The caller owns every input and output buffer.  The library owns the
 *     device ELT table, its scratch, and any device copy it makes of the YET.
 *   - All work is enqueued on the context stream (cfg.stream or a library
 *     stream).  Every call that returns results synchronises that stream
 *     before returning.
 *   - A context is not thread-safe; distinct contexts are independent.
 *   - Multi-GPU (world > 1): one process and one context per GPU.  Calls
 *     marked COLLECTIVE must be made by every rank in the same order.
 *
 * Numerics: fp64 arithmetic, round-to-nearest, no FMA contraction on the
 * term path.  Per event the ELT losses are summed sequentially in the layer's
 * ELT order (so the lossy-occurrence counts are bit-exact against the paper's
 * sequential Alg. 3); per trial the occurrence-net losses are summed in an
 * order fixed by the trial's own events -- lane-strided + warp tree in the
 * dense kernels, the trial's occupied events dealt round-robin to the lanes +
 * warp tree in the sparse kernel -- so results are deterministic and
 * independent of sharding, chunking and alignment, and within the A21 bound
 * (|dY| <= 1e-9 * sum of the trial's event losses) of the sequential sum.
 *
 * Deviations from the SURVEY.md 8(b) sketch (deliberate):
 * lossy-occurrence counts are an ara_run OUTPUT ARGUMENT (host or device
 * buffer, like the YLT) rather than a pointer inside ara_run_stats, so the
 * stats struct is plain data; ara_metrics returns the ranks k[] (host, may be
 * NULL) and the metrics kernels' device time instead of a `ranks` argument
 * after the outputs.  ara_load_yet_packed, ara_set_elt_terms and
 * ara_run_portfolio are additions (F3, P:197 re-pricing, F4).
 */
#ifndef ARA_H
#define ARA_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ARA_ABI_VERSION 1
#define ARA_NCCL_ID_BYTES 128   /* sizeof(ncclUniqueId) */
#define ARA_MAX_LAYERS 64       /* layers per ara_run call */
#define ARA_MAX_RP 64           /* return periods per ara_metrics call */
#define ARA_MAX_PROGRAMS 64     /* programs per ara_run_portfolio call */
#define ARA_MAX_EP_POINTS 4096  /* thresholds per ara_ep_curve call */

typedef struct ara_ctx ara_ctx;

typedef enum {
    ARA_OK = 0,
    ARA_ERR_INVALID_ARG = 1,   /* malformed argument (NULL, sizes, duplicate ids, bad ranges) */
    ARA_ERR_OUT_OF_RANGE = 2,  /* an event id outside [1, catalog_size], or non-monotone offsets */
    ARA_ERR_DOMAIN = 3,        /* a value outside its mathematical domain (loss < 0, R outside [1,T]) */
    ARA_ERR_STATE = 4,         /* call order violated (run before loads, metrics before run) */
    ARA_ERR_OOM = 5,           /* device or pinned allocation failed */
    ARA_ERR_CUDA = 6,          /* CUDA runtime error (message in ara_last_error) */
    ARA_ERR_NCCL = 7           /* NCCL error (message in ara_last_error) */
} ara_status;

typedef enum {
    ARA_F64 = 0,           /* direct-access table stored in fp64 */
    ARA_F32_STORAGE = 1    /* table stored in fp32 (losses rounded once), arithmetic in fp64 (A13) */
} ara_precision;

typedef enum {
    ARA_LOAD_ALL_AT_ONCE = 0,  /* host YET copied to HBM inside ara_load_yet (paper's "concurrent" mode analogue) */
    ARA_LOAD_CHUNKED = 1       /* host YET streamed in trial chunks inside ara_run, copy/compute overlapped
                                  (paper's "sequential" transfer mode analogue) */
} ara_load_mode;

typedef enum {
    ARA_RUN_DIRECT = 0,   /* per occurrence: gather the layer's row window and apply every term (Alg. 3 as written) */
    ARA_RUN_FOLD = 1      /* per run: fold the catalogue once (o(e) for every event id, P:373 per-occurrence
                             independence), then gather one value per occurrence; YLT bit-identical to the
                             dense direct kernels (same lane order), within A21 of the sparse one */
} ara_run_mode;

typedef struct {
    int device;               /* CUDA device ordinal */
    ara_precision precision;
    void* stream;             /* cudaStream_t to enqueue on; NULL = library-created stream */
    int rank, world;          /* world >= 1, 0 <= rank < world */
    const void* nccl_unique_id; /* world > 1: ARA_NCCL_ID_BYTES from ara_nccl_unique_id() on rank 0,
                                   distributed by the caller (e.g. torch.distributed); else NULL */
    ara_load_mode load_mode;
    uint64_t chunk_trials;    /* CHUNKED: trials per H2D chunk; 0 = 65536 */
    int l2_persist;           /* nonzero: put the ELT table under an L2 persisting access-policy window */
    ara_run_mode run_mode;    /* ARA_RUN_DIRECT (default) or ARA_RUN_FOLD */
} ara_config;

/* Per-ELT financial terms I_j (Eq. 2; applied per lookup):
 * f = min(max(x - deductible, 0), limit).  deductible >= 0, limit > 0, +INFINITY allowed. */
typedef struct { double deductible, limit; } ara_elt_terms;

/* A layer (Eq. 3): ELTs [elt_begin, elt_end) of the loaded set, in that order,
 * plus the layer terms T (P:373 occurrence, P:375 aggregate).  Retentions >= 0,
 * limits > 0 (+INFINITY allowed). */
typedef struct {
    uint32_t elt_begin, elt_end;
    double occ_retention, occ_limit, agg_retention, agg_limit;
} ara_layer;

/* A layer with an explicit ELT list (ara_run_portfolio): `elts` (host) holds
 * n_elts strictly ascending indices into the loaded ELT set; the layer's ELT
 * losses are summed in that order.  Terms as in ara_layer. */
typedef struct {
    const uint32_t* elts;
    uint32_t n_elts;
    double occ_retention, occ_limit, agg_retention, agg_limit;
} ara_layer_list;

typedef struct {
    uint64_t n_trials_local, n_events_local, n_lookups_local;
    double kernel_ms;        /* ARA kernel(s): CUDA events on the launch stream */
    double h2d_ms;           /* YET bytes copied host->device inside this run (CHUNKED), event span */
    double allgather_ms;     /* YLT assembly across ranks (world > 1) */
    double total_ms;         /* whole ara_run on the stream, first enqueue to completion */
    uint64_t h2d_bytes;      /* bytes copied host->device inside this run */
    uint32_t n_kernel_launches;
    int32_t kernel_variant;  /* trial kernel of the last direct launch (ARA_KERNEL numbering): 30 ballot-
                                compacted rounds over packed rows (sparse column blocks), 12 cooperative
                                cp.async ring (dense fp64), 5 / 0 register pipeline (dense fp32, wide
                                windows); -2 = fold mode, -1 = none */
    double occupancy;        /* fraction of row windows the last direct launch gathers: the occupied-row
                                fraction of its column block when zero rows are skipped, else 1.0 */
} ara_run_stats;

/* ---- host-only helpers (no GPU needed) ---------------------------------- */

const char* ara_version(void);
const char* ara_status_string(ara_status s);

/* Balanced contiguous split of n_trials over world ranks (Alg. 1 l.3 "Split
 * YET to YET_i"; reading A17): the first n_trials % world ranks get
 * ceil(n/world) trials, the rest floor(n/world).  Pure host arithmetic. */
ara_status ara_partition(uint64_t n_trials, int world, int rank, uint64_t* first, uint64_t* count);

/* k = ceil(T / R) for return period R in [1, T] (reading A10); ARA_ERR_DOMAIN otherwise. */
ara_status ara_return_period_rank(uint64_t n_trials, double return_period, uint64_t* k);

/* NCCL bootstrap: rank 0 calls this and ships the bytes to the other ranks. */
ara_status ara_nccl_unique_id(void* out /* ARA_NCCL_ID_BYTES */);

/* ---- context -------------------------------------------------------------- */

/* Create a context for a catalogue of event ids [1, catalog_size] (A14).
 * COLLECTIVE when cfg->world > 1 (initialises the NCCL communicator).
 * Errors: INVALID_ARG (catalog_size == 0, bad rank/world, missing NCCL id),
 * CUDA, NCCL. */
ara_status ara_create(uint32_t catalog_size, const ara_config* cfg, ara_ctx** out);

void ara_destroy(ara_ctx* ctx);
const char* ara_last_error(const ara_ctx* ctx);

/* ELT ingest (Eq. 2) and densification into the interleaved direct-access table
 * tab[event][elt] (redesigned: one event's losses across all ELTs are
 * contiguous).
 *   elt_offsets [n_elts+1] u64, elt_offsets[0] == 0; ELT j owns records
 *   [elt_offsets[j], elt_offsets[j+1]) of event_ids (u32, in [1, catalog]) and
 *   losses (f64, finite, >= 0), event ids strictly ascending within each ELT
 *   (an ELT is a map: no duplicates).
 *   terms [n_elts] or NULL (identity: deductible 0, limit +inf).
 * Arrays may be host or device memory; they are not referenced after return.
 * Besides the table, the call builds a row-occupancy bitmap per 128-B column
 * block and, for blocks with at most half of their rows occupied, a packed
 * copy of every occupied row (one 32-B sector: non-zero mask, event id, first
 * non-zero losses), which the default sparse kernel gathers instead of the row.
 * COLLECTIVE when world > 1: rank 0's arrays are authoritative; rank 0
 * validates them and broadcasts the sparse records over NVLink (ncclBroadcast),
 * then every rank densifies its own copy of the table.  Other ranks may pass
 * NULL arrays but must pass the same n_elts (and their own terms).
 * Errors: INVALID_ARG (n_elts == 0 or > 65535, NULL arrays, bad offsets, ids
 * not strictly ascending within an ELT),
 * OUT_OF_RANGE (event id outside [1, catalog]), DOMAIN (negative / non-finite
 * loss, negative deductible, non-positive limit), OOM, CUDA, NCCL. */
ara_status ara_load_elts(ara_ctx* ctx, uint32_t n_elts, const uint64_t* elt_offsets,
                         const uint32_t* event_ids, const double* losses,
                         const ara_elt_terms* terms);

/* Replace the per-ELT terms without reloading the table (real-time re-pricing). */
ara_status ara_set_elt_terms(ara_ctx* ctx, uint32_t n_elts, const ara_elt_terms* terms);

/* YET ingest (Alg. 2): this rank's trials [first_trial, first_trial + n_trials_local)
 * of a YET with n_trials_global trials, as CSR:
 *   trial_offsets [n_trials_local + 1] u64, non-decreasing; trial i owns events
 *   event_ids[trial_offsets[i] - trial_offsets[0] ... trial_offsets[i+1] - trial_offsets[0]).
 *   event_ids u32 in [1, catalog], stored in the trial's timestamp order.
 * HOST pointers: ALL_AT_ONCE copies them into library-owned HBM before
 * returning; CHUNKED keeps the pointers (they must stay valid, ideally pinned,
 * until the last ara_run that uses them) and streams them inside ara_run.
 * DEVICE pointers are borrowed without a copy and must stay valid likewise;
 * the sparse kernel streams them with 16-B aligned bulk copies, which may read
 * up to 12 bytes before the first and after the last id inside the same
 * 16-B-aligned block (never across a page boundary).
 * Offsets monotonicity and id ranges are validated inside the ARA kernel and
 * reported by ara_run (OUT_OF_RANGE).  Local call (not collective); ara_run
 * checks that the ranks' ranges tile [0, n_trials_global).
 * Errors: INVALID_ARG (NULL, first + n > global), OOM, CUDA. */
ara_status ara_load_yet(ara_ctx* ctx, uint64_t n_trials_global, uint64_t first_trial,
                        uint64_t n_trials_local, const uint64_t* trial_offsets,
                        const uint32_t* event_ids);

/* Packed YET transfer: the same as ara_load_yet, but the
 * event ids arrive bit-packed, `bits` per id (1..32), id i of this shard at
 * bit offset i*bits of the little-endian u32 word stream `packed_ids`
 * (ara_pack_ids produces it; ara_packed_words gives its length, which
 * includes one padding word).  Only the packed words cross PCIe; a device
 * kernel unpacks them (per chunk in CHUNKED mode, overlapped with the copies).
 * With C <= 2^21 (the paper's 2M-event catalogue) 21-bit ids move 34 % fewer
 * bytes than u32.  Ids >= 2^bits cannot be represented (caller's choice of
 * bits); ids outside [1, C] are reported by ara_run as usual.
 * Errors: as ara_load_yet, plus INVALID_ARG for bits outside [1, 32]. */
ara_status ara_load_yet_packed(ara_ctx* ctx, uint64_t n_trials_global, uint64_t first_trial,
                               uint64_t n_trials_local, const uint64_t* trial_offsets,
                               const uint32_t* packed_ids, uint32_t bits);

/* Host helpers for the packed format (no GPU needed). */
uint64_t ara_packed_words(uint64_t n_ids, uint32_t bits);
/* Pack n_ids ids into out[ara_packed_words(n_ids, bits)] (host memory);
 * INVALID_ARG if an id does not fit in `bits` bits or bits is outside [1, 32]. */
ara_status ara_pack_ids(const uint32_t* ids, uint64_t n_ids, uint32_t bits, uint32_t* out);

/* Aggregate Risk Analysis (Alg. 1 lines 1-8 per layer; Alg. 3 per trial).
 * For each layer l and each trial t (readings A1-A8):
 *   l_e   = sum_{j in layer, in order} min(max(tab[e][j] - D_j, 0), Lim_j)
 *   o_e   = min(max(l_e - OccR, 0), OccL)
 *   Y[l][t] = min(max(sum_e o_e - AggR, 0), AggL)
 *   Y[n_layers][t] = sum_l Y[l][t] (portfolio, layer order)
 *   m[l][t] = #{e : o_e > 0}
 *   ylt   [(n_layers+1)][n_trials_global] f64, host or device, or NULL: the
 *         GLOBAL YLT, portfolio last.  With world > 1 the YLT is assembled
 *         across ranks (a9) either by the kernels themselves -- each
 *         trial's entries stored into every rank's global buffer over NVLink
 *         (CUDA IPC mappings made on the first run) -- or by ncclAllGather.
 *   lossy [n_layers][n_trials_local] u32, host or device, or NULL.
 *   stats nullable.
 * The YLT also stays resident on the device for ara_metrics.
 * COLLECTIVE when world > 1.
 * Errors: STATE (no ELTs / YET loaded), INVALID_ARG (n_layers 0 or >
 * ARA_MAX_LAYERS, empty or out-of-range ELT range, ranks not tiling the YET),
 * DOMAIN (negative retention, non-positive limit), OUT_OF_RANGE (YET id outside
 * [1, catalog] or decreasing offsets, detected on the device), CUDA, NCCL. */
ara_status ara_run(ara_ctx* ctx, uint32_t n_layers, const ara_layer* layers,
                   double* ylt, uint32_t* lossy, ara_run_stats* stats);

/* A portfolio of programs (Alg. 1 lines 1-2 "for each Program, for
 * each Layer"): n_layers layers with explicit ELT lists, grouped into
 * n_programs programs — program q owns layers [program_layers[q],
 * program_layers[q+1]) (program_layers [n_programs+1], host, from 0 to
 * n_layers, every program non-empty; n_programs may be 0).
 *   ylt [(n_layers + n_programs + 1)][n_trials_global]: the layer rows, then
 *       one row per program (sum of its layers, in layer order), then the
 *       portfolio (sum of all layers, in layer order).
 *   lossy, stats, collective semantics and errors: as ara_run.
 * ara_metrics then reports every one of those rows. */
ara_status ara_run_portfolio(ara_ctx* ctx, uint32_t n_programs, const uint32_t* program_layers,
                             uint32_t n_layers, const ara_layer_list* layers, double* ylt, uint32_t* lossy,
                             ara_run_stats* stats);

/* PML / TVaR of the last ara_run's YLT, for every layer and the portfolio:
 *   k[r]   = ceil(T / R_r)                                          (A10)
 *   pml [rows][n_rp]  = k-th largest Y                              (A9)
 *   tvar[rows][n_rp]  = mean of the k largest Y                     (A9)
 *   rows = n_layers + 1 after ara_run, n_layers + n_programs + 1 after
 *   ara_run_portfolio (the YLT rows, in the same order)
 * computed on the device by radix select over the fp64 bit patterns plus a
 * masked tail sum.  Outputs are HOST pointers (k may be NULL).  device_ms
 * (nullable) receives the metrics kernels' event time.  Every rank obtains
 * the same values.  COLLECTIVE when world > 1: on large global YLTs (>= 3M
 * trials) each rank selects over its own shard and the per-pass histograms
 * and tail sums are all-reduced (the distributed select); NCCL failures are
 * reported as ARA_ERR_NCCL.
 * Errors: STATE (no run yet), INVALID_ARG (n_rp 0 or > ARA_MAX_RP, NULL),
 * DOMAIN (R outside [1, T]), CUDA, NCCL. */
ara_status ara_metrics(ara_ctx* ctx, uint32_t n_rp, const double* return_periods,
                       uint64_t* k, double* pml, double* tvar, double* device_ms);

/* Aggregate exceedance-probability (EP) curve of every row of the last
 * ara_run's YLT (SURVEY 8f F4 "full EP curve"; the risk-metric stage of P:273;
 * reading A23):
 *   counts[row][i] = #{t : Y[row][t] > thresholds[i]},  EP(x_i) = counts / n_trials_global
 * (strict exceedance: the fraction of simulated years whose loss is larger).
 * The other direction of the curve, the loss at exceedance probability p, is
 * PML(1/p): ara_metrics with return period 1/p.
 *   thresholds [n_points] HOST doubles, non-decreasing, no NaN (+-inf allowed)
 *   counts     [rows][n_points] HOST u64, rows as in ara_metrics
 * Exact integers, computed on the device (one sweep of the YLT, binary search
 * over the thresholds, integer histograms).  COLLECTIVE when world > 1: each
 * rank counts its own trials and the counts are all-reduced.
 * Errors: STATE (no run yet), INVALID_ARG (n_points 0 or > ARA_MAX_EP_POINTS,
 * NULL or device arrays), DOMAIN (NaN or decreasing thresholds), CUDA, NCCL. */
ara_status ara_ep_curve(ara_ctx* ctx, uint32_t n_points, const double* thresholds, uint64_t* counts);

#ifdef __cplusplus
}
#endif
#endif /* ARA_H */
