// ara_host.cu — C-ABI host runtime of the B200 ARA library (include/ara.h).
//
// Context, validation, pointer classification, H2D loading (all-at-once or
// chunked with copy/compute overlap, Alg. 2 P:321-337 and the
// transfer modes of P:523-542), layer batching, the NCCL YLT all-gather
// (Alg. 1 l.9 "Populate YLT from YLT_i") and the metrics driver.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <new>
#include <chrono>
#include <thread>

#include <nvtx3/nvToolsExt.h>

#include "ara_internal.cuh"

using namespace ara;

namespace {

// NVTX range around each API call and each streamed chunk (host side: the
// enqueue structure; an nsys timeline pairs it with the copy / kernel rows)
// ARA_HOST_TRACE=1: host timestamps (us) of the API calls' phases on stderr,
// to see where a step's GPU idle time comes from (diagnostic only)
inline void host_trace(const char* what) {
    static const bool on = [] { const char* v = getenv("ARA_HOST_TRACE"); return v && atoi(v); }();
    if (!on) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
    fprintf(stderr, "HT %.1f %s\n", us, what);
}

struct Nvtx {
    explicit Nvtx(const char* name) : name_(name) { nvtxRangePushA(name); host_trace(name_); }
    ~Nvtx() { nvtxRangePop(); host_trace("return"); }
    const char* name_;
    Nvtx(const Nvtx&) = delete;
    Nvtx& operator=(const Nvtx&) = delete;
};

ara_status fail(ara_ctx* ctx, ara_status st, const char* fmt, ...) {
    if (ctx) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        ctx->last_error = buf;
    }
    return st;
}

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess) {                                                               \
            cudaGetLastError();                                                                \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? ARA_ERR_OOM : ARA_ERR_CUDA,     \
                        "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__); \
        }                                                                                      \
    } while (0)

#define NK(x)                                                                             \
    do {                                                                                  \
        ncclResult_t r_ = (x);                                                            \
        if (r_ != ncclSuccess)                                                            \
            return fail(ctx, ARA_ERR_NCCL, "%s failed: %s", #x, ncclGetErrorString(r_));  \
    } while (0)

enum class Mem { Host, Pinned, Device };

Mem classify(const void* p) {
    if (!p) return Mem::Host;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return Mem::Host;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return Mem::Device;
    if (a.type == cudaMemoryTypeHost) return Mem::Pinned;
    return Mem::Host;
}

bool valid_retention(double r) { return r >= 0.0 && r <= 1.7976931348623157e308; }
bool valid_limit(double l) { return l > 0.0; }   // +inf allowed, NaN rejected

template <typename T>
ara_status ensure(ara_ctx* ctx, T*& p, size_t& cap, size_t n) {
    if (cap >= n && p) return ARA_OK;
    cudaFree(p);
    p = nullptr;
    cap = 0;
    CK(cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
    cap = n;
    return ARA_OK;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) {
        cudaGetLastError();
        return 0.f;
    }
    return ms;
}

void release_yet(ara_ctx* ctx) {
    if (ctx->h_registered) {
        cudaHostUnregister(ctx->h_registered);
        cudaGetLastError();
        ctx->h_registered = nullptr;
    }
    ctx->d_off = nullptr;
    ctx->d_ids = nullptr;
    ctx->h_off = nullptr;
    ctx->h_ids = nullptr;
    ctx->h_packed = nullptr;
    ctx->pack_bits = 0;
    ctx->chunked_pending = false;
    ctx->yet_loaded = false;
    ctx->tiling_checked = false;
}

// Error bits written by the kernels -> status.
ara_status device_errors(ara_ctx* ctx, uint32_t bits) {
    if (!bits) return ARA_OK;
    if (bits & ERRBIT_EVENT_RANGE)
        return fail(ctx, ARA_ERR_OUT_OF_RANGE, "YET event id outside [1, %u]", ctx->catalog);
    if (bits & ERRBIT_OFFSETS) return fail(ctx, ARA_ERR_OUT_OF_RANGE, "YET trial offsets decrease");
    if (bits & ERRBIT_ELT_RANGE)
        return fail(ctx, ARA_ERR_OUT_OF_RANGE, "ELT event id outside [1, %u]", ctx->catalog);
    if (bits & ERRBIT_ELT_ORDER)
        return fail(ctx, ARA_ERR_INVALID_ARG, "ELT event ids not strictly ascending (duplicate id)");
    if (bits & ERRBIT_ELT_LOSS)
        return fail(ctx, ARA_ERR_DOMAIN, "ELT loss negative, non-finite or not representable");
    return fail(ctx, ARA_ERR_CUDA, "unknown device error bits 0x%x", bits);
}

}  // namespace

// ============================================================ host-only helpers
extern "C" const char* ara_version(void) { return "ara-b200 1.0 (sm_100a)"; }

extern "C" const char* ara_status_string(ara_status s) {
    switch (s) {
        case ARA_OK: return "ARA_OK";
        case ARA_ERR_INVALID_ARG: return "ARA_ERR_INVALID_ARG";
        case ARA_ERR_OUT_OF_RANGE: return "ARA_ERR_OUT_OF_RANGE";
        case ARA_ERR_DOMAIN: return "ARA_ERR_DOMAIN";
        case ARA_ERR_STATE: return "ARA_ERR_STATE";
        case ARA_ERR_OOM: return "ARA_ERR_OOM";
        case ARA_ERR_CUDA: return "ARA_ERR_CUDA";
        case ARA_ERR_NCCL: return "ARA_ERR_NCCL";
    }
    return "ARA_ERR_UNKNOWN";
}

extern "C" ara_status ara_partition(uint64_t n, int world, int rank, uint64_t* first, uint64_t* count) {
    if (world < 1 || rank < 0 || rank >= world || !first || !count) return ARA_ERR_INVALID_ARG;
    const uint64_t q = n / (uint64_t)world, rem = n % (uint64_t)world, r = (uint64_t)rank;
    *first = r * q + (r < rem ? r : rem);
    *count = q + (r < rem ? 1 : 0);
    return ARA_OK;
}

extern "C" ara_status ara_return_period_rank(uint64_t T, double R, uint64_t* k) {
    if (!k) return ARA_ERR_INVALID_ARG;
    if (!(R >= 1.0) || !(R <= (double)T)) return ARA_ERR_DOMAIN;
    if (R == std::floor(R)) {
        const uint64_t r = (uint64_t)R;
        *k = T / r + (T % r ? 1 : 0);
    } else {
        *k = (uint64_t)std::ceil((long double)T / (long double)R);
    }
    return ARA_OK;
}

extern "C" ara_status ara_nccl_unique_id(void* out) {
    if (!out) return ARA_ERR_INVALID_ARG;
    static_assert(sizeof(ncclUniqueId) == ARA_NCCL_ID_BYTES, "nccl id size");
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return ARA_ERR_NCCL;
    std::memcpy(out, &id, sizeof id);
    return ARA_OK;
}

// ============================================================ context
extern "C" ara_status ara_create(uint32_t catalog_size, const ara_config* cfg, ara_ctx** out) {
    if (!out || !cfg) return ARA_ERR_INVALID_ARG;
    *out = nullptr;
    if (catalog_size == 0 || catalog_size == 0xFFFFFFFFu) return ARA_ERR_INVALID_ARG;
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) return ARA_ERR_INVALID_ARG;
    if (cfg->world > 1 && !cfg->nccl_unique_id) return ARA_ERR_INVALID_ARG;
    if (cfg->precision != ARA_F64 && cfg->precision != ARA_F32_STORAGE) return ARA_ERR_INVALID_ARG;
    if (cfg->load_mode != ARA_LOAD_ALL_AT_ONCE && cfg->load_mode != ARA_LOAD_CHUNKED) return ARA_ERR_INVALID_ARG;
    if (cfg->run_mode != ARA_RUN_DIRECT && cfg->run_mode != ARA_RUN_FOLD) return ARA_ERR_INVALID_ARG;
    ara_ctx* ctx = new (std::nothrow) ara_ctx();
    if (!ctx) return ARA_ERR_OOM;
    ctx->device = cfg->device;
    ctx->rank = cfg->rank;
    ctx->world = cfg->world;
    ctx->precision = cfg->precision;
    ctx->load_mode = cfg->load_mode;
    ctx->chunk_trials = cfg->chunk_trials ? cfg->chunk_trials : 65536;
    ctx->l2_persist = cfg->l2_persist;
    ctx->run_mode = cfg->run_mode;
    ctx->catalog = catalog_size;
    if (const char* v = getenv("ARA_GRID_MULT")) ctx->grid_mult = atof(v);
    if (const char* v = getenv("ARA_KERNEL")) ctx->kernel_variant = atoi(v);
    if (const char* v = getenv("ARA_FOLD_BC")) ctx->fold_bc = atoi(v) != 0;   // 0: the dense fold pass (A/B)
    if (const char* v = getenv("ARA_NO_SKIP")) ctx->no_skip = atoi(v) != 0;
    if (const char* v = getenv("ARA_NO_P2P")) ctx->use_p2p = atoi(v) == 0;
    if (const char* v = getenv("ARA_METRICS_DIST")) ctx->metrics_dist = atoi(v);
    if (const char* v = getenv("ARA_LOOPBACK")) {
        int w = 0, r = 0;
        if (cfg->world != 1 || sscanf(v, "%d,%d", &w, &r) != 2 || w < 1 || w > ara::kMaxPeers || r < 0 || r >= w) {
            delete ctx;
            return ARA_ERR_INVALID_ARG;
        }
        ctx->lb_world = w;
        ctx->lb_rank = r;
    }
    auto bail = [&](ara_status st) {
        ara_destroy(ctx);
        return st;
    };
    if (cudaSetDevice(cfg->device) != cudaSuccess) {
        cudaGetLastError();
        return bail(ARA_ERR_CUDA);
    }
    cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, cfg->device);
    if (cfg->stream) {
        ctx->stream = (cudaStream_t)cfg->stream;
    } else {
        if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(ARA_ERR_CUDA);
        ctx->own_stream = true;
    }
    if (cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess) return bail(ARA_ERR_CUDA);
    for (auto& e : ctx->ev)
        if (cudaEventCreate(&e) != cudaSuccess) return bail(ARA_ERR_CUDA);
    if (cudaMalloc(&ctx->d_err, 64) != cudaSuccess) return bail(ARA_ERR_OOM);
    if (cudaMalloc(&ctx->d_small, 64 * sizeof(uint64_t)) != cudaSuccess) return bail(ARA_ERR_OOM);
    if (cudaMallocHost(&ctx->h_small, 64 * sizeof(uint64_t)) != cudaSuccess) return bail(ARA_ERR_OOM);
    if (cudaMemset(ctx->d_err, 0, 64) != cudaSuccess) return bail(ARA_ERR_CUDA);
    if (ctx->l2_persist) {
        cudaDeviceProp prop{};
        if (cudaGetDeviceProperties(&prop, cfg->device) == cudaSuccess && prop.persistingL2CacheMaxSize > 0)
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, prop.persistingL2CacheMaxSize);
        cudaGetLastError();
    }
    if (cfg->world > 1) {
        ncclUniqueId id;
        std::memcpy(&id, cfg->nccl_unique_id, sizeof id);
        if (ncclCommInitRank(&ctx->comm, cfg->world, id, cfg->rank) != ncclSuccess) {
            ctx->comm = nullptr;
            return bail(ARA_ERR_NCCL);
        }
    }
    *out = ctx;
    return ARA_OK;
}

extern "C" void ara_destroy(ara_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    release_yet(ctx);
    for (int b = 0; b < 2; ++b) {   // peers' global YLTs mapped by IPC, then our own
        for (int r = 0; r < ctx->world && r < ara::kMaxPeers; ++r)
            if (ctx->peer_p2p[b][r] && r != ctx->rank) cudaIpcCloseMemHandle(ctx->peer_p2p[b][r]);
        cudaFree(ctx->d_p2p[b]);
    }
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    cudaFree(ctx->d_table);
    cudaFree(ctx->d_off_own);
    cudaFree(ctx->d_ids_own);
    cudaFree(ctx->d_packed_own);
    cudaFree(ctx->d_ylt_local);
    cudaFree(ctx->d_ylt_gather);
    cudaFree(ctx->d_ylt_global);
    cudaFree(ctx->d_lossy);
    cudaFree(ctx->d_fold);
    cudaFree(ctx->d_ep);
    cudaFree(ctx->d_sp_off);
    cudaFree(ctx->d_sp_ev);
    cudaFree(ctx->d_sp_ls);
    cudaFree(ctx->d_err);
    cudaFree(ctx->d_small);
    cudaFreeHost(ctx->h_small);
    metrics_free(ctx->ms);
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    cudaGetLastError();
    delete ctx;
}

extern "C" const char* ara_last_error(const ara_ctx* ctx) { return ctx ? ctx->last_error.c_str() : "null context"; }

// ============================================================ ELTs
namespace {

ara_status check_terms(ara_ctx* ctx, uint32_t n, const ara_elt_terms* t) {
    if (!t) return ARA_OK;
    if (classify(t) == Mem::Device) return fail(ctx, ARA_ERR_INVALID_ARG, "ELT terms must be host memory");
    for (uint32_t j = 0; j < n; ++j)
        if (!valid_retention(t[j].deductible) || !valid_limit(t[j].limit))
            return fail(ctx, ARA_ERR_DOMAIN, "ELT %u terms: deductible must be >= 0 and finite, limit > 0", j);
    return ARA_OK;
}

// (Re)allocate the column-blocked table for n_elts ELTs (ara::TableGeo).
ara_status alloc_table(ara_ctx* ctx, uint32_t n_elts) {
    const TableGeo g = table_geometry(n_elts, ctx->catalog, ctx->precision == ARA_F32_STORAGE);
    if (g.bytes != ctx->table_bytes || g.epb != ctx->geo.epb || g.n_blocks != ctx->geo.n_blocks) {
        ctx->table_clean = false;
        if (g.bytes != ctx->table_bytes) {
            cudaFree(ctx->d_table);
            ctx->d_table = nullptr;
            ctx->table_bytes = 0;
            CK(cudaMalloc(&ctx->d_table, g.bytes));
            ctx->table_bytes = g.bytes;
        }
    }
    ctx->geo = g;
    return ARA_OK;
}

// Validate the ELT offsets on the host and return them (rank 0 / single rank).
ara_status read_elt_offsets(ara_ctx* ctx, uint32_t n_elts, const uint64_t* elt_offsets, const uint32_t* event_ids,
                            const double* losses, std::vector<uint64_t>& hoff) {
    if (!elt_offsets) return fail(ctx, ARA_ERR_INVALID_ARG, "elt_offsets is NULL");
    hoff.resize(n_elts + 1);
    if (classify(elt_offsets) == Mem::Device)
        CK(cudaMemcpy(hoff.data(), elt_offsets, (n_elts + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    else
        std::memcpy(hoff.data(), elt_offsets, (n_elts + 1) * sizeof(uint64_t));
    if (hoff[0] != 0) return fail(ctx, ARA_ERR_INVALID_ARG, "elt_offsets[0] must be 0");
    for (uint32_t j = 0; j < n_elts; ++j)
        if (hoff[j + 1] < hoff[j]) return fail(ctx, ARA_ERR_INVALID_ARG, "elt_offsets decrease at ELT %u", j);
    if (hoff[n_elts] && (!event_ids || !losses)) return fail(ctx, ARA_ERR_INVALID_ARG, "event_ids/losses NULL");
    return ARA_OK;
}

// Device view of the sparse ELT records: the caller's device arrays, or the
// context's staging buffers (filled by H2D copies or an NVLink broadcast).
struct SparseDev {
    const uint64_t* off = nullptr;
    const uint32_t* ev = nullptr;
    const double* ls = nullptr;
};

ara_status stage_sparse(ara_ctx* ctx, uint32_t n_elts, uint64_t nrec, const uint64_t* hoff,
                        const uint64_t* elt_offsets, const uint32_t* event_ids, const double* losses,
                        bool to_staging, SparseDev* out) {
    ara_status st;
    if ((st = ensure(ctx, ctx->d_sp_off, ctx->sp_off_cap, (size_t)n_elts + 1)) != ARA_OK) return st;
    if ((st = ensure(ctx, ctx->d_sp_ev, ctx->sp_ev_cap, (size_t)nrec)) != ARA_OK) return st;
    if ((st = ensure(ctx, ctx->d_sp_ls, ctx->sp_ls_cap, (size_t)nrec)) != ARA_OK) return st;
    *out = SparseDev{ctx->d_sp_off, ctx->d_sp_ev, ctx->d_sp_ls};
    if (hoff) {   // this rank holds the arrays
        if (classify(elt_offsets) == Mem::Device && !to_staging) out->off = elt_offsets;
        else CK(cudaMemcpyAsync(ctx->d_sp_off, hoff, (n_elts + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                ctx->stream));
        if (nrec) {
            const bool dev_ev = classify(event_ids) == Mem::Device, dev_ls = classify(losses) == Mem::Device;
            if (dev_ev && !to_staging) out->ev = event_ids;
            else CK(cudaMemcpyAsync(ctx->d_sp_ev, event_ids, nrec * sizeof(uint32_t),
                                    dev_ev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
            if (dev_ls && !to_staging) out->ls = losses;
            else CK(cudaMemcpyAsync(ctx->d_sp_ls, losses, nrec * sizeof(double),
                                    dev_ls ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, ctx->stream));
        }
    }
    return ARA_OK;
}

// (Re)build this rank's table from device-resident sparse records: zero-fill,
// scatter + validate (densify kernel), read back the error bits.
ara_status densify_local(ara_ctx* ctx, uint32_t n_elts, uint64_t nrec, const SparseDev& sp) {
    const int fp32 = ctx->precision == ARA_F32_STORAGE;
    ara_status ast = alloc_table(ctx, n_elts);
    if (ast != ARA_OK) return ast;
    // a table whose non-zero rows are all marked in its bitmaps (a previous
    // densify) is cleared row by row; otherwise the whole allocation is zeroed
    host_trace("densify_local");
    if (ctx->table_clean) CK(launch_clear_rows(ctx->d_table, ctx->geo, ctx->catalog, ctx->stream));
    else CK(cudaMemsetAsync(ctx->d_table, 0, ctx->geo.pk_off, ctx->stream));   // packed slots: written before read
    ctx->table_clean = false;
    CK(cudaMemsetAsync(ctx->d_err, 0, sizeof(uint32_t), ctx->stream));
    CK(launch_densify(sp.off, sp.ev, sp.ls, n_elts, nrec, ctx->catalog, ctx->d_table, ctx->geo, fp32, ctx->d_err,
                      ctx->stream));
    CK(cudaMemcpyAsync(ctx->h_small, ctx->d_err, sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    // occupied-row counters per column block: into the pinned scratch when they fit (same sync)
    const uint32_t nb = ctx->geo.n_blocks;
    const void* d_occ = static_cast<const char*>(ctx->d_table) + ctx->geo.occ_off;
    uint32_t* h_occ = reinterpret_cast<uint32_t*>(ctx->h_small + 16);
    const bool small = nb <= 96;
    if (small) CK(cudaMemcpyAsync(h_occ, d_occ, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    host_trace("densify launched");
    CK(cudaStreamSynchronize(ctx->stream));
    host_trace("densify synced");
    ctx->occ_rows.assign(nb, 0u);
    if (small) std::memcpy(ctx->occ_rows.data(), h_occ, nb * sizeof(uint32_t));
    else CK(cudaMemcpy(ctx->occ_rows.data(), d_occ, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    ctx->table_clean = true;   // every stored element's row is marked (even for rejected ELTs)
    if (!ctx->no_skip) CK(launch_pack_rows(ctx->d_table, ctx->geo, ctx->catalog, fp32, ctx->stream));
    return device_errors(ctx, (uint32_t)(ctx->h_small[0] & 0xffffffffu));
}

// L2 persisting access-policy window (cfg.l2_persist; north star "HBM layout":
// keep the hot ELT data resident in B200's L2) over the bytes a launch
// actually gathers: for the sparse kernel the block's packed rows (the
// occupied slots are touched at random), for the dense
// kernels the window's column block of the table (256 MB at the paper's
// catalogue in fp64, 128 MB in fp32).  hitRatio = persisting carve-out /
// window bytes, so the persisting lines are a random subset of the window.
// Set on the context stream before the launch, cleared after the run (the
// stream may be the caller's).
void set_l2_window(ara_ctx* ctx, const void* base, size_t bytes) {
    if (!ctx->l2_persist) return;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, ctx->device) != cudaSuccess) { cudaGetLastError(); return; }
    const size_t win = bytes < (size_t)prop.accessPolicyMaxWindowSize ? bytes : (size_t)prop.accessPolicyMaxWindowSize;
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = const_cast<void*>(base);
    v.accessPolicyWindow.num_bytes = base ? win : 0;
    const double hr = win ? (double)prop.persistingL2CacheMaxSize / (double)win : 0.0;
    v.accessPolicyWindow.hitRatio = (float)(hr > 1.0 ? 1.0 : hr);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaGetLastError();
}

}  // namespace

extern "C" ara_status ara_load_elts(ara_ctx* ctx, uint32_t n_elts, const uint64_t* elt_offsets,
                                    const uint32_t* event_ids, const double* losses,
                                    const ara_elt_terms* terms) {
    Nvtx nvtx_("ara_load_elts");
    if (!ctx) return ARA_ERR_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    if (n_elts == 0 || n_elts > 65535) return fail(ctx, ARA_ERR_INVALID_ARG, "n_elts must be in [1, 65535]");
    const bool root = ctx->rank == 0;
    ara_status st = check_terms(ctx, n_elts, terms);
    std::vector<uint64_t> hoff;
    if (st == ARA_OK && root) st = read_elt_offsets(ctx, n_elts, elt_offsets, event_ids, losses, hoff);
    uint64_t nrec = (st == ARA_OK && root) ? hoff[n_elts] : 0;
    SparseDev sp;
    if (ctx->world > 1) {
        // Agree on (status, n_elts, records) first so that no failing rank
        // can strand the others in the broadcasts below: one max-all-reduce of
        // [status, n_elts, ~n_elts, records] gives every rank the worst
        // status, whether all n_elts agree (max == min), and rank 0's record
        // count (the others contribute 0).  Then rank 0's sparse records (a
        // few MB) go over NVLink and every rank densifies locally — instead of
        // N host copies of the replicated data or a
        // broadcast of the whole table.
        ctx->h_small[0] = (uint64_t)st;
        ctx->h_small[1] = n_elts;
        ctx->h_small[2] = ~(uint64_t)n_elts;
        ctx->h_small[3] = root ? nrec : 0;
        CK(cudaMemcpyAsync(ctx->d_small, ctx->h_small, 4 * sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
        NK(ncclAllReduce(ctx->d_small, ctx->d_small, 4, ncclUint64, ncclMax, ctx->comm, ctx->stream));
        CK(cudaMemcpyAsync(ctx->h_small + 8, ctx->d_small, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        const ara_status rst = (ara_status)ctx->h_small[8];
        if (rst != ARA_OK) return st != ARA_OK ? st : fail(ctx, rst, "another rank rejected the ELTs");
        if (ctx->h_small[9] != ~ctx->h_small[10])
            return fail(ctx, ARA_ERR_INVALID_ARG, "ranks disagree on n_elts");
        nrec = ctx->h_small[11];
        ara_status s2 = stage_sparse(ctx, n_elts, nrec, root ? hoff.data() : nullptr, elt_offsets, event_ids, losses,
                                     /*to_staging=*/true, &sp);
        if (s2 != ARA_OK) return s2;
        NK(ncclGroupStart());
        NK(ncclBroadcast(ctx->d_sp_off, ctx->d_sp_off, n_elts + 1, ncclUint64, 0, ctx->comm, ctx->stream));
        if (nrec) {
            NK(ncclBroadcast(ctx->d_sp_ev, ctx->d_sp_ev, nrec, ncclUint32, 0, ctx->comm, ctx->stream));
            NK(ncclBroadcast(ctx->d_sp_ls, ctx->d_sp_ls, nrec, ncclDouble, 0, ctx->comm, ctx->stream));
        }
        NK(ncclGroupEnd());
    } else {
        if (st != ARA_OK) return st;
        ara_status s2 = stage_sparse(ctx, n_elts, nrec, hoff.data(), elt_offsets, event_ids, losses,
                                     /*to_staging=*/false, &sp);
        if (s2 != ARA_OK) return s2;
    }
    // From here the table changes: until this load succeeds there are no
    // usable ELTs (ara_run -> STATE) and no run whose metrics could be read.
    ctx->n_elts = 0;
    ctx->last_layers = 0;
    st = densify_local(ctx, n_elts, nrec, sp);   // every rank sees the same records: same verdict
    if (st != ARA_OK) return st;
    ctx->n_elts = n_elts;
    ctx->terms.assign(n_elts, ara_elt_terms{0.0, INFINITY});
    if (terms)
        for (uint32_t j = 0; j < n_elts; ++j) ctx->terms[j] = terms[j];
    return ARA_OK;
}

extern "C" ara_status ara_set_elt_terms(ara_ctx* ctx, uint32_t n_elts, const ara_elt_terms* terms) {
    if (!ctx) return ARA_ERR_INVALID_ARG;
    if (ctx->n_elts == 0) return fail(ctx, ARA_ERR_STATE, "no ELTs loaded");
    if (n_elts != ctx->n_elts || !terms) return fail(ctx, ARA_ERR_INVALID_ARG, "need %u ELT terms", ctx->n_elts);
    ara_status st = check_terms(ctx, n_elts, terms);
    if (st != ARA_OK) return st;
    for (uint32_t j = 0; j < n_elts; ++j) ctx->terms[j] = terms[j];
    return ARA_OK;
}

// ============================================================ YET
namespace {

// YET ingest shared by ara_load_yet (bits == 0: u32 ids) and
// ara_load_yet_packed (bits > 0: bit-packed ids, unpacked on the device).
ara_status load_yet_impl(ara_ctx* ctx, uint64_t n_trials_global, uint64_t first_trial, uint64_t n_trials_local,
                         const uint64_t* trial_offsets, const uint32_t* event_ids, uint32_t bits) {
    Nvtx nvtx_("ara_load_yet");
    if (!ctx) return ARA_ERR_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    if (n_trials_global == 0) return fail(ctx, ARA_ERR_INVALID_ARG, "n_trials_global must be >= 1");
    if (first_trial > n_trials_global || n_trials_local > n_trials_global - first_trial)
        return fail(ctx, ARA_ERR_INVALID_ARG, "trial range [%llu, +%llu) exceeds %llu",
                    (unsigned long long)first_trial, (unsigned long long)n_trials_local,
                    (unsigned long long)n_trials_global);
    if (!trial_offsets) return fail(ctx, ARA_ERR_INVALID_ARG, "trial_offsets is NULL");
    if (bits > 32) return fail(ctx, ARA_ERR_INVALID_ARG, "bits must be in [1, 32]");
    // Later work on the stream is ordered after any run still reading the old
    // YET; only unregistering a host range we pinned needs the copies done.
    if (ctx->h_registered) CK(cudaStreamSynchronize(ctx->copy_stream));
    release_yet(ctx);

    const Mem mo = classify(trial_offsets);
    const Mem mi = classify(event_ids);
    uint64_t n_ev = 0;
    bool n_ev_known = false;
    if (mo != Mem::Device) {
        if (trial_offsets[n_trials_local] < trial_offsets[0])
            return fail(ctx, ARA_ERR_OUT_OF_RANGE, "YET trial offsets decrease");
        n_ev = trial_offsets[n_trials_local] - trial_offsets[0];
        n_ev_known = true;
    }
    if (!event_ids && !(n_ev_known && n_ev == 0)) return fail(ctx, ARA_ERR_INVALID_ARG, "event_ids is NULL");
    if ((mi != Mem::Device || bits) && !n_ev_known) {
        CK(cudaMemcpy(ctx->h_small, trial_offsets, sizeof(uint64_t), cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(ctx->h_small + 1, trial_offsets + n_trials_local, sizeof(uint64_t), cudaMemcpyDeviceToHost));
        if (ctx->h_small[1] < ctx->h_small[0]) return fail(ctx, ARA_ERR_OUT_OF_RANGE, "YET trial offsets decrease");
        n_ev = ctx->h_small[1] - ctx->h_small[0];
        n_ev_known = true;
    }
    ctx->n_events_host = n_ev_known ? n_ev : 0;
    const bool chunked = ctx->load_mode == ARA_LOAD_CHUNKED;
    const uint64_t words = bits ? ara_packed_words(n_ev, bits) : 0;

    // offsets
    if (mo == Mem::Device) {
        ctx->d_off = trial_offsets;
    } else {
        ara_status st = ensure(ctx, ctx->d_off_own, ctx->own_off_cap, n_trials_local + 1);
        if (st != ARA_OK) return st;
        ctx->d_off = ctx->d_off_own;
        if (chunked) ctx->h_off = trial_offsets;
        else CK(cudaMemcpyAsync(ctx->d_off_own, trial_offsets, (n_trials_local + 1) * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, ctx->stream));
    }
    // event ids
    if (mi == Mem::Device && !bits) {
        ctx->d_ids = event_ids;
    } else {
        ara_status st = ensure(ctx, ctx->d_ids_own, ctx->own_ids_cap, n_ev);
        if (st != ARA_OK) return st;
        ctx->d_ids = ctx->d_ids_own;
        if (bits && mi == Mem::Device) {            // packed, already on the device: unpack now
            CK(launch_unpack(event_ids, bits, 0, n_ev, ctx->d_ids_own, ctx->stream));
        } else if (chunked) {
            const size_t host_bytes = bits ? words * sizeof(uint32_t) : n_ev * sizeof(uint32_t);
            if (bits) {
                ctx->h_packed = event_ids;
                st = ensure(ctx, ctx->d_packed_own, ctx->packed_cap, words);
                if (st != ARA_OK) return st;
            } else {
                ctx->h_ids = event_ids;
            }
            if (mi == Mem::Host && n_ev) {   // pageable: pin for async DMA (once per load)
                if (cudaHostRegister((void*)event_ids, host_bytes, cudaHostRegisterReadOnly) == cudaSuccess)
                    ctx->h_registered = (void*)event_ids;
                cudaGetLastError();
            }
        } else if (n_ev) {
            if (bits) {
                st = ensure(ctx, ctx->d_packed_own, ctx->packed_cap, words);
                if (st != ARA_OK) return st;
                CK(cudaMemcpyAsync(ctx->d_packed_own, event_ids, words * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                   ctx->stream));
                CK(launch_unpack(ctx->d_packed_own, bits, 0, n_ev, ctx->d_ids_own, ctx->stream));
            } else {
                CK(cudaMemcpyAsync(ctx->d_ids_own, event_ids, n_ev * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                   ctx->stream));
            }
        }
    }
    ctx->pack_bits = bits;
    ctx->chunked_pending = chunked && (ctx->h_off || ctx->h_ids || ctx->h_packed);
    // Host sources are released to the caller on return (ALL_AT_ONCE copies
    // must be complete); device-resident inputs need no sync.
    if (!ctx->chunked_pending && (mo != Mem::Device || (mi != Mem::Device && n_ev)))
        CK(cudaStreamSynchronize(ctx->stream));
    ctx->T_global = n_trials_global;
    ctx->first = first_trial;
    ctx->T_local = n_trials_local;
    ctx->yet_loaded = true;
    ctx->tiling_checked = false;
    return ARA_OK;
}

}  // namespace

extern "C" uint64_t ara_packed_words(uint64_t n_ids, uint32_t bits) {
    if (bits == 0 || bits > 32) return 0;
    return (n_ids * bits + 31) / 32 + 1;   // + one padding word (two-word reads)
}

extern "C" ara_status ara_pack_ids(const uint32_t* ids, uint64_t n, uint32_t bits, uint32_t* out) {
    if (bits == 0 || bits > 32 || (!ids && n) || !out) return ARA_ERR_INVALID_ARG;
    const uint64_t words = ara_packed_words(n, bits);
    const uint64_t lim = bits == 32 ? 0x100000000ull : (1ull << bits);
    // 32 consecutive ids fill exactly `bits` whole words, so groups of 32 ids
    // pack independently (threads over groups).
    const uint64_t groups = (n + 31) / 32;
    unsigned nt = std::thread::hardware_concurrency();
    if (nt < 1) nt = 1;
    if (nt > 64) nt = 64;
    if (n < (1u << 20)) nt = 1;
    std::vector<int> bad(nt, 0);
    auto work = [&](unsigned k) {
        const uint64_t g0 = groups * k / nt, g1 = groups * (k + 1) / nt;
        for (uint64_t w = g0 * bits; w < g1 * bits && w < words; ++w) out[w] = 0u;
        for (uint64_t i = g0 * 32; i < g1 * 32 && i < n; ++i) {
            const uint64_t v = ids[i];
            if (v >= lim) { bad[k] = 1; continue; }
            const uint64_t b = i * bits;
            const uint64_t w = b >> 5;
            const uint64_t x = v << (b & 31);
            out[w] |= (uint32_t)x;
            if ((x >> 32) != 0) out[w + 1] |= (uint32_t)(x >> 32);
        }
    };
    std::vector<std::thread> th;
    for (unsigned k = 1; k < nt; ++k) th.emplace_back(work, k);
    work(0);
    for (auto& t : th) t.join();
    for (uint64_t w = groups * bits; w < words; ++w) out[w] = 0u;
    for (int b : bad)
        if (b) return ARA_ERR_INVALID_ARG;
    return ARA_OK;
}

extern "C" ara_status ara_load_yet(ara_ctx* ctx, uint64_t n_trials_global, uint64_t first_trial,
                                   uint64_t n_trials_local, const uint64_t* trial_offsets,
                                   const uint32_t* event_ids) {
    return load_yet_impl(ctx, n_trials_global, first_trial, n_trials_local, trial_offsets, event_ids, 0);
}

extern "C" ara_status ara_load_yet_packed(ara_ctx* ctx, uint64_t n_trials_global, uint64_t first_trial,
                                          uint64_t n_trials_local, const uint64_t* trial_offsets,
                                          const uint32_t* packed_ids, uint32_t bits) {
    if (ctx && (bits == 0 || bits > 32)) return fail(ctx, ARA_ERR_INVALID_ARG, "bits must be in [1, 32]");
    return load_yet_impl(ctx, n_trials_global, first_trial, n_trials_local, trial_offsets, packed_ids, bits);
}

// ============================================================ run
namespace {

struct Group {
    uint32_t l0, nl;      // layers [l0, l0+nl), all on one sector window
    uint32_t q0, nsec;    // window = column sectors [q0, q0 + nsec)
    bool wide;            // nsec > kMaxSec: generic kernel
};

}  // namespace

namespace {

// A layer as the run sees it: its ELT span [elt_begin, elt_end) and, for
// ara_run_portfolio, the explicit ascending member list (null = the whole span).
struct LayerI {
    uint32_t elt_begin, elt_end;
    double occ_retention, occ_limit, agg_retention, agg_limit;
    const uint32_t* list;
    uint32_t n_list;
    bool member(uint32_t col) const {
        if (col < elt_begin || col >= elt_end) return false;
        if (!list) return true;
        uint32_t lo = 0, hi = n_list;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) / 2;
            if (list[mid] == col) return true;
            if (list[mid] < col) lo = mid + 1; else hi = mid;
        }
        return false;
    }
    uint32_t n_members() const { return list ? n_list : elt_end - elt_begin; }
};

ara_status run_impl(ara_ctx* ctx, uint32_t n_layers, const LayerI* layers, uint32_t n_programs,
                    const uint32_t* program_layers, double* ylt, uint32_t* lossy, ara_run_stats* stats);

ara_status check_layer_terms(ara_ctx* ctx, uint32_t l, double occr, double occl, double aggr, double aggl) {
    if (!valid_retention(occr) || !valid_retention(aggr) || !valid_limit(occl) || !valid_limit(aggl))
        return fail(ctx, ARA_ERR_DOMAIN, "layer %u terms: retentions >= 0 finite, limits > 0", l);
    return ARA_OK;
}

}  // namespace

extern "C" ara_status ara_run(ara_ctx* ctx, uint32_t n_layers, const ara_layer* layers, double* ylt,
                              uint32_t* lossy, ara_run_stats* stats) {
    if (!ctx) return ARA_ERR_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    if (!ctx->d_table || ctx->n_elts == 0) return fail(ctx, ARA_ERR_STATE, "ara_load_elts has not succeeded");
    if (!ctx->yet_loaded) return fail(ctx, ARA_ERR_STATE, "ara_load_yet has not succeeded");
    if (n_layers == 0 || n_layers > ARA_MAX_LAYERS || !layers)
        return fail(ctx, ARA_ERR_INVALID_ARG, "n_layers must be in [1, %d]", ARA_MAX_LAYERS);
    if (classify(layers) == Mem::Device) return fail(ctx, ARA_ERR_INVALID_ARG, "layers must be host memory");
    std::vector<LayerI> li(n_layers);
    for (uint32_t l = 0; l < n_layers; ++l) {
        const ara_layer& L = layers[l];
        if (L.elt_begin >= L.elt_end || L.elt_end > ctx->n_elts)
            return fail(ctx, ARA_ERR_INVALID_ARG, "layer %u ELT range [%u,%u) invalid for %u ELTs", l, L.elt_begin,
                        L.elt_end, ctx->n_elts);
        ara_status st = check_layer_terms(ctx, l, L.occ_retention, L.occ_limit, L.agg_retention, L.agg_limit);
        if (st != ARA_OK) return st;
        li[l] = LayerI{L.elt_begin, L.elt_end, L.occ_retention, L.occ_limit, L.agg_retention, L.agg_limit, nullptr, 0};
    }
    return run_impl(ctx, n_layers, li.data(), 0, nullptr, ylt, lossy, stats);
}

extern "C" ara_status ara_run_portfolio(ara_ctx* ctx, uint32_t n_programs, const uint32_t* program_layers,
                                        uint32_t n_layers, const ara_layer_list* layers, double* ylt,
                                        uint32_t* lossy, ara_run_stats* stats) {
    if (!ctx) return ARA_ERR_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    if (!ctx->d_table || ctx->n_elts == 0) return fail(ctx, ARA_ERR_STATE, "ara_load_elts has not succeeded");
    if (!ctx->yet_loaded) return fail(ctx, ARA_ERR_STATE, "ara_load_yet has not succeeded");
    if (n_layers == 0 || n_layers > ARA_MAX_LAYERS || !layers)
        return fail(ctx, ARA_ERR_INVALID_ARG, "n_layers must be in [1, %d]", ARA_MAX_LAYERS);
    if (n_programs > ARA_MAX_PROGRAMS || (n_programs && !program_layers))
        return fail(ctx, ARA_ERR_INVALID_ARG, "n_programs must be in [0, %d] with program_layers", ARA_MAX_PROGRAMS);
    if (n_programs) {
        if (program_layers[0] != 0 || program_layers[n_programs] != n_layers)
            return fail(ctx, ARA_ERR_INVALID_ARG, "program_layers must run from 0 to n_layers");
        for (uint32_t q = 0; q < n_programs; ++q)
            if (program_layers[q + 1] <= program_layers[q])
                return fail(ctx, ARA_ERR_INVALID_ARG, "program %u has no layers", q);
    }
    std::vector<LayerI> li(n_layers);
    for (uint32_t l = 0; l < n_layers; ++l) {
        const ara_layer_list& L = layers[l];
        if (L.n_elts == 0 || !L.elts) return fail(ctx, ARA_ERR_INVALID_ARG, "layer %u has no ELTs", l);
        for (uint32_t q = 0; q < L.n_elts; ++q) {
            if (L.elts[q] >= ctx->n_elts)
                return fail(ctx, ARA_ERR_INVALID_ARG, "layer %u ELT %u not loaded", l, L.elts[q]);
            if (q && L.elts[q] <= L.elts[q - 1])
                return fail(ctx, ARA_ERR_INVALID_ARG, "layer %u ELT list not strictly ascending", l);
        }
        ara_status st = check_layer_terms(ctx, l, L.occ_retention, L.occ_limit, L.agg_retention, L.agg_limit);
        if (st != ARA_OK) return st;
        li[l] = LayerI{L.elts[0], L.elts[L.n_elts - 1] + 1, L.occ_retention, L.occ_limit, L.agg_retention,
                       L.agg_limit, L.elts, L.n_elts};
    }
    return run_impl(ctx, n_layers, li.data(), n_programs, program_layers, ylt, lossy, stats);
}

namespace {

// ---- fused YLT assembly over NVLink (world > 1; SURVEY §8e "fused P2P epilogue")
void p2p_release(ara_ctx* ctx) {
    for (int b = 0; b < 2; ++b) {
        for (int r = 0; r < ctx->world && r < kMaxPeers; ++r)
            if (ctx->peer_p2p[b][r] && r != ctx->rank) cudaIpcCloseMemHandle(ctx->peer_p2p[b][r]);
        for (int r = 0; r < kMaxPeers; ++r) ctx->peer_p2p[b][r] = nullptr;
        cudaFree(ctx->d_p2p[b]);
        ctx->d_p2p[b] = nullptr;
    }
    ctx->p2p_cap = 0;
    cudaGetLastError();
}

// Collective: make sure both global-YLT buffers hold `need` doubles and every
// rank has every other rank's buffers mapped (CUDA IPC handles exchanged with
// one NCCL all-gather).  All ranks reach the same verdict (an all-reduce of
// the per-rank outcome); on failure the run falls back to ncclAllGather.
ara_status p2p_ensure(ara_ctx* ctx, size_t need) {
    if (ctx->p2p_state < 0) return ARA_OK;
    if (ctx->p2p_state > 0 && ctx->p2p_cap >= need) return ARA_OK;
    const int world = ctx->world, rank = ctx->rank;
    cudaStream_t s = ctx->stream;
    p2p_release(ctx);
    uint64_t ok = 1;
    cudaIpcMemHandle_t mine[2];
    for (int b = 0; b < 2 && ok; ++b) {
        if (cudaMalloc(&ctx->d_p2p[b], need * sizeof(double)) != cudaSuccess ||
            cudaIpcGetMemHandle(&mine[b], ctx->d_p2p[b]) != cudaSuccess)
            ok = 0;
    }
    if (!ok) std::memset(mine, 0, sizeof(mine));
    cudaGetLastError();
    // exchange the handles: [world][2] x 64 B
    const size_t hb = sizeof(mine);
    char* d_h = nullptr;
    CK(cudaMalloc(&d_h, hb * (size_t)(world + 1)));
    CK(cudaMemcpyAsync(d_h + hb * (size_t)world, mine, hb, cudaMemcpyHostToDevice, s));
    NK(ncclAllGather(d_h + hb * (size_t)world, d_h, hb, ncclChar, ctx->comm, s));
    std::vector<cudaIpcMemHandle_t> all((size_t)world * 2);
    CK(cudaMemcpyAsync(all.data(), d_h, hb * (size_t)world, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(d_h);
    for (int r = 0; r < world && ok; ++r)
        for (int b = 0; b < 2 && ok; ++b) {
            if (r == rank) { ctx->peer_p2p[b][r] = ctx->d_p2p[b]; continue; }
            void* ptr = nullptr;
            if (cudaIpcOpenMemHandle(&ptr, all[(size_t)r * 2 + b], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) ok = 0;
            else ctx->peer_p2p[b][r] = static_cast<double*>(ptr);
        }
    cudaGetLastError();
    // every rank must agree
    ctx->h_small[0] = ok;
    CK(cudaMemcpyAsync(ctx->d_small, ctx->h_small, sizeof(uint64_t), cudaMemcpyHostToDevice, s));
    NK(ncclAllReduce(ctx->d_small, ctx->d_small, 1, ncclUint64, ncclMin, ctx->comm, s));
    CK(cudaMemcpyAsync(ctx->h_small, ctx->d_small, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (ctx->h_small[0] == 1) {
        ctx->p2p_state = 1;
        ctx->p2p_cap = need;
    } else {
        p2p_release(ctx);
        ctx->p2p_state = -1;
    }
    return ARA_OK;
}

ara_status run_impl(ara_ctx* ctx, uint32_t n_layers, const LayerI* layers, uint32_t n_programs,
                    const uint32_t* program_layers, double* ylt, uint32_t* lossy, ara_run_stats* stats) {
    Nvtx nvtx_("ara_run");
    const uint32_t world = (uint32_t)ctx->world;
    const uint64_t T_local = ctx->T_local, T_global = ctx->T_global;

    // Ranks must hold ara_partition's split (checked once per load, collective).
    if (ctx->lb_world) {
        uint64_t f = 0, c = 0;
        ara_partition(T_global, ctx->lb_world, ctx->lb_rank, &f, &c);
        if (f != ctx->first || c != T_local)
            return fail(ctx, ARA_ERR_INVALID_ARG, "loopback: the YET must be ara_partition(%llu, %d)[%d]",
                        (unsigned long long)T_global, ctx->lb_world, ctx->lb_rank);
    } else if (world == 1 && (ctx->first != 0 || T_local != T_global))
        return fail(ctx, ARA_ERR_INVALID_ARG, "a single-rank context must load the whole YET (first 0, %llu trials)",
                    (unsigned long long)T_global);
    if (world > 1 && !ctx->tiling_checked) {
        uint64_t f = 0, c = 0;
        ara_partition(T_global, ctx->world, ctx->rank, &f, &c);
        ctx->h_small[0] = (f == ctx->first && c == T_local) ? 0 : 1;
        CK(cudaMemcpyAsync(ctx->d_small, ctx->h_small, sizeof(uint64_t), cudaMemcpyHostToDevice, ctx->stream));
        NK(ncclAllReduce(ctx->d_small, ctx->d_small, 1, ncclUint64, ncclSum, ctx->comm, ctx->stream));
        CK(cudaMemcpyAsync(ctx->h_small, ctx->d_small, sizeof(uint64_t), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->h_small[0] != 0)
            return fail(ctx, ARA_ERR_INVALID_ARG, "ranks' YET ranges do not follow ara_partition(%llu, %d)",
                        (unsigned long long)T_global, ctx->world);
        ctx->tiling_checked = true;
    }

    const int fp32 = ctx->precision == ARA_F32_STORAGE;
    const uint32_t eps = fp32 ? 8 : 4;   // elements per 32-B sector
    const uint64_t Tpad = world > 1 ? (T_global + world - 1) / world : T_local;
    const uint64_t ld = world > 1 ? Tpad : (T_local ? T_local : 1);
    const uint32_t rows = n_layers + n_programs + 1;   // layers, programs, portfolio

    ara_status st = ensure(ctx, ctx->d_ylt_local, ctx->ylt_local_cap, (size_t)rows * ld);
    if (st != ARA_OK) return st;
    uint32_t* d_lossy = nullptr;
    const Mem ml = lossy ? classify(lossy) : Mem::Host;
    if (lossy) {
        if (ml == Mem::Device && ld == T_local) {
            d_lossy = lossy;
        } else {
            st = ensure(ctx, ctx->d_lossy, ctx->lossy_cap, (size_t)n_layers * ld);
            if (st != ARA_OK) return st;
            d_lossy = ctx->d_lossy;
        }
    }

    // Layer groups: consecutive layers on the same sector window share one
    // launch (one row load serves up to kMaxLB tower layers); a layer wider
    // than kMaxSec sectors runs alone in the generic kernel.
    // Fold mode: layers are folded in chunks of nlc (power of two <= 8) per
    // folded trial launch; groups never straddle a chunk.
    bool fold = ctx->run_mode == ARA_RUN_FOLD;
    for (uint32_t l = 0; l < n_layers && fold; ++l)
        if ((layers[l].elt_end + eps - 1) / eps - layers[l].elt_begin / eps > (uint32_t)kMaxSec) fold = false;
    uint32_t nlc = 1;
    while (nlc < n_layers && nlc < (uint32_t)kMaxFoldL) nlc <<= 1;
    std::vector<Group> groups;
    for (uint32_t l = 0; l < n_layers; ++l) {
        const uint32_t q0 = layers[l].elt_begin / eps, q1 = (layers[l].elt_end + eps - 1) / eps;
        const bool wide = q1 - q0 > (uint32_t)kMaxSec;
        if (!wide && !groups.empty() && !(fold && l % nlc == 0)) {
            Group& g = groups.back();
            if (!g.wide && g.q0 == q0 && g.nsec == q1 - q0 && g.nl < (uint32_t)kMaxLB) {
                ++g.nl;
                continue;
            }
        }
        groups.push_back({l, 1, q0, q1 - q0, wide});
    }
    cudaStream_t s = ctx->stream;
    host_trace("run prepared");
    CK(cudaEventRecord(ctx->ev[0], s));
    CK(cudaMemsetAsync(ctx->d_err, 0, 16, s));   // error word + the sparse kernel's gathered-slot counter

    // Chunk plan: CHUNKED streams the host YET in whole-trial chunks on the copy
    // stream, each chunk's kernels waiting only for that chunk.
    const bool stream_in = ctx->chunked_pending;
    std::vector<std::pair<uint64_t, uint64_t>> chunks;
    if (stream_in && T_local) {
        for (uint64_t t = 0; t < T_local; t += ctx->chunk_trials)
            chunks.push_back({t, (t + ctx->chunk_trials < T_local) ? t + ctx->chunk_trials : T_local});
    } else {
        chunks.push_back({0, T_local});
    }
    std::vector<cudaEvent_t> chunk_ev;
    // ARA_TIMELINE=<file>: a chunked run writes its copy/compute timeline (per
    // chunk: H2D copy start/end on the copy stream, kernels start/end on the
    // compute stream, ms from the first copy) as JSON -- the B200 analogue of
    // the paper's transfer/compute life-cycle grids
    static const char* tl_path = getenv("ARA_TIMELINE");
    std::vector<cudaEvent_t> tl_c0, tl_k0, tl_k1;   // chunk_ev is the copy end
    std::vector<uint64_t> ho_chunk;   // event index (relative) of each chunk boundary
    uint64_t h2d_bytes = 0;
    if (stream_in) {
        CK(cudaEventRecord(ctx->ev[5], s));
        CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->ev[5], 0));   // copies after prior work on s
        CK(cudaEventRecord(ctx->ev[6], ctx->copy_stream));
        const uint64_t* hoff = ctx->h_off;
        if (hoff) {
            CK(cudaMemcpyAsync(ctx->d_off_own, hoff, (T_local + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice,
                               ctx->copy_stream));
            h2d_bytes += (T_local + 1) * sizeof(uint64_t);
        }
        // host offsets are needed to size the id chunks
        std::vector<uint64_t> tmp;
        const uint64_t* ho = hoff;
        if (!ho) {
            tmp.resize(T_local + 1);
            CK(cudaMemcpy(tmp.data(), ctx->d_off, (T_local + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
            ho = tmp.data();
        }
        chunk_ev.resize(chunks.size());
        for (size_t c = 0; c < chunks.size(); ++c) {
            if (cudaEventCreateWithFlags(&chunk_ev[c], tl_path ? cudaEventDefault : cudaEventDisableTiming) !=
                cudaSuccess) {
                for (size_t q = 0; q < c; ++q) cudaEventDestroy(chunk_ev[q]);
                return fail(ctx, ARA_ERR_CUDA, "cudaEventCreate failed");
            }
        }
        ho_chunk.resize(chunks.size() + 1);
        for (size_t c = 0; c < chunks.size(); ++c) ho_chunk[c] = ho[chunks[c].first] - ho[0];
        ho_chunk[chunks.size()] = ho[T_local] - ho[0];
        const uint64_t nev_all = ho[T_local] - ho[0];
        const uint32_t pb = ctx->pack_bits;
        const uint64_t words_all = pb ? ara_packed_words(nev_all, pb) : 0;
        for (size_t c = 0; c < chunks.size(); ++c) {
            const uint64_t e0 = ho[chunks[c].first] - ho[0], e1 = ho[chunks[c].second] - ho[0];
            if (tl_path) {   // timeline: the chunk's copy start
                cudaEvent_t ev0 = nullptr;
                CK(cudaEventCreate(&ev0));
                tl_c0.push_back(ev0);
                CK(cudaEventRecord(ev0, ctx->copy_stream));
            }
            if (ctx->h_ids && e1 > e0) {
                CK(cudaMemcpyAsync(ctx->d_ids_own + e0, ctx->h_ids + e0, (e1 - e0) * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, ctx->copy_stream));
                h2d_bytes += (e1 - e0) * sizeof(uint32_t);
            }
            if (ctx->h_packed && e1 > e0) {   // the chunk's packed words (+ the word its last id spills into)
                const uint64_t w0 = (e0 * pb) >> 5;
                uint64_t w1 = ((e1 * pb + 31) >> 5) + 1;
                if (w1 > words_all) w1 = words_all;
                CK(cudaMemcpyAsync(ctx->d_packed_own + w0, ctx->h_packed + w0, (w1 - w0) * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, ctx->copy_stream));
                h2d_bytes += (w1 - w0) * sizeof(uint32_t);
            }
            CK(cudaEventRecord(chunk_ev[c], ctx->copy_stream));
        }
        CK(cudaEventRecord(ctx->ev[7], ctx->copy_stream));
    }

    // Kernels.
    const TableGeo& geo = ctx->geo;
    const uint32_t spb = geo.epb / eps;   // sectors per block row
    // Fused YLT assembly: one launch group per chunk (no wide layers, no
    // programs, one fold chunk) with a kernel whose epilogue stores to peers.
    bool p2p_ok_kernel = true;   // every trial kernel has the peer-store epilogue
    bool single_group = groups.size() == 1 && !groups[0].wide && n_programs == 0 &&
                        (!fold || (n_layers + nlc - 1) / nlc == 1) && world <= (uint32_t)kMaxPeers;
    bool use_p2p = false;
    if (world > 1 && ctx->use_p2p && p2p_ok_kernel && single_group) {
        st = p2p_ensure(ctx, (size_t)rows * T_global);
        if (st != ARA_OK) return st;
        use_p2p = ctx->p2p_state > 0;
    } else if (ctx->lb_world) {
        if (!p2p_ok_kernel || !single_group)
            return fail(ctx, ARA_ERR_INVALID_ARG, "loopback: needs a single-launch run with a peer-store kernel");
        // the two global-YLT buffers are local; bytes 0xff (NaN) wherever no store lands
        const size_t need = (size_t)rows * T_global;
        if (ctx->p2p_cap < need) {
            for (int b = 0; b < 2; ++b) {
                cudaFree(ctx->d_p2p[b]);
                ctx->d_p2p[b] = nullptr;
            }
            ctx->p2p_cap = 0;
            for (int b = 0; b < 2; ++b) {
                CK(cudaMalloc(&ctx->d_p2p[b], need * sizeof(double)));
                CK(cudaMemsetAsync(ctx->d_p2p[b], 0xff, need * sizeof(double), ctx->stream));
                ctx->peer_p2p[b][0] = ctx->d_p2p[b];
            }
            ctx->p2p_cap = need;
        }
        use_p2p = true;
    }
    const int p2p_buf = ctx->p2p_next;
    TrialParams base{};
    if (use_p2p) {
        base.n_peers = world;   // loopback: 1, the local buffer
        for (uint32_t r = 0; r < world; ++r) base.peer_ylt[r] = ctx->peer_p2p[p2p_buf][r];
        base.peer_ld = T_global;
        base.peer_t0 = ctx->first;
    }
    base.off = ctx->d_off;
    base.ids = ctx->d_ids;
    base.catalog = ctx->catalog;
    base.table = ctx->d_table;
    base.row_stride = geo.epb;
    base.block_stride = geo.block_elems;
    base.ylt = ctx->d_ylt_local;
    base.ld = ld;
    base.lossy = d_lossy;
    base.err = ctx->d_err;
    base.n_gathered = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ctx->d_err) + 8);
    uint32_t bc_launches = 0;   // launches of the sparse kernel (their gathered slots are counted)
    base.portfolio_row = n_layers + n_programs;
    uint32_t launches = 0;
    int used_variant = fold ? -2 : -1;
    double used_occupancy = 1.0;
    std::vector<void*> wide_free;   // per-run column lists / terms of wide layers
    // per-group window setup shared by the direct and fold launches
    auto setup_window = [&](const Group& g, TrialParams& p) {
        for (uint32_t q = 0; q < g.nl; ++q) {
            const LayerI& L = layers[g.l0 + q];
            p.lw[q] = {L.occ_retention, L.occ_limit, L.agg_retention, L.agg_limit};
        }
        for (uint32_t sct = 0; sct < (uint32_t)kMaxSec; ++sct) {
            const uint32_t qq = g.q0 + (sct < g.nsec ? sct : 0);
            p.sec_off[sct] = (uint64_t)(qq / spb) * geo.block_elems + (uint64_t)(qq % spb) * eps;
        }
        // Row-occupancy bitmap of the window's column block (windows inside one
        // block), used when at most half of the block's rows are occupied: the
        // paper's ELTs hold 10k-30k losses over a catalogue of millions,
        // so most lookups hit all-zero rows; on dense tables the extra occupancy
        // read would only cost time (measured: +7 % at 100 % occupancy).
        const uint32_t blk = g.q0 / spb;
        const bool sparse = blk < ctx->occ_rows.size() && 2ull * ctx->occ_rows[blk] <= (uint64_t)ctx->catalog + 1;
        p.bm = (g.nsec <= spb && (g.q0 % spb) + g.nsec <= spb && !ctx->no_skip && sparse)
                   ? reinterpret_cast<const uint32_t*>(static_cast<const char*>(ctx->d_table) + geo.bm_off) +
                         (uint64_t)(g.q0 / spb) * geo.bm_words
                   : nullptr;
        // packed rows of the block (built by load_elts for sparse blocks)
        p.pk = p.bm ? static_cast<const void*>(static_cast<const char*>(ctx->d_table) + geo.pk_off +
                                               (size_t)(g.q0 / spb) * ((size_t)ctx->catalog + 1) * kPackBytes)
                    : nullptr;
        p.pk_col0 = (g.q0 % spb) * eps;
        p.pk_wmask = g.nsec * eps >= 32 ? 0xffffffffu : (1u << (g.nsec * eps)) - 1u;
        for (uint32_t q = 0; q < g.nl; ++q) {
            const LayerI& L = layers[g.l0 + q];
            for (uint32_t w = 0; w < (uint32_t)kMaxWin; ++w) {
                const uint32_t col = g.q0 * eps + w;
                if (w / eps < g.nsec && L.member(col))
                    p.term[q][w] = make_double2(ctx->terms[col].deductible, ctx->terms[col].limit);
                else
                    p.term[q][w] = make_double2(INFINITY, INFINITY);   // contributes exactly +0
            }
        }
        p.same_terms = 1u;
        for (uint32_t q = 1; q < g.nl; ++q)
            for (uint32_t w = 0; w < (uint32_t)kMaxWin; ++w)
                if (std::memcmp(&p.term[q][w], &p.term[0][w], sizeof(double2)) != 0) p.same_terms = 0u;
    };
    const uint32_t n_chunks_fold = (n_layers + nlc - 1) / nlc;
    const uint64_t fold_rows = (uint64_t)ctx->catalog + 1;
    CK(cudaEventRecord(ctx->ev[1], s));
    if (fold) {
        // a0': fold the catalogue once per run (all layers), bit-identical per-event values
        st = ensure(ctx, ctx->d_fold, ctx->fold_cap, (size_t)n_chunks_fold * fold_rows * nlc);
        if (st != ARA_OK) return st;
        for (const Group& g : groups) {
            TrialParams p = base;
            p.n_layers = g.nl;
            setup_window(g, p);
            p.fold = ctx->d_fold + (uint64_t)(g.l0 / nlc) * fold_rows * nlc;
            p.fold_stride = nlc;
            p.fold_col0 = g.l0 % nlc;
            CK(launch_fold(p, fp32, g.nsec, s));
            ++launches;
        }
    }
    const bool tl = tl_path && stream_in && tl_c0.size() == chunks.size();
    auto tl_mark = [&](std::vector<cudaEvent_t>& v) -> cudaError_t {
        cudaEvent_t e = nullptr;
        cudaError_t r = cudaEventCreate(&e);
        if (r == cudaSuccess) { v.push_back(e); r = cudaEventRecord(e, s); }
        return r;
    };
    for (size_t c = 0; c < chunks.size(); ++c) {
        Nvtx nvtx_chunk(stream_in ? "ara_run chunk" : "ara_run launch");
        if (tl && c > 0) CK(tl_mark(tl_k1));   // the previous chunk's kernels are done
        if (stream_in) CK(cudaStreamWaitEvent(s, chunk_ev[c], 0));
        if (tl) CK(tl_mark(tl_k0));
        if (stream_in && ctx->h_packed) {   // F3: unpack this chunk's ids on the device
            const uint64_t e0 = ho_chunk[c], e1 = ho_chunk[c + 1];
            CK(launch_unpack(ctx->d_packed_own, ctx->pack_bits, e0, e1, ctx->d_ids_own, s));
        }
        if (fold) {
            for (uint32_t fc = 0; fc < n_chunks_fold; ++fc) {
                TrialParams p = base;
                p.t_begin = chunks[c].first;
                p.t_end = chunks[c].second;
                p.n_layers = (n_layers - fc * nlc) < nlc ? (n_layers - fc * nlc) : nlc;
                p.ylt_row0 = fc * nlc;
                p.portfolio_mode = fc == 0 ? 0 : 1;
                for (uint32_t q = 0; q < p.n_layers; ++q) {
                    const LayerI& L = layers[fc * nlc + q];
                    p.lw[q] = {L.occ_retention, L.occ_limit, L.agg_retention, L.agg_limit};
                }
                p.fold = ctx->d_fold + (uint64_t)fc * fold_rows * nlc;
                p.fold_stride = nlc;
                // The sparse kernel gathers o(e) for the occupied rows only when
                // every layer of the chunk lies in one sparse column block (a
                // zero row folds to o = 0, so skipping it adds an exact +0); the
                // result equals the direct sparse kernel's bit for bit.
                int bc_blk = ctx->fold_bc && nlc <= 4 && !ctx->no_skip ? 0 : -1;
                for (uint32_t q = 0; q < p.n_layers && bc_blk >= 0; ++q) {
                    const LayerI& L = layers[fc * nlc + q];
                    const uint32_t q0 = L.elt_begin / eps, q1 = (L.elt_end + eps - 1) / eps;
                    const int blk = (int)(q0 / spb);
                    if ((q1 - 1) / spb != q0 / spb || (q > 0 && blk != bc_blk)) bc_blk = -1;
                    else bc_blk = blk;
                }
                if (bc_blk >= 0 && (size_t)bc_blk < ctx->occ_rows.size() &&
                    2ull * ctx->occ_rows[bc_blk] <= (uint64_t)ctx->catalog + 1) {
                    p.bm = reinterpret_cast<const uint32_t*>(static_cast<const char*>(ctx->d_table) + geo.bm_off) +
                           (uint64_t)bc_blk * geo.bm_words;
                    p.pk = nullptr;
                    used_variant = 31;
                    used_occupancy = (double)ctx->occ_rows[bc_blk] / ((double)ctx->catalog + 1.0);
                    CK(launch_trials_bc(p, -1, ctx->n_sm, s));
                } else {
                    CK(launch_trials_folded(p, (int)(100 * ctx->grid_mult), s));
                }
                ++launches;
            }
            continue;
        }
        for (size_t gi = 0; gi < groups.size(); ++gi) {
            const Group& g = groups[gi];
            TrialParams p = base;
            p.t_begin = chunks[c].first;
            p.t_end = chunks[c].second;
            p.n_layers = g.nl;
            p.ylt_row0 = g.l0;
            p.portfolio_mode = gi == 0 ? 0 : 1;
            for (uint32_t q = 0; q < g.nl; ++q) {
                const LayerI& L = layers[g.l0 + q];
                p.lw[q] = {L.occ_retention, L.occ_limit, L.agg_retention, L.agg_limit};
            }
            if (g.wide) {
                const LayerI& L = layers[g.l0];
                std::vector<uint32_t> wcols;
                std::vector<double2> wterms;
                for (uint32_t col = L.elt_begin; col < L.elt_end; ++col)
                    if (L.member(col)) {
                        wcols.push_back(col);
                        wterms.push_back(make_double2(ctx->terms[col].deductible, ctx->terms[col].limit));
                    }
                uint32_t* d_wc = nullptr;
                double2* d_wt = nullptr;
                CK(cudaMallocAsync(&d_wc, wcols.size() * sizeof(uint32_t), s));
                CK(cudaMallocAsync(&d_wt, wterms.size() * sizeof(double2), s));
                CK(cudaMemcpyAsync(d_wc, wcols.data(), wcols.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
                CK(cudaMemcpyAsync(d_wt, wterms.data(), wterms.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
                wide_free.push_back(d_wc);
                wide_free.push_back(d_wt);
                const int grid = trial_kernel_grid(fp32, g.nsec, 1, 0);
                CK(launch_trials_wide(p, fp32, d_wc, d_wt, (uint32_t)wcols.size(), grid, s));
            } else {
                setup_window(g, p);
                // Kernel choice (measured): windows over a sparse
                // column block (occupancy bitmap + packed rows set) use the
                // ballot-compacted rounds kernel (30); dense fp64 windows of <= 4
                // sectors the cooperative cp.async ring (12); other dense windows the
                // register pipeline at 3 CTAs/SM (5) for single layers, 2 CTAs/SM
                // (0) for shared-window towers.  ARA_KERNEL forces one (A/B runs).
                int variant = ctx->kernel_variant;
                if (variant == 30 && !p.bm) variant = -1;   // bc needs the bitmap and packed rows
                if (variant < 0 && p.bm) variant = 30;
                if (variant != 30) p.bm = nullptr, p.pk = nullptr;   // the dense kernels read every row
                used_occupancy = p.bm ? (double)ctx->occ_rows[g.q0 / spb] / ((double)ctx->catalog + 1.0) : 1.0;
                if (variant == 30) ++bc_launches;
                if (variant < 0) variant = (!fp32 && g.nsec <= 4) ? 12 : (g.nl == 1 ? 5 : 0);
                used_variant = variant;
                if (ctx->l2_persist) {
                    const char* tb = static_cast<const char*>(ctx->d_table);
                    const size_t blk = g.q0 / spb;
                    if (p.bm)   // the block's packed rows (its 250 KB bitmap is hot in any case)
                        set_l2_window(ctx, p.pk, ((size_t)ctx->catalog + 1) * kPackBytes);
                    else
                        set_l2_window(ctx, tb + blk * geo.block_elems * geo.esz, geo.block_elems * geo.esz);
                }
                const int grid = (int)(trial_kernel_grid(fp32, g.nsec, (int)g.nl, variant) * ctx->grid_mult);
                CK(launch_trials(p, fp32, g.nsec, grid > 0 ? grid : 1, variant, s));
            }
            ++launches;
        }
    }
    if (tl && !chunks.empty()) CK(tl_mark(tl_k1));
    if (n_programs) {   // program rows from the layer rows (Alg. 1 l.1)
        uint32_t* d_pl = nullptr;
        CK(cudaMallocAsync(&d_pl, (n_programs + 1) * sizeof(uint32_t), s));
        CK(cudaMemcpyAsync(d_pl, program_layers, (n_programs + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        CK(launch_program_sums(ctx->d_ylt_local, ld, T_local, n_programs, d_pl, n_layers, s));
        wide_free.push_back(d_pl);
        ++launches;
    }
    CK(cudaEventRecord(ctx->ev[2], s));
    if (ctx->l2_persist) set_l2_window(ctx, nullptr, 0);   // the stream may be the caller's
    for (void* q : wide_free) CK(cudaFreeAsync(q, s));
    if (!tl)
        for (auto e : chunk_ev) cudaEventDestroy(e);   // safe: destruction defers until complete
    if (stream_in) {
        ctx->chunked_pending = false;   // later runs reuse the device copy
    }

    // YLT assembly across ranks (a9).  Fused path: the kernels already stored
    // every trial's YLT entries into every rank's global buffer over NVLink;
    // the all-reduce of the error words below is the barrier after which all
    // of them are complete.  Otherwise one ncclAllGather per YLT row.
    double* d_full = ctx->d_ylt_local;
    uint64_t ld_full = ld;
    CK(cudaEventRecord(ctx->ev[3], s));
    if (use_p2p) {
        d_full = ctx->d_p2p[p2p_buf];
        ld_full = T_global;
    } else if (world > 1) {
        st = ensure(ctx, ctx->d_ylt_gather, ctx->ylt_gather_cap, (size_t)rows * world * Tpad);
        if (st != ARA_OK) return st;
        NK(ncclGroupStart());
        for (uint32_t r = 0; r < rows; ++r)
            NK(ncclAllGather(ctx->d_ylt_local + (uint64_t)r * ld, ctx->d_ylt_gather + (uint64_t)r * world * Tpad, Tpad,
                             ncclDouble, ctx->comm, s));
        NK(ncclGroupEnd());
        if (Tpad * world == T_global) {
            d_full = ctx->d_ylt_gather;
        } else {
            st = ensure(ctx, ctx->d_ylt_global, ctx->ylt_global_cap, (size_t)rows * T_global);
            if (st != ARA_OK) return st;
            for (uint32_t rk = 0; rk < world; ++rk) {
                uint64_t f = 0, c = 0;
                ara_partition(T_global, ctx->world, (int)rk, &f, &c);
                if (c)
                    CK(cudaMemcpy2DAsync(ctx->d_ylt_global + f, T_global * sizeof(double),
                                         ctx->d_ylt_gather + (uint64_t)rk * Tpad, world * Tpad * sizeof(double),
                                         c * sizeof(double), rows, cudaMemcpyDeviceToDevice, s));
            }
            d_full = ctx->d_ylt_global;
        }
        ld_full = T_global;
    }
    if (world > 1) {   // every rank must see the same verdict: max of the error words, on the device
        CK(cudaMemsetAsync(ctx->d_small, 0, sizeof(uint64_t), s));
        CK(cudaMemcpyAsync(ctx->d_small, ctx->d_err, sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        NK(ncclAllReduce(ctx->d_small, ctx->d_small, 1, ncclUint64, ncclMax, ctx->comm, s));
        CK(cudaMemcpyAsync(ctx->h_small, ctx->d_small, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaEventRecord(ctx->ev[4], s));

    // Outputs.
    if (ylt) {
        const cudaMemcpyKind kind = classify(ylt) == Mem::Device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (ld_full == T_global)
            CK(cudaMemcpyAsync(ylt, d_full, (size_t)rows * T_global * sizeof(double), kind, s));
        else
            CK(cudaMemcpy2DAsync(ylt, T_global * sizeof(double), d_full, ld_full * sizeof(double),
                                 T_global * sizeof(double), rows, kind, s));
    }
    if (lossy && d_lossy != lossy && T_local) {
        const cudaMemcpyKind kind = ml == Mem::Device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        CK(cudaMemcpy2DAsync(lossy, T_local * sizeof(uint32_t), d_lossy, ld * sizeof(uint32_t),
                             T_local * sizeof(uint32_t), n_layers, kind, s));
    }
    CK(cudaMemcpyAsync(ctx->h_small + 4, ctx->d_err, 16, cudaMemcpyDeviceToHost, s));   // [4] error word, [5] gathered
    if (T_local) {
        CK(cudaMemcpyAsync(ctx->h_small + 1, ctx->d_off, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->h_small + 2, ctx->d_off + T_local, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    }
    CK(cudaEventRecord(ctx->ev[5], s));
    host_trace("run launched");
    CK(cudaStreamSynchronize(s));
    host_trace("run synced");
    if (stream_in) CK(cudaStreamSynchronize(ctx->copy_stream));
    if (tl && tl_k0.size() == chunks.size() && tl_k1.size() == chunks.size()) {
        if (FILE* f = fopen(tl_path, "w")) {
            auto rel = [&](cudaEvent_t e) { float ms = 0.f; cudaEventElapsedTime(&ms, tl_c0[0], e); return ms; };
            fprintf(f, "{\"chunks\": [");
            for (size_t c = 0; c < chunks.size(); ++c)
                fprintf(f, "%s{\"chunk\": %zu, \"trials\": [%llu, %llu], \"copy_ms\": [%.4f, %.4f], \"kernel_ms\": [%.4f, %.4f]}",
                        c ? ", " : "", c, (unsigned long long)chunks[c].first, (unsigned long long)chunks[c].second,
                        rel(tl_c0[c]), rel(chunk_ev[c]), rel(tl_k0[c]), rel(tl_k1[c]));
            fprintf(f, "]}\n");
            fclose(f);
        }
    }
    if (tl)
        for (auto e : chunk_ev) cudaEventDestroy(e);
    for (auto e : tl_c0) cudaEventDestroy(e);
    for (auto e : tl_k0) cudaEventDestroy(e);
    for (auto e : tl_k1) cudaEventDestroy(e);
    const uint32_t bits = (uint32_t)(ctx->h_small[world == 1 ? 4 : 0] & 0xffffffffu);   // world > 1: all-reduced
    st = device_errors(ctx, bits);
    if (st != ARA_OK) {
        ctx->last_layers = 0;
        return st;
    }
    ctx->last_layers = n_layers;
    ctx->last_rows = rows;
    ctx->d_last_full = d_full;
    ctx->last_ld_local = ld;
    ctx->run_T_global = T_global;
    ctx->run_T_local = T_local;
    if (use_p2p) ctx->p2p_next ^= 1;
    if (stats) {
        const uint64_t nev = T_local ? ctx->h_small[2] - ctx->h_small[1] : 0;
        uint64_t lookups = 0;
        for (uint32_t l = 0; l < n_layers; ++l) lookups += nev * layers[l].n_members();
        stats->n_trials_local = T_local;
        stats->n_events_local = nev;
        stats->n_lookups_local = lookups;
        stats->kernel_ms = ev_ms(ctx->ev[1], ctx->ev[2]);
        stats->allgather_ms = ev_ms(ctx->ev[3], ctx->ev[4]);
        stats->total_ms = ev_ms(ctx->ev[0], ctx->ev[5]);
        stats->h2d_ms = stream_in ? ev_ms(ctx->ev[6], ctx->ev[7]) : 0.0;
        stats->h2d_bytes = h2d_bytes;
        stats->n_kernel_launches = launches;
        stats->kernel_variant = used_variant;
        // fraction of events whose packed slot the sparse kernel gathered (its
        // shared-memory filter's pair part adds the unoccupied partners of
        // occupied rows), else the table's occupied-row fraction / 1.0
        stats->occupancy = bc_launches && nev ? (double)ctx->h_small[5] / ((double)nev * bc_launches) : used_occupancy;
    }
    return ARA_OK;
}

}  // namespace

// ============================================================ metrics
extern "C" ara_status ara_metrics(ara_ctx* ctx, uint32_t n_rp, const double* return_periods, uint64_t* k,
                                  double* pml, double* tvar, double* device_ms) {
    Nvtx nvtx_("ara_metrics");
    if (!ctx) return ARA_ERR_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    if (ctx->last_layers == 0) return fail(ctx, ARA_ERR_STATE, "no successful ara_run yet");
    if (n_rp == 0 || n_rp > ARA_MAX_RP || !return_periods || !pml || !tvar)
        return fail(ctx, ARA_ERR_INVALID_ARG, "n_rp must be in [1, %d] with non-NULL arrays", ARA_MAX_RP);
    // the last run's YET (a later ara_load_yet does not change it); loopback:
    // the shard, as if it were the whole YLT
    const uint64_t T = ctx->lb_world ? ctx->run_T_local : ctx->run_T_global;
    uint64_t hk[ARA_MAX_RP];
    for (uint32_t r = 0; r < n_rp; ++r)
        if (ara_return_period_rank(T, return_periods[r], &hk[r]) != ARA_OK)
            return fail(ctx, ARA_ERR_DOMAIN, "return period %g outside [1, %llu]", return_periods[r],
                        (unsigned long long)T);
    const uint32_t rows = ctx->last_rows;
    const double* d_y;
    uint64_t ld;
    if (ctx->world > 1) {
        d_y = ctx->d_last_full;   // the run's global YLT (fused buffer or all-gather output)
        ld = T;
    } else {
        d_y = ctx->d_ylt_local;
        ld = ctx->last_ld_local;
    }
    int nblk = (int)((T + 4095) / 4096);
    // grid: ARA_METRICS_BLOCKS blocks per SM over all rows (A/B knob; fractional allowed)
    static const double blk_mult = [] { const char* v = getenv("ARA_METRICS_BLOCKS"); return v ? atof(v) : 1.0; }();
    int maxblk = (int)(blk_mult * ctx->n_sm / rows + 0.5);
    if (maxblk < 1) maxblk = 1;
    if (nblk > maxblk) nblk = maxblk;
    if (nblk < 1) nblk = 1;
    CK(metrics_alloc(ctx->ms, rows, n_rp, nblk > 2 * ctx->n_sm ? nblk : 2 * ctx->n_sm));   // + cooperative grid
    cudaStream_t s = ctx->stream;
    CK(cudaEventRecord(ctx->ev[0], s));
    // Distributed select (F4) on large global YLTs: every rank histograms only
    // its own shard and the histograms are all-reduced, instead of every rank
    // sweeping the whole global YLT (which grows with N under weak scaling).
    // Crossover measured at N = 4 weak (4M trials): the graph-launched global
    // sweep 0.198 ms vs the eager distributed select 0.274 ms, so the
    // distributed form starts at 6M trials (profiles/r02_final2_fw_n4*.json).
    // (world 1 with ARA_METRICS_DIST=1 or loopback: the same passes with an identity reduce)
    const bool dist = ctx->lb_world > 0 || ctx->metrics_dist > 0 ||
                      (ctx->world > 1 && ctx->metrics_dist < 0 && T >= 6000000);
    if (dist) {
        int nerr = 0;
        const uint64_t Tl = ctx->run_T_local;
        int nb = (int)((Tl + 4095) / 4096);
        if (nb > maxblk) nb = maxblk;
        if (nb < 1) nb = 1;
        CK(launch_metrics_dist(ctx->d_ylt_local, Tl, ctx->last_ld_local, rows, n_rp, hk,
                               ctx->ms, nb, ctx->comm, s, &nerr));
        if (nerr) return fail(ctx, ARA_ERR_NCCL, "NCCL all-reduce in the distributed metrics failed");
    } else {
        CK(launch_metrics(d_y, T, ld, rows, n_rp, hk, ctx->ms, nblk, s));
    }
    CK(cudaEventRecord(ctx->ev[1], s));
    std::vector<double> out((size_t)rows * n_rp * 2);
    CK(cudaMemcpyAsync(out.data(), ctx->ms.out, out.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    host_trace("metrics launched");
    CK(cudaStreamSynchronize(s));
    host_trace("metrics synced");
    for (uint32_t r = 0; r < rows; ++r)
        for (uint32_t q = 0; q < n_rp; ++q) {
            pml[(size_t)r * n_rp + q] = out[((size_t)r * n_rp + q) * 2 + 0];
            tvar[(size_t)r * n_rp + q] = out[((size_t)r * n_rp + q) * 2 + 1];
        }
    if (k)
        for (uint32_t q = 0; q < n_rp; ++q) k[q] = hk[q];
    if (device_ms) *device_ms = ev_ms(ctx->ev[0], ctx->ev[1]);
    return ARA_OK;
}

// ============================================================ EP curve
extern "C" ara_status ara_ep_curve(ara_ctx* ctx, uint32_t n_points, const double* thresholds, uint64_t* counts) {
    Nvtx nvtx_("ara_ep_curve");
    if (!ctx) return ARA_ERR_INVALID_ARG;
    CK(cudaSetDevice(ctx->device));
    if (ctx->last_layers == 0) return fail(ctx, ARA_ERR_STATE, "no successful ara_run yet");
    if (n_points == 0 || n_points > ARA_MAX_EP_POINTS || !thresholds || !counts)
        return fail(ctx, ARA_ERR_INVALID_ARG, "n_points must be in [1, %d] with non-NULL arrays", ARA_MAX_EP_POINTS);
    if (classify(thresholds) == Mem::Device || classify(counts) == Mem::Device)
        return fail(ctx, ARA_ERR_INVALID_ARG, "thresholds and counts must be host memory");
    for (uint32_t i = 0; i < n_points; ++i) {
        if (std::isnan(thresholds[i])) return fail(ctx, ARA_ERR_DOMAIN, "threshold %u is NaN", i);
        if (i && thresholds[i] < thresholds[i - 1])
            return fail(ctx, ARA_ERR_DOMAIN, "thresholds must be non-decreasing (index %u)", i);
    }
    const uint32_t rows = ctx->last_rows;
    const size_t n = n_points;
    const size_t bytes = n * sizeof(double) + (n + 1) * rows * sizeof(unsigned long long) + n * rows * sizeof(uint64_t);
    ara_status st = ensure(ctx, ctx->d_ep, ctx->ep_cap, bytes);
    if (st != ARA_OK) return st;
    double* d_x = reinterpret_cast<double*>(ctx->d_ep);
    unsigned long long* d_hist = reinterpret_cast<unsigned long long*>(ctx->d_ep + n * sizeof(double));
    uint64_t* d_cnt = reinterpret_cast<uint64_t*>(ctx->d_ep + n * sizeof(double) +
                                                  (n + 1) * rows * sizeof(unsigned long long));
    cudaStream_t s = ctx->stream;
    CK(cudaMemcpyAsync(d_x, thresholds, n * sizeof(double), cudaMemcpyHostToDevice, s));
    // this rank's trials of the last run (world 1: all of them); the shards' counts add up
    CK(launch_ep_curve(ctx->d_ylt_local, ctx->run_T_local, ctx->last_ld_local, rows, d_x, n_points, d_hist, d_cnt,
                       ctx->n_sm, s));
    if (ctx->world > 1) NK(ncclAllReduce(d_cnt, d_cnt, n * rows, ncclUint64, ncclSum, ctx->comm, s));
    CK(cudaMemcpyAsync(counts, d_cnt, n * rows * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return ARA_OK;
}
