// ara_api.cu -- the C ABI of libara (include/ara.h): validation, the host
// planner that lays the portfolio out in HBM (event-major direct-access
// index, presence bitmap, slot tables), YET handling, and launch plumbing.
// All arithmetic of the method runs in the kernels (ara_kernels.cu,
// ara_measures.cu); this file only validates, lays out and copies.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>     // header-only NVTX v3: host ranges for nsys / ncu --nvtx

#include "ara_internal.cuh"
#include "ara_measures.cuh"

using namespace ara;

namespace {

thread_local std::string g_err;

// NVTX range for the lifetime of a scope (entry points of the C ABI)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int fail(int code, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CU(call)                                                                        \
    do {                                                                                \
        cudaError_t _e = (call);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(ARA_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(_e),     \
                        __FILE__, __LINE__);                                            \
    } while (0)

// Every entry point starts here: launches are checked with cudaGetLastError, so
// an error some earlier runtime call left behind (a destroy's cudaFree, a probe)
// must not be reported against this call.
cudaError_t enter_device(int device) {
    cudaGetLastError();
    return cudaSetDevice(device);
}

bool is_device_ptr(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

template <typename T>
cudaError_t dalloc(T **p, size_t n) {
    return cudaMalloc(reinterpret_cast<void **>(p), (n ? n : 1) * sizeof(T));
}

// grow-once device scratch
template <typename T>
cudaError_t grow(T **p, uint64_t &cap, uint64_t need) {
    if (cap >= need) return cudaSuccess;
    cudaFree(*p);
    *p = nullptr;
    cap = 0;
    cudaError_t e = dalloc(p, need);
    if (e == cudaSuccess) cap = need;
    return e;
}

uint64_t env_u64(const char *name, uint64_t dflt) {
    const char *v = getenv(name);
    return v && *v ? strtoull(v, nullptr, 10) : dflt;
}

}  // namespace

constexpr uint32_t kOutDoubles = 3 * 4 * (ARA_MAX_PORTFOLIO_LAYERS + 1);   // batched measures: 3 x n_rp x tables
constexpr uint32_t kMaxBatches = 256;       // trial batches of one split-path run

struct ara_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int num_sms = 0;
    RunStatus *d_status = nullptr;
    RunStatus *h_status = nullptr;     // pinned
    double *h_out = nullptr;           // pinned [kOutDoubles]: measures results (pml, tvar, var) per RP (x layers)
    uint32_t *d_ep = nullptr;          // exceedance-curve sort scratch
    uint64_t ep_capacity = 0;
    MeasuresScratch ms;
    // split path: the compaction runs on its own stream, a batch ahead of the
    // sampler on the context stream (two pair slots)
    cudaStream_t cstream = nullptr;
    unsigned char *d_slots = nullptr;  // 2 slots of batch x cap pairs
    uint64_t slots_capacity = 0;       // bytes
    unsigned char *d_pool = nullptr;   // overflow pool (exactly sized per run)
    uint64_t pool_capacity = 0;        // bytes
    uint64_t *d_pool_off = nullptr;
    uint64_t pool_off_capacity = 0;
    uint32_t *d_counts = nullptr;      // pairs per trial
    uint64_t counts_capacity = 0;
    unsigned long long *d_sched = nullptr;   // [2 kMaxBatches + 4] scheduler counters of one run
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};   // run begin / end, redo begin / end
    cudaEvent_t tev[4 * kMaxBatches] = {};                      // per-batch kernel timings
    double last_ms[3] = {0.0, 0.0, 0.0};                        // compact, sample, redo
    uint32_t last_launches = 0, last_batches = 0;               // kernels launched by the last ara_run
    // ARA_ASYNC: errors latched on the device until ara_ctx_synchronize, the
    // last run's timings computed when asked for
    bool async_pending = false;
    unsigned int latched_bad = 0, latched_nonconv = 0, latched_short = 0;
    bool timing_pending = false, timing_tail = false;
    uint32_t timing_batches = 0;
};

// fold the error counters latched by ARA_ASYNC runs into the host latch and
// clear them on the device (synchronises the context stream)
static cudaError_t fold_latched(ara_ctx *c) {
    if (!c->async_pending) return cudaSuccess;
    cudaError_t e = cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return e;
    c->latched_bad += c->h_status->bad_event;
    c->latched_nonconv += c->h_status->nonconverged;
    c->latched_short += c->h_status->pool_short;
    c->async_pending = false;
    return cudaMemsetAsync(reinterpret_cast<unsigned char *>(c->d_status) + kRunCounters, 0,
                           sizeof(RunStatus) - kRunCounters, c->stream);
}

// device times of the last run's kernels (waits for its last event)
static cudaError_t compute_timings(ara_ctx *c) {
    if (!c->timing_pending) return cudaSuccess;
    cudaError_t e = cudaEventSynchronize(c->timing_tail ? c->ev[3] : c->ev[1]);
    if (e != cudaSuccess) return e;
    double a = 0.0, b = 0.0, r = 0.0;
    for (uint32_t q = 0; q < c->timing_batches; ++q) {
        float x = 0, z = 0;
        if ((e = cudaEventElapsedTime(&x, c->tev[4 * q], c->tev[4 * q + 1])) != cudaSuccess) return e;
        if ((e = cudaEventElapsedTime(&z, c->tev[4 * q + 2], c->tev[4 * q + 3])) != cudaSuccess) return e;
        a += x; b += z;
    }
    if (!c->timing_batches) {
        float x = 0;
        if ((e = cudaEventElapsedTime(&x, c->ev[0], c->ev[1])) != cudaSuccess) return e;
        b = x;
    }
    if (c->timing_tail) {
        float x = 0;
        if ((e = cudaEventElapsedTime(&x, c->ev[2], c->ev[3])) != cudaSuccess) return e;
        r = x;
    }
    c->last_ms[0] = a; c->last_ms[1] = b; c->last_ms[2] = r;
    c->timing_pending = false;
    return cudaSuccess;
}

// Per input XELT record, shared by every (layer, XELT) slot and every
// kernel group that covers the record's XELT: the beta parameters, the mean
// loss and the quantile table are a function of the record alone, built once
// (NEXT-2: one table per record, not one per (layer, record)).
struct RecordStore {
    int device = 0;
    uint64_t n = 0;                    // input records
    BetaRec *d_recs = nullptr;         // [n]
    float *d_mu = nullptr;             // [n]
    float2 *d_nodes = nullptr;         // kTabPad + [n][kTabNodes] quantile-table nodes (internal.cuh)
    uint32_t n_exact = 0;              // records whose table failed its midpoint check
    std::vector<uint32_t> pos;         // store position of each input record (the store follows the first
                                       // kernel group's event-major device order, so for a portfolio of one
                                       // group without shared XELTs a pair's table is its device record's)
    ~RecordStore() {
        cudaSetDevice(device);
        cudaFree(d_recs); cudaFree(d_mu); cudaFree(d_nodes);
    }
    uint64_t bytes() const { return n * (sizeof(BetaRec) + sizeof(float) + kTabNodes * sizeof(float2)); }
};

struct ara_portfolio {
    ara_ctx *ctx = nullptr;
    int device = 0;                    // (destroy uses this, not ctx: the context may be gone first)
    PortfolioDev dev{};
    uint32_t *d_bitmap = nullptr, *d_rec_orig = nullptr;
    uint2 *d_cidx = nullptr;
    uint32_t *d_cidx4 = nullptr;       // [C] packed index entries (compaction), if every first < 2^24
    SplitRec *d_srecs = nullptr;
    uint2 *d_mm = nullptr;             // (mean loss bits, meta) per device record (primary uncertainty)
    std::shared_ptr<RecordStore> store;   // per input record (shared by the groups)
    SlotInfo *d_slots = nullptr;
    LayerInfo *d_layers = nullptr;
    float *d_occ = nullptr;            // [catalog][occ_lp] occurrence losses without draws (fast path)
    uint32_t *d_occ_bitmap = nullptr;  // [bitmap words] nonzero occurrence losses (the fast path's filter)
    float *d_rec_z = nullptr;          // ARA_RNG_SUPPLIED: z_(E) per device record (ara_portfolio_set_z)
    std::vector<uint32_t> rec_src;     // input record of each device record
    uint32_t max_prog = 0;             // largest program id of the layers
    uint64_t n_input_records = 0;
    double *d_slot_terms = nullptr;    // [n_slots][4] XELT terms in fp64 (retention, limit, share, on)
    // a portfolio larger than one kernel group (> kSplitMaxLayers layers or
    // > ARA_MAX_SLOTS slots) is a list of groups of consecutive layers, each a
    // complete portfolio of its own, run one after the other over the YET
    std::vector<ara_portfolio *> groups;
    std::vector<uint32_t> group_layer0;   // first layer of each group
    uint32_t n_layers_total = 0;
};

struct ara_yet {
    ara_ctx *ctx = nullptr;
    int device = 0;                    // (destroy uses this, not ctx: the context may be gone first)
    YetDev dev{};
    uint32_t *d_events = nullptr;
    uint64_t *d_offsets = nullptr;
    uint32_t *d_redo = nullptr;        // trials to re-run with the fp64 kernel
    uint32_t *d_ovf = nullptr;         // trials whose pairs overflowed their batch region
    uint32_t *d_ovf_n = nullptr;       // ... and their exact pair counts
    uint32_t *d_max = nullptr;         // largest event id (device word)
    uint32_t *d_packed = nullptr;      // staging of packed uploads (+2 zero words)
    float *d_zprog = nullptr;          // ARA_RNG_SUPPLIED: z_(Prog,E) [program][occurrence] (ara_yet_set_z)
    uint32_t zprog_programs = 0;
    uint64_t packed_capacity = 0;
    uint64_t avg_len_x1000 = 0;        // mean events per trial x 1000
    uint64_t max_len = 0;              // longest trial
};

extern "C" {

const char *ara_last_error(void) { return g_err.c_str(); }

int ara_version(void) { return 100; }

int ara_ctx_create(int device, void *cuda_stream, ara_ctx **out) {
    if (!out) return fail(ARA_EINVAL, "out is NULL");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(ARA_ECUDA, "no CUDA device available (%s); libara has no CPU path",
                    cudaGetErrorString(e));
    if (device < 0 || device >= n) return fail(ARA_EINVAL, "device %d out of range [0,%d)", device, n);
    CU(enter_device(device));
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(ARA_ECUDA, "device %d is sm_%d%d; libara is built for sm_100a", device,
                    prop.major, prop.minor);
    ara_ctx *c = new ara_ctx();
    c->device = device;
    c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    c->num_sms = prop.multiProcessorCount;
    if (cudaMalloc(&c->d_status, sizeof(RunStatus)) != cudaSuccess ||
        cudaMallocHost(&c->h_status, sizeof(RunStatus)) != cudaSuccess ||
        cudaMallocHost(&c->h_out, kOutDoubles * sizeof(double)) != cudaSuccess ||
        dalloc(&c->ms.buf, kSortCap) != cudaSuccess || dalloc(&c->ms.hist, 4 * 256) != cudaSuccess ||
        dalloc(&c->ms.state, 1) != cudaSuccess || dalloc(&c->ms.d_rps, 64) != cudaSuccess ||
        dalloc(&c->ms.d_out, kOutDoubles) != cudaSuccess ||
        dalloc(&c->ms.mhist, kMultiHistWords) != cudaSuccess || dalloc(&c->ms.macc, 8) != cudaSuccess ||
        dalloc(&c->ms.states, kMaxRanks) != cudaSuccess ||
        dalloc(&c->ms.part_sum, kRedBlocks) != cudaSuccess ||
        dalloc(&c->ms.part_cnt, kRedBlocks) != cudaSuccess || cudaEventCreate(&c->ev[0]) != cudaSuccess ||
        cudaEventCreate(&c->ev[1]) != cudaSuccess || cudaEventCreate(&c->ev[2]) != cudaSuccess ||
        cudaEventCreate(&c->ev[3]) != cudaSuccess || dalloc(&c->d_sched, 2 * kMaxBatches + 4) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking) != cudaSuccess) {
        ara_ctx_destroy(c);
        return fail(ARA_ENOMEM, "device allocation failed in ara_ctx_create");
    }
    for (cudaEvent_t &e : c->tev)
        if (cudaEventCreate(&e) != cudaSuccess) {
            ara_ctx_destroy(c);
            return fail(ARA_ECUDA, "event creation failed in ara_ctx_create");
        }
    // the joint select's histograms and tail sums start zeroed; each launch
    // leaves them zeroed for the next (select_multi_kernel)
    if (cudaMemset(c->ms.mhist, 0, kMultiHistWords * sizeof(unsigned int)) != cudaSuccess ||
        cudaMemset(c->ms.macc, 0, 8 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess) {
        ara_ctx_destroy(c);
        return fail(ARA_ECUDA, "scratch initialisation failed in ara_ctx_create");
    }
    *out = c;
    return ARA_OK;
}

void ara_ctx_destroy(ara_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaFree(c->d_status);
    cudaFreeHost(c->h_status);
    cudaFreeHost(c->h_out);
    cudaFree(c->d_ep);
    cudaFree(c->ms.vals);
    cudaFree(c->ms.buf);
    cudaFree(c->ms.hist);
    cudaFree(c->ms.mhist);
    cudaFree(c->ms.macc);
    cudaFree(c->ms.state);
    cudaFree(c->ms.d_rps);
    cudaFree(c->ms.d_out);
    cudaFree(c->ms.states);
    cudaFree(c->ms.part_sum);
    cudaFree(c->ms.part_cnt);
    cudaFree(c->d_slots);
    cudaFree(c->d_pool);
    cudaFree(c->d_pool_off);
    cudaFree(c->d_counts);
    cudaFree(c->d_sched);
    for (cudaEvent_t e : c->ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : c->tev)
        if (e) cudaEventDestroy(e);
    if (c->cstream) cudaStreamDestroy(c->cstream);
    delete c;
}

int ara_ctx_synchronize(ara_ctx *c) {
    if (!c) return fail(ARA_EINVAL, "ctx is NULL");
    CU(enter_device(c->device));
    CU(cudaStreamSynchronize(c->stream));
    CU(fold_latched(c));
    CU(cudaStreamSynchronize(c->stream));
    const unsigned int bad = c->latched_bad, nc = c->latched_nonconv, sh = c->latched_short;
    c->latched_bad = c->latched_nonconv = c->latched_short = 0;
    if (bad) return fail(ARA_ERANGE, "an ARA_ASYNC run met event ids >= catalog_size (its YLT is not written)");
    if (sh)
        return fail(ARA_ENOMEM, "%u overflowing trials of ARA_ASYNC runs did not fit the overflow pool (their YLT "
                                "entries are not written): rerun without ARA_ASYNC", sh);
    if (nc) return fail(ARA_ECONVERGE, "beta quantile did not converge for %u samples (ARA_ASYNC runs)", nc);
    return ARA_OK;
}

int ara_validate_portfolio(uint32_t C, uint32_t n_elts, const uint64_t *eoff, const ara_record *rec,
                           const ara_elt_terms *et, uint32_t n_layers, const uint32_t *lprog,
                           const uint64_t *loff, const uint32_t *lelts, const ara_layer_terms *lt) {
    if (C == 0) return fail(ARA_EINVAL, "catalog_size must be >= 1");
    if (!eoff) return fail(ARA_EINVAL, "elt_rec_offsets is NULL");
    if (eoff[0] != 0) return fail(ARA_EINVAL, "elt_rec_offsets[0] must be 0");
    for (uint32_t j = 0; j < n_elts; ++j)
        if (eoff[j + 1] < eoff[j]) return fail(ARA_EINVAL, "elt_rec_offsets not monotone at XELT %u", j);
    const uint64_t R = eoff[n_elts];
    if (R && !rec) return fail(ARA_EINVAL, "records is NULL");
    if (R >= (1ull << 32)) return fail(ARA_EINVAL, "too many records (%llu)", (unsigned long long)R);
    std::vector<uint32_t> seen(C, 0xffffffffu);
    for (uint32_t j = 0; j < n_elts; ++j) {
        for (uint64_t r = eoff[j]; r < eoff[j + 1]; ++r) {
            const ara_record &q = rec[r];
            if (q.event_id >= C)
                return fail(ARA_ERANGE, "XELT %u record %llu: event %u >= catalog_size %u", j,
                            (unsigned long long)(r - eoff[j]), q.event_id, C);
            if (seen[q.event_id] == j)
                return fail(ARA_EDUP, "XELT %u: duplicate event %u (record %llu)", j, q.event_id,
                            (unsigned long long)(r - eoff[j]));
            seen[q.event_id] = j;
            const bool fin = std::isfinite(q.mean_loss) && std::isfinite(q.sigma_i) &&
                             std::isfinite(q.sigma_c) && std::isfinite(q.max_loss);
            if (!fin || q.max_loss <= 0.0f || q.mean_loss < 0.0f || q.mean_loss > q.max_loss ||
                q.sigma_i < 0.0f || q.sigma_c < 0.0f)
                return fail(ARA_EINVAL,
                            "XELT %u record %llu (event %u): need finite 0 <= mean <= max, max > 0, "
                            "sigmas >= 0 (mean=%g sI=%g sC=%g max=%g)",
                            j, (unsigned long long)(r - eoff[j]), q.event_id, q.mean_loss, q.sigma_i,
                            q.sigma_c, q.max_loss);
        }
        if (et) {
            const ara_elt_terms &t = et[j];
            if (!(t.retention >= 0.0 && std::isfinite(t.retention)) || !(t.limit > 0.0) ||
                std::isnan(t.limit) || !(t.share > 0.0 && t.share <= 1.0))
                return fail(ARA_EINVAL, "XELT %u terms: need retention >= 0, limit > 0, 0 < share <= 1", j);
        }
    }
    if (n_layers == 0) return fail(ARA_EINVAL, "portfolio has no layers");
    if (n_layers > ARA_MAX_PORTFOLIO_LAYERS)
        return fail(ARA_EINVAL, "n_layers %u > %d", n_layers, ARA_MAX_PORTFOLIO_LAYERS);
    if (!lprog || !loff || !lt) return fail(ARA_EINVAL, "layer arrays are NULL");
    if (n_elts > ARA_MAX_XELTS) return fail(ARA_EINVAL, "n_elts %u > %u", n_elts, ARA_MAX_XELTS);
    for (uint32_t l = 0; l < n_layers; ++l)
        if (lprog[l] >= ARA_MAX_PROGRAMS)
            return fail(ARA_EINVAL, "layer %u: program %u >= %u", l, lprog[l], ARA_MAX_PROGRAMS);
    if (loff[0] != 0) return fail(ARA_EINVAL, "layer_elt_offsets[0] must be 0");
    const uint64_t nslots = loff[n_layers];
    if (nslots > ARA_MAX_PORTFOLIO_SLOTS)
        return fail(ARA_EINVAL, "sum of XELTs over layers %llu > %d", (unsigned long long)nslots,
                    ARA_MAX_PORTFOLIO_SLOTS);
    if (nslots && !lelts) return fail(ARA_EINVAL, "layer_elts is NULL");
    for (uint32_t l = 0; l < n_layers; ++l) {
        if (loff[l + 1] <= loff[l]) return fail(ARA_EINVAL, "layer %u covers no XELT", l);
        if (loff[l + 1] - loff[l] > ARA_MAX_SLOTS)
            return fail(ARA_EINVAL, "layer %u covers %llu XELTs > %d", l,
                        (unsigned long long)(loff[l + 1] - loff[l]), ARA_MAX_SLOTS);
        for (uint64_t x = loff[l]; x < loff[l + 1]; ++x) {
            if (lelts[x] >= n_elts)
                return fail(ARA_ERANGE, "layer %u: XELT id %u >= n_elts %u", l, lelts[x], n_elts);
            for (uint64_t y = loff[l]; y < x; ++y)
                if (lelts[y] == lelts[x]) return fail(ARA_EDUP, "layer %u: duplicate XELT %u", l, lelts[x]);
        }
        const ara_layer_terms &t = lt[l];
        if (!(t.occ_retention >= 0.0 && std::isfinite(t.occ_retention)) ||
            !(t.agg_retention >= 0.0 && std::isfinite(t.agg_retention)) || !(t.occ_limit > 0.0) ||
            !(t.agg_limit > 0.0) || std::isnan(t.occ_limit) || std::isnan(t.agg_limit))
            return fail(ARA_EINVAL, "layer %u terms: need retentions >= 0 finite, limits > 0", l);
    }
    return ARA_OK;
}

static int create_group(ara_ctx *c, uint32_t C, uint32_t n_elts, const uint64_t *eoff,
                        const ara_record *rec, const ara_elt_terms *et, uint32_t n_layers,
                        const uint32_t *lprog, const uint64_t *loff, const uint32_t *lelts,
                        const ara_layer_terms *lt, std::shared_ptr<RecordStore> &store,
                        ara_portfolio **out);

// the record store: upload the input records, derive their beta parameters and
// quantile tables on the device (one thread per record, fp64)
static int create_store(ara_ctx *c, const ara_record *rec, uint64_t R, const std::vector<uint32_t> &first_order,
                        std::shared_ptr<RecordStore> &out) {
    auto st = std::make_shared<RecordStore>();
    st->device = c->device;
    st->n = R;
    // order: the input records in the first group's device-record order (first
    // occurrence), then every other record
    std::vector<uint32_t> order;
    order.reserve(R);
    st->pos.assign(R, 0xffffffffu);
    for (uint32_t src : first_order)
        if (st->pos[src] == 0xffffffffu) { st->pos[src] = (uint32_t)order.size(); order.push_back(src); }
    for (uint64_t src = 0; src < R; ++src)
        if (st->pos[src] == 0xffffffffu) { st->pos[src] = (uint32_t)order.size(); order.push_back((uint32_t)src); }
    ara_record *d_raw = nullptr;
    uint32_t *d_order = nullptr;
    cudaStream_t s = c->stream;
    if (dalloc(&st->d_recs, R) || dalloc(&st->d_mu, R) || dalloc(&st->d_nodes, R * kTabNodes + kTabPad) ||
        dalloc(&d_raw, R) || dalloc(&d_order, R)) {
        cudaGetLastError();
        cudaFree(d_raw); cudaFree(d_order);
        return fail(ARA_ENOMEM, "device allocation of %llu records failed in ara_create_portfolio",
                    (unsigned long long)R);
    }
    cudaError_t e = R ? cudaMemcpyAsync(d_raw, rec, R * sizeof(ara_record), cudaMemcpyHostToDevice, s) : cudaSuccess;
    // table-less records keep zero nodes (the split sampler reads them, then redoes the trial)
    if (e == cudaSuccess) e = cudaMemsetAsync(st->d_nodes, 0, (R * kTabNodes + kTabPad) * sizeof(float2), s);
    if (e == cudaSuccess && R) e = cudaMemcpyAsync(d_order, order.data(), R * sizeof(uint32_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(c->d_status, 0, sizeof(RunStatus), s);
    if (e == cudaSuccess) {
        launch_prep_records(d_raw, d_order, R, st->d_recs, st->d_mu, st->d_nodes + kTabPad,
                            &c->d_status->nonconverged, s);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d_raw); cudaFree(d_order);
    if (e != cudaSuccess) return fail(ARA_ECUDA, "record preparation: %s", cudaGetErrorString(e));
    st->n_exact = c->h_status->nonconverged;
    out = st;
    return ARA_OK;
}

int ara_create_portfolio(ara_ctx *c, uint32_t C, uint32_t n_elts, const uint64_t *eoff,
                         const ara_record *rec, const ara_elt_terms *et, uint32_t n_layers,
                         const uint32_t *lprog, const uint64_t *loff, const uint32_t *lelts,
                         const ara_layer_terms *lt, ara_portfolio **out) {
    NvtxRange nvtx("ara_create_portfolio");
    if (!c || !out) return fail(ARA_EINVAL, "ctx/out is NULL");
    *out = nullptr;
    int st = ara_validate_portfolio(C, n_elts, eoff, rec, et, n_layers, lprog, loff, lelts, lt);
    if (st != ARA_OK) return st;
    CU(enter_device(c->device));
    // Kernel groups of consecutive layers: <= kSplitMaxLayers layers, <=
    // ARA_MAX_SLOTS slots, and -- so that each pass's gathered tables stay
    // L2-resident -- at most ARA_GROUP_BYTES (default 128 MiB)
    // of per-record sampler data (SplitRec + hot table rows, 160 B per
    // (layer, record)) plus the catalogue index (8 B per event); a single
    // layer always forms a group.  Each group re-streams the YET.
    const uint64_t budget = env_u64("ARA_GROUP_BYTES", 128ull << 20);
    auto layer_records = [&](uint32_t l) {
        uint64_t r = 0;
        for (uint64_t x = loff[l]; x < loff[l + 1]; ++x) r += eoff[lelts[x] + 1] - eoff[lelts[x]];
        return r;
    };
    auto fits = [&](uint32_t l0, uint32_t l1) {       // layers [l0, l1] in one group?
        if (l1 - l0 + 1 > (uint32_t)kSplitMaxLayers || loff[l1 + 1] - loff[l0] > ARA_MAX_SLOTS) return false;
        uint64_t recs = 0;
        for (uint32_t l = l0; l <= l1; ++l) recs += layer_records(l);
        return l1 == l0 || recs * 160 + (uint64_t)C * 8 <= budget;
    };
    CU(enter_device(c->device));
    std::shared_ptr<RecordStore> store;              // built by the first group (its device order)
    if (fits(0, n_layers - 1))
        return create_group(c, C, n_elts, eoff, rec, et, n_layers, lprog, loff, lelts, lt, store, out);
    ara_portfolio *p = new ara_portfolio();
    p->ctx = c;
    p->device = c->device;
    p->n_layers_total = n_layers;
    for (uint32_t l0 = 0; l0 < n_layers;) {
        uint32_t l1 = l0 + 1;
        while (l1 < n_layers && fits(l0, l1)) ++l1;
        std::vector<uint64_t> sub(l1 - l0 + 1);
        for (uint32_t l = l0; l <= l1; ++l) sub[l - l0] = loff[l] - loff[l0];
        ara_portfolio *g = nullptr;
        st = create_group(c, C, n_elts, eoff, rec, et, l1 - l0, lprog + l0, sub.data(), lelts + loff[l0], lt + l0,
                          store, &g);
        if (st != ARA_OK) {
            ara_portfolio_destroy(p);
            return st;
        }
        p->groups.push_back(g);
        p->group_layer0.push_back(l0);
        p->store = store;
        l0 = l1;
    }
    *out = p;
    return ARA_OK;
}

static int create_group(ara_ctx *c, uint32_t C, uint32_t n_elts, const uint64_t *eoff,
                        const ara_record *rec, const ara_elt_terms *et, uint32_t n_layers,
                        const uint32_t *lprog, const uint64_t *loff, const uint32_t *lelts,
                        const ara_layer_terms *lt, std::shared_ptr<RecordStore> &store,
                        ara_portfolio **out) {
    CU(enter_device(c->device));

    // slots: (layer, XELT) pairs, layer-major
    const uint32_t S = (uint32_t)loff[n_layers];
    std::vector<SlotInfo> slots(S);
    for (uint32_t l = 0; l < n_layers; ++l)
        for (uint64_t x = loff[l]; x < loff[l + 1]; ++x) {
            SlotInfo &s = slots[x];
            const uint32_t j = lelts[x];
            s.elt = j; s.prog = lprog[l]; s.layer = l;
            s.has_terms = et ? 1u : 0u;
            s.ret = et ? (float)et[j].retention : 0.0f;
            s.lim = et ? (float)et[j].limit : INFINITY;
            s.share = et ? (float)et[j].share : 1.0f;
            s.pad = 0.0f;
        }
    std::vector<LayerInfo> layers(n_layers);
    for (uint32_t l = 0; l < n_layers; ++l)
        layers[l] = {lt[l].occ_retention, lt[l].occ_limit, lt[l].agg_retention, lt[l].agg_limit};
    std::vector<double> slot_terms(4 * (size_t)S, 0.0);    // the XELT terms as given (fp64)
    for (uint32_t x = 0; x < S; ++x)
        if (et) {
            const ara_elt_terms &q = et[slots[x].elt];
            slot_terms[4 * x] = q.retention; slot_terms[4 * x + 1] = q.limit;
            slot_terms[4 * x + 2] = q.share; slot_terms[4 * x + 3] = 1.0;
        }
    // no record of the portfolio carries a sigma: no draw is ever taken (G10)
    bool all_sigma_zero = true;
    for (uint32_t x = 0; x < S && all_sigma_zero; ++x)
        for (uint64_t r = eoff[slots[x].elt]; r < eoff[slots[x].elt + 1]; ++r)
            if (rec[r].sigma_i != 0.0f || rec[r].sigma_c != 0.0f) { all_sigma_zero = false; break; }
    const uint32_t occ_lp = n_layers <= 1 ? 1 : n_layers <= 2 ? 2 : n_layers <= 4 ? 4 : 8;

    // event-major direct-access index: per event the slots with a record
    const uint32_t MW = (S + 31) / 32;
    const uint32_t stride = MW + 1;                 // host-side planning index: first record, slot mask words
    std::vector<uint32_t> index((size_t)C * stride, 0u);
    for (uint32_t s = 0; s < S; ++s) {
        const uint32_t j = slots[s].elt;
        for (uint64_t r = eoff[j]; r < eoff[j + 1]; ++r)
            index[(size_t)rec[r].event_id * stride + 1 + (s >> 5)] |= 1u << (s & 31);
    }
    uint64_t total = 0;
    for (uint32_t e = 0; e < C; ++e) {
        uint32_t *ix = &index[(size_t)e * stride];
        ix[0] = (uint32_t)total;
        for (uint32_t w = 0; w < MW; ++w) total += (uint32_t)__builtin_popcount(ix[1 + w]);
    }
    if (total >= (1ull << 32)) return fail(ARA_EINVAL, "too many (layer, record) pairs");
    std::vector<uint32_t> rec_src(total), rec_orig(total);
    std::vector<uint32_t> rec_meta(total);      // slot | run_end << 8 | layer << 16
    std::vector<uint2> cidx(C);                  // (first record, record count) per event
    for (uint32_t e = 0; e < C; ++e) {
        const uint32_t *ix = &index[(size_t)e * stride];
        uint32_t n = 0;
        for (uint32_t w = 0; w < MW; ++w) n += (uint32_t)__builtin_popcount(ix[1 + w]);
        cidx[e] = make_uint2(ix[0], n);
    }
    for (uint32_t s = 0; s < S; ++s) {
        const uint32_t j = slots[s].elt;
        for (uint64_t r = eoff[j]; r < eoff[j + 1]; ++r) {
            const uint32_t *ix = &index[(size_t)rec[r].event_id * stride];
            uint32_t rank = 0;
            for (uint32_t w = 0; w < (s >> 5); ++w) rank += (uint32_t)__builtin_popcount(ix[1 + w]);
            rank += (uint32_t)__builtin_popcount(ix[1 + (s >> 5)] & ((1u << (s & 31)) - 1u));
            rec_src[ix[0] + rank] = (uint32_t)r;
            rec_orig[ix[0] + rank] = (uint32_t)(r - eoff[j]);
            rec_meta[ix[0] + rank] = s | (slots[s].layer << 16);
        }
    }
    for (uint32_t e = 0; e < C; ++e)
        for (uint32_t r = cidx[e].x; r < cidx[e].x + cidx[e].y; ++r) {
            const bool last = r + 1 == cidx[e].x + cidx[e].y ||
                              slots[rec_meta[r + 1] & 0xffu].layer != slots[rec_meta[r] & 0xffu].layer;
            if (last) rec_meta[r] |= 0x100u;
        }
    // presence bitmap (any slot present), at most 2^20 bits (128 KiB of smem)
    uint32_t shift = 0;
    while (((uint64_t)C + (1ull << shift) - 1) >> shift > (1ull << 20)) ++shift;
    const uint64_t bits = ((uint64_t)C + (1ull << shift) - 1) >> shift;
    const uint32_t words = (uint32_t)((bits + 31) / 32);
    std::vector<uint32_t> bitmap(words, 0u);
    for (uint32_t e = 0; e < C; ++e) {
        bool any = false;
        for (uint32_t w = 0; w < MW; ++w) any |= index[(size_t)e * stride + 1 + w] != 0;
        if (any) bitmap[(e >> shift) >> 5] |= 1u << ((e >> shift) & 31);
    }

    if (!store) {
        const int st = create_store(c, rec, eoff[n_elts], rec_src, store);
        if (st != ARA_OK) return st;
    }
    std::vector<uint32_t> tab(total);           // store position (table) of each device record
    for (uint64_t r = 0; r < total; ++r) tab[r] = store->pos[rec_src[r]];
    ara_portfolio *p = new ara_portfolio();
    p->ctx = c;
    p->device = c->device;
    p->store = store;
    cudaStream_t s = c->stream;
    uint32_t *d_rec_meta = nullptr, *d_rec_src = nullptr;   // build-time arrays
    auto cleanup = [&](int code) {
        cudaFree(d_rec_meta); cudaFree(d_rec_src);
        ara_portfolio_destroy(p);
        return code;
    };
    if (dalloc(&p->d_bitmap, words) ||
        dalloc(&p->d_cidx, (size_t)C) || (total < (1ull << 24) && dalloc(&p->d_cidx4, (size_t)C)) ||
        dalloc(&d_rec_meta, (size_t)total) || dalloc(&p->d_srecs, (size_t)total) ||
        dalloc(&p->d_mm, (size_t)total) || dalloc(&p->d_rec_orig, total) || dalloc(&d_rec_src, total) ||
        dalloc(&p->d_slots, S) || dalloc(&p->d_layers, n_layers) ||
        dalloc(&p->d_occ, (size_t)C * occ_lp) || dalloc(&p->d_occ_bitmap, words) ||
        dalloc(&p->d_slot_terms, slot_terms.size())) {
        cudaGetLastError();
        return cleanup(fail(ARA_ENOMEM, "device allocation failed in ara_create_portfolio"));
    }
    cudaError_t e = cudaSuccess;
#define UP(dst, src, n) if (e == cudaSuccess && (n)) e = cudaMemcpyAsync(dst, src, (n) * sizeof(*(src)), cudaMemcpyHostToDevice, s)
    UP(p->d_bitmap, bitmap.data(), (size_t)words);
    UP(p->d_rec_orig, rec_orig.data(), (size_t)total);
    UP(p->d_cidx, cidx.data(), (size_t)C);
    std::vector<uint32_t> cidx4;
    if (p->d_cidx4) {                                   // first | count << 24 (count <= ARA_MAX_SLOTS < 256)
        cidx4.resize(C);
        for (uint32_t ev = 0; ev < C; ++ev) cidx4[ev] = cidx[ev].x | (cidx[ev].y << 24);
        UP(p->d_cidx4, cidx4.data(), (size_t)C);
    }
    UP(d_rec_meta, rec_meta.data(), (size_t)total);
    UP(p->d_slots, slots.data(), (size_t)S);
    UP(p->d_layers, layers.data(), (size_t)n_layers);
    UP(d_rec_src, tab.data(), (size_t)total);
    UP(p->d_slot_terms, slot_terms.data(), slot_terms.size());
#undef UP
    if (e != cudaSuccess) return cleanup(fail(ARA_ECUDA, "upload: %s", cudaGetErrorString(e)));
    if (e == cudaSuccess) {
        launch_split_recs(store->d_recs, d_rec_src, d_rec_meta, p->d_slots, store->d_mu, total, p->d_srecs,
                          p->d_mm, s);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) {       // lines 6-11 per (event, layer) at the mean losses (fast path)
        launch_occ_table(p->d_cidx, p->d_mm, p->d_slot_terms, p->d_layers, n_layers, occ_lp, C,
                         p->d_occ, s);
        launch_occ_bitmap(p->d_occ, occ_lp, C, shift, words, p->d_occ_bitmap, s);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);     // host vectors die at return
    cudaFree(d_rec_meta); cudaFree(d_rec_src);          // (build-time only)
    d_rec_meta = nullptr; d_rec_src = nullptr;
    if (e != cudaSuccess) return cleanup(fail(ARA_ECUDA, "portfolio layout: %s", cudaGetErrorString(e)));

    PortfolioDev &d = p->dev;
    d.catalog = C; d.n_slots = S; d.n_layers = n_layers;
    d.bitmap_shift = shift; d.bitmap_words = words; d.n_dev_records = total;
    {   // sentinel event for the compaction's partial chunks: a presence bit that is 0
        d.sentinel_ok = 0; d.sentinel_event = 0;
        const uint64_t cand = ((uint64_t)words * 32u) << shift;     // the appended zero word
        if (cand <= 0xffffffffull) { d.sentinel_event = (uint32_t)cand; d.sentinel_ok = 1; }
        else
            for (uint64_t b = 0; b < bits && !d.sentinel_ok; ++b)
                if (!((bitmap[b >> 5] >> (b & 31)) & 1u) && (b << shift) <= 0xffffffffull) {
                    d.sentinel_event = (uint32_t)(b << shift); d.sentinel_ok = 1;
                }
    }
    d.n_exact_records = store->n_exact;
    d.n_tables = store->n;
    d.bitmap = p->d_bitmap; d.recs = store->d_recs; d.rec_mu = store->d_mu;
    d.tables = TablePtr{store->d_nodes + kTabPad};
    d.rec_orig = p->d_rec_orig; d.slots = p->d_slots; d.layers = p->d_layers;
    d.cidx = p->d_cidx; d.cidx4 = p->d_cidx4; d.srecs = p->d_srecs; d.mu_meta = p->d_mm;
    d.any_terms = et ? 1u : 0u;
    p->rec_src = std::move(rec_src);
    p->n_input_records = eoff[n_elts];
    for (uint32_t l = 0; l < n_layers; ++l) p->max_prog = std::max(p->max_prog, lprog[l]);
    d.all_sigma_zero = all_sigma_zero ? 1u : 0u;
    d.occ_lp = occ_lp;
    d.occ = p->d_occ;
    d.occ_bitmap = p->d_occ_bitmap;
    *out = p;
    return ARA_OK;
}

static uint64_t group_bytes(const ara_portfolio *g) {          // per-group arrays (not the record store)
    const PortfolioDev &d = g->dev;
    return (uint64_t)d.catalog * (sizeof(uint2) + (d.cidx4 ? 4 : 0) + d.occ_lp * sizeof(float)) +
           (uint64_t)d.bitmap_words * 8 +
           d.n_dev_records * (sizeof(SplitRec) + sizeof(uint2) + sizeof(uint32_t)) +
           d.n_slots * (sizeof(SlotInfo) + 4 * sizeof(double)) + d.n_layers * sizeof(LayerInfo);
}

int ara_portfolio_info(const ara_portfolio *p, uint64_t *n_dev, uint64_t *n_tl, uint64_t *bytes) {
    if (!p) return fail(ARA_EINVAL, "portfolio is NULL");
    uint64_t a = 0, c = 0;
    if (!p->groups.empty()) {                          // sums over the groups
        for (const ara_portfolio *g : p->groups) {
            a += g->dev.n_dev_records;
            c += group_bytes(g);
        }
    } else {
        a = p->dev.n_dev_records;
        c = group_bytes(p);
    }
    if (n_dev) *n_dev = a;
    if (n_tl) *n_tl = p->store ? p->store->n_exact : 0;
    if (bytes) *bytes = c + (p->store ? p->store->bytes() : 0);
    return ARA_OK;
}

void ara_portfolio_destroy(ara_portfolio *p) {
    if (!p) return;
    for (ara_portfolio *g : p->groups) ara_portfolio_destroy(g);
    cudaSetDevice(p->device);
    cudaFree(p->d_bitmap); cudaFree(p->d_rec_orig);
    cudaFree(p->d_cidx); cudaFree(p->d_cidx4); cudaFree(p->d_srecs); cudaFree(p->d_mm);
    cudaFree(p->d_slots); cudaFree(p->d_layers);
    cudaFree(p->d_occ); cudaFree(p->d_occ_bitmap); cudaFree(p->d_slot_terms); cudaFree(p->d_rec_z);
    delete p;
    cudaGetLastError();                    // (a destroy cannot report: leave no stale error behind)
}

int ara_load_yet(ara_ctx *c, uint64_t n_trials, uint64_t first_trial, const uint64_t *toff,
                 uint32_t fixed_len, const uint32_t *events, const float *ts, ara_yet **out) {
    if (!c || !out) return fail(ARA_EINVAL, "ctx/out is NULL");
    *out = nullptr;
    if (first_trial + n_trials > (1ull << 32))
        return fail(ARA_EINVAL, "first_trial + n_trials must be <= 2^32 (Philox counter word)");
    uint64_t total;
    if (toff) {
        if (toff[0] != 0) return fail(ARA_EINVAL, "trial_offsets[0] must be 0");
        for (uint64_t t = 0; t < n_trials; ++t) {
            if (toff[t + 1] < toff[t])
                return fail(ARA_EINVAL, "trial_offsets not monotone at trial %llu", (unsigned long long)t);
            if (toff[t + 1] - toff[t] > ARA_MAX_EVENTS_PER_TRIAL)
                return fail(ARA_EINVAL, "trial %llu has more than 2^24 events", (unsigned long long)t);
        }
        total = toff[n_trials];
    } else {
        if (fixed_len > ARA_MAX_EVENTS_PER_TRIAL) return fail(ARA_EINVAL, "fixed_len > 2^24");
        total = n_trials * (uint64_t)fixed_len;
    }
    // (events may be NULL: the ids start as 0, to be filled by ara_yet_refill[_packed])
    if (ts) {
        for (uint64_t t = 0; t < n_trials; ++t) {
            const uint64_t b = toff ? toff[t] : t * fixed_len, e = toff ? toff[t + 1] : b + fixed_len;
            for (uint64_t x = b; x < e; ++x) {
                if (!std::isfinite(ts[x])) return fail(ARA_EINVAL, "trial %llu: non-finite timestamp", (unsigned long long)t);
                if (x > b && ts[x] < ts[x - 1])
                    return fail(ARA_EINVAL, "trial %llu: timestamps not sorted (P:58)", (unsigned long long)t);
            }
        }
    }
    CU(enter_device(c->device));
    ara_yet *y = new ara_yet();
    y->ctx = c;
    y->device = c->device;
    // +4 words: the compaction kernel's bulk copies round each piece up to 16 B
    if (dalloc(&y->d_events, total + 4) != cudaSuccess || dalloc(&y->d_redo, n_trials) != cudaSuccess ||
        dalloc(&y->d_ovf, n_trials) != cudaSuccess || dalloc(&y->d_ovf_n, n_trials) != cudaSuccess ||
        dalloc(&y->d_max, 1) != cudaSuccess ||
        (toff && dalloc(&y->d_offsets, n_trials + 1) != cudaSuccess)) {
        cudaGetLastError();
        ara_yet_destroy(y);
        return fail(ARA_ENOMEM, "device allocation of %llu event ids failed", (unsigned long long)total);
    }
    cudaError_t e = cudaSuccess;
    if (total && events)
        e = cudaMemcpyAsync(y->d_events, events, total * sizeof(uint32_t),
                            is_device_ptr(events) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                            c->stream);
    else if (total)
        e = cudaMemsetAsync(y->d_events, 0, total * sizeof(uint32_t), c->stream);
    if (e == cudaSuccess && toff)
        e = cudaMemcpyAsync(y->d_offsets, toff, (n_trials + 1) * sizeof(uint64_t),
                            cudaMemcpyHostToDevice, c->stream);
    if (e == cudaSuccess) e = launch_yet_max(y->d_events, total, y->d_max, c->stream, c->num_sms);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) {
        ara_yet_destroy(y);
        return fail(ARA_ECUDA, "YET upload: %s", cudaGetErrorString(e));
    }
    y->dev.n_trials = n_trials; y->dev.first_trial = first_trial;
    y->dev.fixed_len = toff ? 0u : fixed_len;
    y->dev.offsets = y->d_offsets; y->dev.events = y->d_events; y->dev.n_events = total;
    y->dev.max_event = y->d_max;
    y->avg_len_x1000 = n_trials ? (total * 1000) / n_trials : 0;
    y->max_len = fixed_len;
    if (toff)
        for (uint64_t q = 0; q < n_trials; ++q) y->max_len = std::max<uint64_t>(y->max_len, toff[q + 1] - toff[q]);
    *out = y;
    return ARA_OK;
}

int ara_yet_refill(ara_ctx *c, ara_yet *y, const uint32_t *events) {
    if (!c || !y) return fail(ARA_EINVAL, "ctx/yet is NULL");
    if (y->dev.n_events == 0) return ARA_OK;
    if (!events) return fail(ARA_EINVAL, "event_ids is NULL");
    CU(enter_device(c->device));
    CU(cudaMemcpyAsync(y->d_events, events, y->dev.n_events * sizeof(uint32_t),
                       is_device_ptr(events) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       c->stream));
    CU(launch_yet_max(y->d_events, y->dev.n_events, y->d_max, c->stream, c->num_sms));
    return ARA_OK;
}

int ara_yet_refill_packed(ara_ctx *c, ara_yet *y, uint32_t bits, const uint32_t *packed) {
    if (!c || !y) return fail(ARA_EINVAL, "ctx/yet is NULL");
    if (bits < 1 || bits > 32) return fail(ARA_EINVAL, "bits %u not in [1, 32]", bits);
    if (y->dev.n_events == 0) return ARA_OK;
    if (!packed) return fail(ARA_EINVAL, "packed is NULL");
    const uint64_t words = (y->dev.n_events * (uint64_t)bits + 31) / 32;
    CU(enter_device(c->device));
    const uint32_t *src = packed;
    if (!is_device_ptr(packed)) {                       // host words: staged on the device first
        if (y->packed_capacity < words) {              // (the staging grows once, then is reused)
            cudaFree(y->d_packed);
            y->d_packed = nullptr;
            y->packed_capacity = 0;
            CU(dalloc(&y->d_packed, words));
            y->packed_capacity = words;
        }
        CU(cudaMemcpyAsync(y->d_packed, packed, words * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
        src = y->d_packed;
    }                                                   // device words: unpacked where they are
    CU(launch_unpack_yet(src, y->dev.n_events, bits, y->d_events, c->stream, c->num_sms));
    CU(launch_yet_max(y->d_events, y->dev.n_events, y->d_max, c->stream, c->num_sms));
    return ARA_OK;
}

int ara_yet_set_z(ara_ctx *c, ara_yet *y, uint32_t n_programs, const float *z_prog) {
    if (!c || !y) return fail(ARA_EINVAL, "ctx/yet is NULL");
    if (n_programs == 0 || !z_prog) return fail(ARA_EINVAL, "need n_programs >= 1 and z_prog");
    const uint64_t n = (uint64_t)n_programs * y->dev.n_events;
    for (uint64_t x = 0; x < n; ++x)
        if (!(z_prog[x] > 0.0f && z_prog[x] < 1.0f))
            return fail(ARA_EINVAL, "z_(Prog,E) must lie in (0,1): program %llu occurrence %llu",
                        (unsigned long long)(x / std::max<uint64_t>(y->dev.n_events, 1)),
                        (unsigned long long)(x % std::max<uint64_t>(y->dev.n_events, 1)));
    CU(enter_device(c->device));
    cudaFree(y->d_zprog);
    y->d_zprog = nullptr;
    y->zprog_programs = 0;
    CU(dalloc(&y->d_zprog, n));
    CU(cudaMemcpyAsync(y->d_zprog, z_prog, n * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    y->zprog_programs = n_programs;
    return ARA_OK;
}

int ara_portfolio_set_z(ara_ctx *c, ara_portfolio *p, const float *z_event) {
    if (!c || !p) return fail(ARA_EINVAL, "ctx/portfolio is NULL");
    if (!z_event) return fail(ARA_EINVAL, "z_event is NULL");
    if (!p->groups.empty()) {
        for (ara_portfolio *g : p->groups) {
            const int st = ara_portfolio_set_z(c, g, z_event);
            if (st != ARA_OK) return st;
        }
        return ARA_OK;
    }
    for (uint64_t r = 0; r < p->n_input_records; ++r)
        if (!(z_event[r] > 0.0f && z_event[r] < 1.0f))
            return fail(ARA_EINVAL, "z_(E) must lie in (0,1): record %llu", (unsigned long long)r);
    std::vector<float> z(p->rec_src.size());           // per device record (layout only, no arithmetic)
    for (size_t r = 0; r < z.size(); ++r) z[r] = z_event[p->rec_src[r]];
    CU(enter_device(c->device));
    cudaFree(p->d_rec_z);
    p->d_rec_z = nullptr;
    CU(dalloc(&p->d_rec_z, z.size()));
    CU(cudaMemcpyAsync(p->d_rec_z, z.data(), z.size() * sizeof(float), cudaMemcpyHostToDevice, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return ARA_OK;
}

uint64_t ara_yet_num_trials(const ara_yet *y) { return y ? y->dev.n_trials : 0; }

void ara_yet_destroy(ara_yet *y) {
    if (!y) return;
    cudaSetDevice(y->device);
    cudaFree(y->d_events);
    cudaFree(y->d_offsets);
    cudaFree(y->d_redo);
    cudaFree(y->d_ovf);
    cudaFree(y->d_ovf_n);
    cudaFree(y->d_max);
    cudaFree(y->d_packed);
    cudaFree(y->d_zprog);
    delete y;
    cudaGetLastError();                    // (a destroy cannot report: leave no stale error behind)
}

// Layout of one split-path run: per-trial pair regions of 2x the expected
// pairs per trial (+128) for uniformly drawn event ids (the size only decides
// which trials take the overflow pass, never the arithmetic), 4-byte pairs
// when record << kbits | k fits, and the trial batches of the two-stream
// pipeline (ARA_BATCH_TRIALS; default: one batch while its slot fits 4 GiB;
// at most kMaxBatches).
struct SplitPlan {
    uint32_t cap, kbits, n_batches;
    uint64_t batch, slot_bytes;
};

static SplitPlan plan_split(const ara_portfolio *p, const ara_yet *y, uint32_t flags) {
    SplitPlan pl{};
    const uint64_t N = y->dev.n_trials;
    const double per_occ = (double)p->dev.n_dev_records / (double)p->dev.catalog;
    const double expect = per_occ * (double)y->avg_len_x1000 / 1000.0;
    uint32_t cap = (uint32_t)((2.0 * expect + 128.0 + 31.0) / 32.0) * 32u;
    if (cap > (1u << 20)) cap = 1u << 20;
    pl.cap = (uint32_t)env_u64("ARA_PAIR_CAP", cap);     // test aid: force the overflow pass
    if (!(flags & ARA_WIDE_PAIRS)) {
        uint32_t kb = 1;
        while (kb < 24 && (1ull << kb) < (uint64_t)y->max_len) ++kb;
        if ((uint64_t)p->dev.n_dev_records <= (1ull << (32 - kb))) pl.kbits = kb;
    }
    // one batch while its pair slot stays within 4 GiB (each batch launch
    // costs a kernel ramp and tail: measured 5.08 ms per cfg3 step in one
    // batch, 5.27 in four), else as many as needed
    const uint64_t per_trial = (uint64_t)pl.cap * (pl.kbits ? 4 : 8);
    uint64_t batch = env_u64("ARA_BATCH_TRIALS", std::max<uint64_t>(1, (4ull << 30) / std::max<uint64_t>(per_trial, 1)));
    batch = std::max<uint64_t>(batch, (N + kMaxBatches - 1) / kMaxBatches);
    batch = std::min<uint64_t>(std::max<uint64_t>(batch, 1), std::max<uint64_t>(N, 1));
    pl.batch = batch;
    pl.n_batches = (uint32_t)((N + batch - 1) / batch);
    pl.slot_bytes = batch * (uint64_t)pl.cap * (pl.kbits ? 4 : 8);
    return pl;
}

// ARA_ASYNC's pre-sized overflow pool: an eighth of the pair slot, at least
// 2^24 pairs (the synchronous path sizes the pool exactly instead)
static uint64_t default_pool_pairs(const SplitPlan &pl, uint64_t n_trials) {
    const uint64_t d = std::max<uint64_t>(1ull << 24, (uint64_t)pl.cap * std::min<uint64_t>(pl.batch, n_trials) / 8);
    return env_u64("ARA_ASYNC_POOL_PAIRS", d);       // (test aid: a small pool)
}

static int run_impl(ara_ctx *c, const ara_portfolio *p, const ara_yet *y, uint64_t seed, uint32_t flags,
                    float *ylt, float *occ_max, uint32_t *dbg_count, uint64_t *dbg_hash);

int ara_run(ara_ctx *c, const ara_portfolio *p, const ara_yet *y, uint64_t seed, uint32_t flags,
            float *ylt, uint32_t *dbg_count, uint64_t *dbg_hash) {
    return run_impl(c, p, y, seed, flags, ylt, nullptr, dbg_count, dbg_hash);
}

int ara_run_ep(ara_ctx *c, const ara_portfolio *p, const ara_yet *y, uint64_t seed, uint32_t flags,
               float *ylt, float *occ_max, uint32_t *dbg_count, uint64_t *dbg_hash) {
    if (!occ_max) return fail(ARA_EINVAL, "occ_max is NULL (use ara_run)");
    return run_impl(c, p, y, seed, flags, ylt, occ_max, dbg_count, dbg_hash);
}

static int run_group(ara_ctx *c, const ara_portfolio *p, const ara_yet *y, uint64_t seed, uint32_t flags,
                     float *ylt, float *occ_max, uint32_t *dbg_count, uint64_t *dbg_hash);

static int run_impl(ara_ctx *c, const ara_portfolio *p, const ara_yet *y, uint64_t seed, uint32_t flags,
                    float *ylt, float *occ_max, uint32_t *dbg_count, uint64_t *dbg_hash) {
    NvtxRange nvtx("ara_run");
    if (!c || !p || !y) return fail(ARA_EINVAL, "ctx/portfolio/yet is NULL");
    if (p->groups.empty()) return run_group(c, p, y, seed, flags, ylt, occ_max, dbg_count, dbg_hash);
    // one run per group of layers over the same YET (the draws do not depend on
    // the layer or its slot, so the YLT equals one run of the whole portfolio)
    const uint64_t N = y->dev.n_trials;
    double ms[3] = {0.0, 0.0, 0.0};
    uint32_t launches = 0, batches = 0;
    for (size_t g = 0; g < p->groups.size(); ++g) {
        const uint64_t off = (uint64_t)p->group_layer0[g] * N;
        const int st = run_group(c, p->groups[g], y, seed, flags, ylt ? ylt + off : nullptr,
                                 occ_max ? occ_max + off : nullptr, dbg_count ? dbg_count + off : nullptr,
                                 dbg_hash ? dbg_hash + off : nullptr);
        if (st != ARA_OK) return st;
        launches += c->last_launches;
        batches += c->last_batches;
        // a synchronous run sums the groups' kernel times; an ARA_ASYNC run
        // must not wait (nor may a run being captured into a CUDA graph): its
        // ara_last_run_timings are those of the last group
        if (flags & ARA_ASYNC) continue;
        CU(compute_timings(c));
        for (int k = 0; k < 3; ++k) ms[k] += c->last_ms[k];
    }
    if (!(flags & ARA_ASYNC))
        for (int k = 0; k < 3; ++k) c->last_ms[k] = ms[k];
    c->last_launches = launches;
    c->last_batches = batches;
    return ARA_OK;
}

static int run_group(ara_ctx *c, const ara_portfolio *p, const ara_yet *y, uint64_t seed, uint32_t flags,
                     float *ylt, float *occ_max, uint32_t *dbg_count, uint64_t *dbg_hash) {
    if (flags & ~(ARA_SU | ARA_DEBUG_LOOKUP | ARA_EXACT | ARA_WIDE_PAIRS | ARA_RNG_RECORD | ARA_RNG_OCCURRENCE |
                  ARA_RNG_SUPPLIED | ARA_ASYNC))
        return fail(ARA_EINVAL, "unknown flags 0x%x", flags);
    if (!!(flags & ARA_RNG_RECORD) + !!(flags & ARA_RNG_OCCURRENCE) + !!(flags & ARA_RNG_SUPPLIED) > 1)
        return fail(ARA_EINVAL, "ARA_RNG_RECORD, ARA_RNG_OCCURRENCE and ARA_RNG_SUPPLIED are exclusive");
    const bool supplied = (flags & ARA_RNG_SUPPLIED) && (flags & ARA_SU);
    if (supplied && (!p->d_rec_z || !y->d_zprog))
        return fail(ARA_EINVAL, "ARA_RNG_SUPPLIED needs ara_portfolio_set_z and ara_yet_set_z");
    if (supplied && p->max_prog >= y->zprog_programs)
        return fail(ARA_EINVAL, "the YET supplies z_(Prog,E) for %u programs; the portfolio uses program %u",
                    y->zprog_programs, p->max_prog);
    if (y->dev.n_trials == 0) return ARA_OK;
    if (!ylt) return fail(ARA_EINVAL, "ylt is NULL");
    if ((dbg_count || dbg_hash) && !(flags & ARA_DEBUG_LOOKUP))
        return fail(ARA_EINVAL, "dbg_count/dbg_hash need ARA_DEBUG_LOOKUP");
    if (!is_device_ptr(ylt)) return fail(ARA_EINVAL, "ylt must be device memory");
    if (occ_max && !is_device_ptr(occ_max)) return fail(ARA_EINVAL, "occ_max must be device memory");
    CU(enter_device(c->device));
    const uint64_t N = y->dev.n_trials;
    const bool exact = (flags & ARA_EXACT) != 0 && (flags & ARA_SU) != 0;
    const bool async = (flags & ARA_ASYNC) != 0;
    if (async) {                                       // per-run counters only; errors stay latched
        CU(cudaMemsetAsync(c->d_status, 0, kRunCounters, c->stream));
    } else {
        CU(fold_latched(c));
        CU(cudaMemsetAsync(c->d_status, 0, sizeof(RunStatus), c->stream));
    }
    c->timing_pending = true;
    c->timing_tail = false;
    c->timing_batches = 0;
    // ARA_RNG_RECORD with occ_max (a rare combination) runs on the fp64-capable kernel
    const bool za_om = (flags & (ARA_RNG_RECORD | ARA_RNG_SUPPLIED)) && (flags & ARA_SU) && occ_max;
    double ms_ovf = 0.0;
    uint32_t n_batches = 0;
    const bool primary = !(flags & ARA_DEBUG_LOOKUP) && (!(flags & ARA_SU) || p->dev.all_sigma_zero) &&
                         env_u64("ARA_NO_PRIMARY_PATH", 0) == 0;
    if (primary) {
        // no draw is taken: one streaming pass over the per-(event, layer)
        // occurrence losses computed at ara_create_portfolio
        PrimaryArgs P{p->dev, y->dev, ylt, occ_max, c->d_status, c->d_sched, p->dev.occ, p->dev.occ_lp};
        CU(cudaMemsetAsync(c->d_sched, 0, sizeof(unsigned long long), c->stream));
        CU(cudaEventRecord(c->ev[0], c->stream));
        CU(launch_primary(P, c->stream, c->num_sms));
        CU(cudaEventRecord(c->ev[1], c->stream));
        c->last_batches = 0;
        c->last_launches = 1;
        if (async) {
            c->async_pending = true;
            return ARA_OK;
        }
        CU(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    } else if (!exact && !za_om && p->dev.n_layers <= kSplitMaxLayers) {
        const SplitPlan pl = plan_split(p, y, flags);
        const uint32_t cap = pl.cap;
        SplitArgs S{};
        S.pf = p->dev; S.yet = y->dev; S.seed = seed; S.flags = flags; S.ylt = ylt;
        S.dbg_count = dbg_count; S.dbg_hash = dbg_hash; S.status = c->d_status; S.cap = cap;
        S.ovf = y->d_ovf; S.ovf_n = y->d_ovf_n; S.redo = y->d_redo;
        S.occ_max = occ_max;
        S.rng_mode = supplied ? 3u : (flags & ARA_RNG_RECORD) ? 1u : (flags & ARA_RNG_OCCURRENCE) ? 2u : 0u;
        S.zp_sup = y->d_zprog; S.zp_stride = y->dev.n_events; S.ze_sup = p->d_rec_z;
        S.ze_mask = S.rng_mode == 2 ? 0u : 0xffffffffu;
        S.ze_tag = S.rng_mode == 2 ? 7u : 2u;
        S.kbits = pl.kbits;
        S.kmask = (1u << pl.kbits) - 1u;
        const uint64_t pair_bytes = S.kbits ? 4 : 8;
        for (int r = 0; r < 10; ++r) {                   // Philox4x32-10 key schedule of the seed
            S.pkey[2 * r] = (uint32_t)seed + (uint32_t)r * 0x9E3779B9u;
            S.pkey[2 * r + 1] = (uint32_t)(seed >> 32) + (uint32_t)r * 0xBB67AE85u;
        }
        // batches of trials: batch b's compaction (stream cs) runs beside batch
        // b-1's sampling (the context stream) on the same SMs; two slots
        const uint64_t batch = pl.batch;
        n_batches = pl.n_batches;
        const bool serial = env_u64("ARA_OVERLAP", 0) == 0;  // two-stream overlap: an experiment (slower)
        cudaStream_t ss = c->stream, cs = serial ? c->stream : c->cstream;
        const uint64_t slot_bytes = pl.slot_bytes;
        CU(grow(&c->d_slots, c->slots_capacity, (serial ? 1 : 2) * slot_bytes));   // (no-op after ara_prepare)
        CU(grow(&c->d_counts, c->counts_capacity, N));
        S.counts = c->d_counts;
        CU(cudaMemsetAsync(c->d_sched, 0, (2 * kMaxBatches + 4) * sizeof(unsigned long long), ss));
        CU(cudaEventRecord(c->ev[0], ss));
        if (cs != ss) CU(cudaStreamWaitEvent(cs, c->ev[0], 0));
        for (uint32_t b = 0; b < n_batches; ++b) {
            SplitArgs B = S;
            B.t0 = (uint32_t)(b * batch);
            B.n_items = (uint32_t)std::min<uint64_t>(batch, N - b * batch);
            B.pairs = reinterpret_cast<uint2 *>(c->d_slots + (serial ? 0 : (b & 1)) * slot_bytes);
            cudaEvent_t *te = c->tev + 4 * b;            // compact begin/end, sample begin/end
            if (b >= 2 && cs != ss) CU(cudaStreamWaitEvent(cs, c->tev[4 * (b - 2) + 3], 0));   // slot free
            CU(cudaEventRecord(te[0], cs));
            B.sched = c->d_sched + 2 * b;
            CU(launch_compact(B, cs, c->num_sms));
            CU(cudaEventRecord(te[1], cs));
            if (cs != ss) CU(cudaStreamWaitEvent(ss, te[1], 0));
            CU(cudaEventRecord(te[2], ss));
            B.sched = c->d_sched + 2 * b + 1;
            CU(launch_sample(B, ss, c->num_sms));
            CU(cudaEventRecord(te[3], ss));
        }
        CU(cudaEventRecord(c->ev[1], ss));
        c->timing_batches = n_batches;
        if (async) {
            // device-sized tail passes, no host decision: the overflow plan
            // (offsets into the pre-sized pool), the overflow compaction and
            // sampling, the fp64 redo of table-less trials
            const uint64_t pool_pairs = default_pool_pairs(pl, N);
            CU(grow(&c->d_pool, c->pool_capacity, pool_pairs * pair_bytes));
            CU(grow(&c->d_pool_off, c->pool_off_capacity, N));
            CU(cudaEventRecord(c->ev[2], ss));
            CU(launch_ovf_plan(c->d_status, y->d_ovf_n, c->d_pool_off, c->pool_capacity / pair_bytes, ss));
            SplitArgs O = S;
            O.n_items = 0;
            O.n_items_dev = &c->d_status->n_ovf_fit;
            O.list = y->d_ovf;
            O.pool_off = c->d_pool_off;
            O.pairs = reinterpret_cast<uint2 *>(c->d_pool);
            O.cap = 0xffffffffu;
            O.sched = c->d_sched + 2 * kMaxBatches;
            CU(launch_compact(O, ss, c->num_sms));
            O.sched = c->d_sched + 2 * kMaxBatches + 1;
            CU(launch_sample(O, ss, c->num_sms));
            CU(launch_scan(p->dev, y->dev, seed, supplied ? flags : flags & ~ARA_RNG_SUPPLIED, ylt, dbg_count,
                           dbg_hash, c->d_status, y->d_redo, 0, nullptr, (flags & ARA_SU) != 0, ss, c->num_sms,
                           occ_max, y->d_zprog, y->dev.n_events, p->d_rec_z, &c->d_status->n_redo));
            CU(cudaEventRecord(c->ev[3], ss));
            c->timing_tail = true;
            c->last_batches = n_batches;
            c->last_launches = 2 * n_batches + 4;
            c->async_pending = true;
            return ARA_OK;
        }
        CU(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, ss));
        CU(cudaStreamSynchronize(ss));
        const uint32_t n_ovf = c->h_status->bad_event ? 0u : c->h_status->n_ovf;
        if (n_ovf) {
            NvtxRange nvtx_ovf("ara_run overflow pass");
            // overflow pass: the listed trials compacted again into exactly sized
            // regions of the pool, then sampled by the same kernel (same arithmetic)
            std::vector<uint32_t> cnt(n_ovf);
            std::vector<uint64_t> off(n_ovf);
            CU(cudaMemcpy(cnt.data(), y->d_ovf_n, n_ovf * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            uint64_t tot = 0;
            for (uint32_t i = 0; i < n_ovf; ++i) { off[i] = tot; tot += cnt[i]; }
            CU(grow(&c->d_pool, c->pool_capacity, std::max<uint64_t>(tot, 1) * pair_bytes));
            CU(grow(&c->d_pool_off, c->pool_off_capacity, n_ovf));
            CU(cudaMemcpyAsync(c->d_pool_off, off.data(), n_ovf * sizeof(uint64_t), cudaMemcpyHostToDevice, ss));
            SplitArgs O = S;
            O.n_items = n_ovf;
            O.list = y->d_ovf;
            O.pool_off = c->d_pool_off;
            O.pairs = reinterpret_cast<uint2 *>(c->d_pool);
            O.cap = 0xffffffffu;
            CU(cudaEventRecord(c->ev[2], ss));
            O.sched = c->d_sched + 2 * kMaxBatches;
            CU(launch_compact(O, ss, c->num_sms));
            O.sched = c->d_sched + 2 * kMaxBatches + 1;
            CU(launch_sample(O, ss, c->num_sms));
            CU(cudaEventRecord(c->ev[3], ss));
            CU(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, ss));
            CU(cudaStreamSynchronize(ss));
            float a = 0;
            CU(cudaEventElapsedTime(&a, c->ev[2], c->ev[3]));
            ms_ovf = a;
        }
    } else {
        // ARA_EXACT (fp64 solve for every sample): the fused kernel
        CU(cudaEventRecord(c->ev[0], c->stream));
        CU(launch_scan(p->dev, y->dev, seed, supplied ? flags : flags & ~ARA_RNG_SUPPLIED, ylt, dbg_count,
                       dbg_hash, c->d_status, nullptr, 0, y->d_redo, exact, c->stream, c->num_sms, occ_max,
                       y->d_zprog, y->dev.n_events, p->d_rec_z));
        CU(cudaEventRecord(c->ev[1], c->stream));
        if (async) {
            c->last_batches = 0;
            c->last_launches = 1;
            c->async_pending = true;
            return ARA_OK;
        }
        CU(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
    }
    const bool redo_launched = c->h_status->n_redo && !c->h_status->bad_event;
    double ms_redo = 0.0;
    if (redo_launched) {
        // trials that met a table-less record: redo them with the fp64 kernel
        const unsigned int n_redo = c->h_status->n_redo;
        CU(cudaMemsetAsync(&c->d_status->next_trial, 0, sizeof(unsigned long long), c->stream));
        CU(cudaEventRecord(c->ev[2], c->stream));
        CU(launch_scan(p->dev, y->dev, seed, supplied ? flags : flags & ~ARA_RNG_SUPPLIED, ylt, dbg_count,
                       dbg_hash, c->d_status, y->d_redo, n_redo, nullptr, (flags & ARA_SU) != 0, c->stream,
                       c->num_sms, occ_max, y->d_zprog, y->dev.n_events, p->d_rec_z));
        CU(cudaEventRecord(c->ev[3], c->stream));
        CU(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        float r = 0;
        CU(cudaEventElapsedTime(&r, c->ev[2], c->ev[3]));
        ms_redo = r;
    }
    c->timing_tail = ms_ovf > 0.0 || redo_launched;
    if (ms_ovf > 0.0 && !redo_launched) CU(cudaEventRecord(c->ev[3], c->stream));   // (ev[3] already after the pass)
    CU(compute_timings(c));
    if (redo_launched && ms_ovf > 0.0) c->last_ms[2] = ms_ovf + ms_redo;   // two tail passes: both timed
    c->last_batches = n_batches;
    c->last_launches = (n_batches ? 2 * n_batches : 1) + (ms_ovf > 0.0 ? 2 : 0) + (redo_launched ? 1 : 0);
    if (c->h_status->bad_event) {      // error path: count the offending occurrences
        CU(launch_count_bad(y->d_events, y->dev.n_events, p->dev.catalog, &c->d_status->bad_event, c->stream,
                            c->num_sms));
        CU(cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        return fail(ARA_ERANGE, "%u event occurrences have event id >= catalog_size %u",
                    c->h_status->bad_event, p->dev.catalog);
    }
    if (c->h_status->nonconverged)
        return fail(ARA_ECONVERGE, "beta quantile did not converge for %u samples",
                    c->h_status->nonconverged);
    return ARA_OK;
}

int ara_prepare(ara_ctx *c, const ara_portfolio *p, const ara_yet *y, uint32_t flags) {
    if (!c || !p || !y) return fail(ARA_EINVAL, "ctx/portfolio/yet is NULL");
    CU(enter_device(c->device));
    if (flags & ARA_ASYNC) {                         // the pre-sized overflow pool of ARA_ASYNC runs
        const std::vector<const ara_portfolio *> gs =
            p->groups.empty() ? std::vector<const ara_portfolio *>{p}
                              : std::vector<const ara_portfolio *>(p->groups.begin(), p->groups.end());
        for (const ara_portfolio *g : gs) {
            const SplitPlan pl = plan_split(g, y, flags);
            CU(grow(&c->d_pool, c->pool_capacity, default_pool_pairs(pl, y->dev.n_trials) * (pl.kbits ? 4 : 8)));
        }
        CU(grow(&c->d_pool_off, c->pool_off_capacity, std::max<uint64_t>(y->dev.n_trials, 1)));
    }
    const std::vector<const ara_portfolio *> groups =
        p->groups.empty() ? std::vector<const ara_portfolio *>{p}
                          : std::vector<const ara_portfolio *>(p->groups.begin(), p->groups.end());
    for (const ara_portfolio *g : groups) {
        const SplitPlan pl = plan_split(g, y, flags);
        CU(grow(&c->d_slots, c->slots_capacity, (env_u64("ARA_OVERLAP", 0) ? 2 : 1) * pl.slot_bytes));
    }
    CU(grow(&c->d_counts, c->counts_capacity, std::max<uint64_t>(y->dev.n_trials, 1)));
    return ARA_OK;
}

int ara_last_run_launches(const ara_ctx *c, uint32_t *kernel_launches, uint32_t *batches) {
    if (!c) return fail(ARA_EINVAL, "ctx is NULL");
    if (kernel_launches) *kernel_launches = c->last_launches;
    if (batches) *batches = c->last_batches;
    return ARA_OK;
}

int ara_last_run_timings(const ara_ctx *cc, double *compact_ms, double *sample_ms, double *redo_ms) {
    if (!cc) return fail(ARA_EINVAL, "ctx is NULL");
    ara_ctx *c = const_cast<ara_ctx *>(cc);        // (the lazy evaluation of an ARA_ASYNC run's events)
    CU(enter_device(c->device));
    CU(compute_timings(c));
    if (compact_ms) *compact_ms = c->last_ms[0];
    if (sample_ms) *sample_ms = c->last_ms[1];
    if (redo_ms) *redo_ms = c->last_ms[2];
    return ARA_OK;
}

static uint64_t needed_rank(uint64_t N, double rp) {
    uint64_t fl, m;
    if (rp == std::floor(rp) && rp < 1.8e19) {
        const uint64_t R = (uint64_t)rp;
        fl = (N + 1) / R;
        m = (N + R - 1) / R;
    } else {
        fl = (uint64_t)std::floor((double)(N + 1) / rp);
        const uint64_t a = (uint64_t)std::floor((1.0 - 1.0 / rp) * (double)N) + 1;
        m = N - (a < N ? a : N) + 1;
    }
    uint64_t k = fl + 1 > m ? fl + 1 : m;
    if (k < 1) k = 1;
    if (k > N) k = N;
    return k;
}

int ara_exceedance_curve(ara_ctx *c, const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                         int32_t layer, float *losses_out) {
    if (!c || !ylt || !losses_out) return fail(ARA_EINVAL, "NULL argument");
    if (n_total == 0) return fail(ARA_EINVAL, "empty YLT");
    if (n_total > 0xffffffffull) return fail(ARA_EINVAL, "n_total must be < 2^32");
    if (n_layers == 0 || n_shards == 0 || n_total % n_shards)
        return fail(ARA_EINVAL, "need n_layers >= 1, n_shards >= 1 dividing n_total");
    if (layer < -1 || layer >= (int32_t)n_layers) return fail(ARA_EINVAL, "layer %d out of range", layer);
    if (!is_device_ptr(ylt) || !is_device_ptr(losses_out)) return fail(ARA_EINVAL, "ylt and losses_out must be device memory");
    CU(enter_device(c->device));
    const uint64_t need = 2 * n_total + 256ull * (2 * (uint64_t)c->num_sms);
    if (c->ep_capacity < need) {                       // scratch grows once, then is reused
        cudaFree(c->d_ep);
        c->d_ep = nullptr;
        c->ep_capacity = 0;
        CU(dalloc(&c->d_ep, need));
        c->ep_capacity = need;
    }
    CU(launch_exceedance_curve(ylt, n_layers, n_total, n_shards, layer, c->d_ep, losses_out, c->stream,
                               c->num_sms));
    return ARA_OK;
}

int ara_risk_measures(ara_ctx *c, const float *ylt, uint32_t n_layers, uint64_t n_total,
                      uint32_t n_shards, int32_t layer, const double *rps, uint32_t n_rp,
                      double *pml_out, double *tvar_out) {
    return ara_risk_measures_var(c, ylt, n_layers, n_total, n_shards, layer, rps, n_rp, pml_out, tvar_out,
                                 nullptr);
}

// the joint-select launches of ara_risk_measures_batch / _async, results to device d_out
static int measures_enqueue(ara_ctx *c, const float *ylt, uint32_t n_layers, uint64_t n_total,
                            uint32_t n_shards, const int32_t *layers, uint32_t n_sel, const double *rps,
                            uint32_t n_rp, double *d_out) {
    if (n_total == 0) return fail(ARA_EINVAL, "empty YLT");
    if (n_layers == 0 || n_shards == 0 || n_total % n_shards)
        return fail(ARA_EINVAL, "need n_layers >= 1, n_shards >= 1 dividing n_total");
    if (n_sel == 0 || n_sel > ARA_MAX_PORTFOLIO_LAYERS + 1) return fail(ARA_EINVAL, "n_sel out of range");
    if (n_rp == 0 || n_rp > 4) return fail(ARA_EINVAL, "n_rp must be in [1, 4] (ara_risk_measures for more)");
    for (uint32_t q = 0; q < n_rp; ++q)
        if (!(rps[q] > 1.0) || !std::isfinite(rps[q]))
            return fail(ARA_EINVAL, "return period %g must be finite and > 1", rps[q]);
    for (uint32_t i = 0; i < n_sel; ++i)
        if (layers[i] < -1 || layers[i] >= (int32_t)n_layers) return fail(ARA_EINVAL, "layer %d out of range", layers[i]);
    if (!is_device_ptr(ylt)) return fail(ARA_EINVAL, "ylt must be device memory");
    CU(enter_device(c->device));
    if (c->ms.capacity < n_total) {
        cudaFree(c->ms.vals);
        c->ms.vals = nullptr;
        c->ms.capacity = 0;
        CU(dalloc(&c->ms.vals, n_total));
        c->ms.capacity = n_total;
    }
    // one joint-select launch per table, back to back on the stream
    for (uint32_t i = 0; i < n_sel; ++i)
        CU(launch_measures_multi(ylt, n_layers, n_total, n_shards, layers[i], rps, n_rp, c->ms,
                                 d_out + 3 * n_rp * i, c->stream));
    return ARA_OK;
}

int ara_risk_measures_async(ara_ctx *c, const float *ylt, uint32_t n_layers, uint64_t n_total,
                            uint32_t n_shards, const int32_t *layers, uint32_t n_sel, const double *rps,
                            uint32_t n_rp, double *d_out) {
    NvtxRange nvtx("ara_risk_measures_async");
    if (!c || !ylt || !layers || !rps || !d_out) return fail(ARA_EINVAL, "NULL argument");
    if (!is_device_ptr(d_out)) return fail(ARA_EINVAL, "d_out must be device memory");
    return measures_enqueue(c, ylt, n_layers, n_total, n_shards, layers, n_sel, rps, n_rp, d_out);
}

int ara_risk_measures_batch(ara_ctx *c, const float *ylt, uint32_t n_layers, uint64_t n_total,
                            uint32_t n_shards, const int32_t *layers, uint32_t n_sel, const double *rps,
                            uint32_t n_rp, double *pml_out, double *tvar_out, double *var_out) {
    NvtxRange nvtx("ara_risk_measures_batch");
    if (!c || !ylt || !layers || !rps || !pml_out || !tvar_out) return fail(ARA_EINVAL, "NULL argument");
    // one read-back for every table
    const int st = measures_enqueue(c, ylt, n_layers, n_total, n_shards, layers, n_sel, rps, n_rp, c->ms.d_out);
    if (st != ARA_OK) return st;
    double *out = c->h_out;
    CU(cudaMemcpyAsync(out, c->ms.d_out, 3 * n_rp * n_sel * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    for (uint32_t i = 0; i < n_sel; ++i)
        for (uint32_t q = 0; q < n_rp; ++q) {
            pml_out[i * n_rp + q] = out[3 * (n_rp * i + q)];
            tvar_out[i * n_rp + q] = out[3 * (n_rp * i + q) + 1];
            if (var_out) var_out[i * n_rp + q] = out[3 * (n_rp * i + q) + 2];
        }
    return ARA_OK;
}

int ara_risk_measures_var(ara_ctx *c, const float *ylt, uint32_t n_layers, uint64_t n_total,
                          uint32_t n_shards, int32_t layer, const double *rps, uint32_t n_rp,
                          double *pml_out, double *tvar_out, double *var_out) {
    NvtxRange nvtx("ara_risk_measures");
    if (!c || !ylt || !rps || !pml_out || !tvar_out) return fail(ARA_EINVAL, "NULL argument");
    if (n_total == 0) return fail(ARA_EINVAL, "empty YLT");
    if (n_layers == 0 || n_shards == 0 || n_total % n_shards)
        return fail(ARA_EINVAL, "need n_layers >= 1, n_shards >= 1 dividing n_total");
    if (layer < -1 || layer >= (int32_t)n_layers) return fail(ARA_EINVAL, "layer %d out of range", layer);
    if (n_rp == 0 || n_rp > 64) return fail(ARA_EINVAL, "n_rp must be in [1, 64]");
    uint64_t k_need = 1;
    for (uint32_t q = 0; q < n_rp; ++q) {
        if (!(rps[q] > 1.0) || !std::isfinite(rps[q]))
            return fail(ARA_EINVAL, "return period %g must be finite and > 1", rps[q]);
        const uint64_t k = needed_rank(n_total, rps[q]);
        if (k > k_need) k_need = k;
    }
    if (!is_device_ptr(ylt)) return fail(ARA_EINVAL, "ylt must be device memory");
    CU(enter_device(c->device));
    if (c->ms.capacity < n_total) {
        cudaFree(c->ms.vals);
        c->ms.vals = nullptr;
        c->ms.capacity = 0;
        CU(dalloc(&c->ms.vals, n_total));
        c->ms.capacity = n_total;
    }
    if (n_rp <= 4 && getenv("ARA_MEASURES_SORT") == nullptr) {   // joint select, one launch
        CU(launch_measures_multi(ylt, n_layers, n_total, n_shards, layer, rps, n_rp, c->ms, c->ms.d_out,
                                 c->stream));
    } else if (k_need <= kSortCap) {
        RpList R{};
        for (uint32_t q = 0; q < n_rp; ++q) R.v[q] = rps[q];
        CU(launch_measures(ylt, n_layers, n_total, n_shards, layer, R, n_rp, k_need, c->ms, c->ms.d_out,
                           c->stream));
    } else {   // deep ranks: a radix select per needed order statistic
        CU(launch_measures_deep(ylt, n_layers, n_total, n_shards, layer, rps, n_rp, c->ms,
                                c->ms.d_out, c->stream));
    }
    double *out = c->h_out;                      // pinned
    CU(cudaMemcpyAsync(out, c->ms.d_out, 3 * n_rp * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    for (uint32_t q = 0; q < n_rp; ++q) {
        pml_out[q] = out[3 * q];
        tvar_out[q] = out[3 * q + 1];
        if (var_out) var_out[q] = out[3 * q + 2];
    }
    return ARA_OK;
}

int ara_sample_losses(ara_ctx *c, uint64_t n, const ara_record *recs, const float *zp,
                      const float *ze, uint32_t flags, float *loss_out) {
    if (flags & ~ARA_EXACT) return fail(ARA_EINVAL, "unknown flags 0x%x", flags);
    if (!c) return fail(ARA_EINVAL, "ctx is NULL");
    if (n == 0) return ARA_OK;
    if (!recs || !zp || !ze || !loss_out) return fail(ARA_EINVAL, "NULL argument");
    for (uint64_t t = 0; t < n; ++t)
        if (!(zp[t] > 0.0f && zp[t] < 1.0f && ze[t] > 0.0f && ze[t] < 1.0f))
            return fail(ARA_EINVAL, "z values must lie in (0,1) (index %llu)", (unsigned long long)t);
    CU(enter_device(c->device));
    ara_record *d_raw = nullptr;
    BetaRec *d_recs = nullptr;
    float2 *d_nodes = nullptr;
    float *d_mu = nullptr, *d_zp = nullptr, *d_ze = nullptr, *d_out = nullptr;
    int code = ARA_OK;
    cudaError_t e = cudaSuccess;
    if (dalloc(&d_raw, n) || dalloc(&d_recs, n) || dalloc(&d_mu, n) || dalloc(&d_zp, n) ||
        dalloc(&d_ze, n) || dalloc(&d_out, n) || dalloc(&d_nodes, n * kTabNodes + kTabPad)) {
        cudaGetLastError();
        code = fail(ARA_ENOMEM, "device allocation failed");
    } else {
        cudaStream_t s = c->stream;
        e = cudaMemcpyAsync(d_raw, recs, n * sizeof(ara_record), cudaMemcpyHostToDevice, s);
        if (!e) e = cudaMemcpyAsync(d_zp, zp, n * sizeof(float), cudaMemcpyHostToDevice, s);
        if (!e) e = cudaMemcpyAsync(d_ze, ze, n * sizeof(float), cudaMemcpyHostToDevice, s);
        if (!e) e = cudaMemsetAsync(c->d_status, 0, sizeof(RunStatus), s);
        if (!e) e = cudaMemsetAsync(d_nodes, 0, (n * kTabNodes + kTabPad) * sizeof(float2), s);
        if (!e) { launch_prep_records(d_raw, nullptr, n, d_recs, d_mu, d_nodes + kTabPad, nullptr, s); e = cudaGetLastError(); }
        if (!e) e = launch_sample_losses(d_recs, TablePtr{d_nodes + kTabPad}, d_zp, d_ze, n, (flags & ARA_EXACT) != 0, d_out,
                                         c->d_status, s);
        if (!e) e = cudaMemcpyAsync(loss_out, d_out, n * sizeof(float), cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, s);
        if (!e) e = cudaStreamSynchronize(s);
        if (e) code = fail(ARA_ECUDA, "ara_sample_losses: %s", cudaGetErrorString(e));
        else if (c->h_status->nonconverged)
            code = fail(ARA_ECONVERGE, "beta quantile did not converge for %u samples", c->h_status->nonconverged);
    }
    cudaFree(d_raw); cudaFree(d_recs); cudaFree(d_mu); cudaFree(d_zp); cudaFree(d_ze); cudaFree(d_out);
    cudaFree(d_nodes);
    return code;
}

int ara_beta_quantiles(ara_ctx *c, uint64_t n, const double *alpha, const double *beta, const double *v,
                       double *x_out, double *y_out) {
    if (!c) return fail(ARA_EINVAL, "ctx is NULL");
    if (n == 0) return ARA_OK;
    if (!alpha || !beta || !v || !x_out || !y_out) return fail(ARA_EINVAL, "NULL argument");
    for (uint64_t t = 0; t < n; ++t)
        if (!(alpha[t] > 0.0 && beta[t] > 0.0 && std::isfinite(alpha[t]) && std::isfinite(beta[t]) &&
              std::isfinite(v[t])))
            return fail(ARA_EINVAL, "need finite alpha, beta > 0 and finite v (index %llu)", (unsigned long long)t);
    CU(enter_device(c->device));
    double *d = nullptr;
    int code = ARA_OK;
    if (dalloc(&d, 5 * n)) {
        cudaGetLastError();
        return fail(ARA_ENOMEM, "device allocation failed");
    }
    cudaStream_t s = c->stream;
    cudaError_t e = cudaMemcpyAsync(d, alpha, n * sizeof(double), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemcpyAsync(d + n, beta, n * sizeof(double), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemcpyAsync(d + 2 * n, v, n * sizeof(double), cudaMemcpyHostToDevice, s);
    if (!e) e = cudaMemsetAsync(c->d_status, 0, sizeof(RunStatus), s);
    if (!e) e = launch_beta_quantiles(d, d + n, d + 2 * n, n, d + 3 * n, d + 4 * n, c->d_status, s);
    if (!e) e = cudaMemcpyAsync(x_out, d + 3 * n, n * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(y_out, d + 4 * n, n * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaMemcpyAsync(c->h_status, c->d_status, sizeof(RunStatus), cudaMemcpyDeviceToHost, s);
    if (!e) e = cudaStreamSynchronize(s);
    if (e) code = fail(ARA_ECUDA, "ara_beta_quantiles: %s", cudaGetErrorString(e));
    else if (c->h_status->nonconverged)
        code = fail(ARA_ECONVERGE, "beta quantile did not converge for %u values", c->h_status->nonconverged);
    cudaFree(d);
    return code;
}

int ara_draw_uniforms(ara_ctx *c, uint64_t seed, uint64_t n, const uint32_t *ctr, float *u_out) {
    if (!c) return fail(ARA_EINVAL, "ctx is NULL");
    if (n == 0) return ARA_OK;
    if (!ctr || !u_out) return fail(ARA_EINVAL, "NULL argument");
    CU(enter_device(c->device));
    uint4 *d_ctr = nullptr;
    float *d_out = nullptr;
    int code = ARA_OK;
    if (dalloc(&d_ctr, n) || dalloc(&d_out, n)) {
        cudaGetLastError();
        code = fail(ARA_ENOMEM, "device allocation failed");
    } else {
        cudaError_t e = cudaMemcpyAsync(d_ctr, ctr, n * sizeof(uint4), cudaMemcpyHostToDevice, c->stream);
        if (!e) e = launch_draw_uniforms(seed, d_ctr, n, d_out, c->stream);
        if (!e) e = cudaMemcpyAsync(u_out, d_out, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream);
        if (!e) e = cudaStreamSynchronize(c->stream);
        if (e) code = fail(ARA_ECUDA, "ara_draw_uniforms: %s", cudaGetErrorString(e));
    }
    cudaFree(d_ctr); cudaFree(d_out);
    return code;
}

int ara_normal_quantiles(ara_ctx *c, uint64_t n, const uint32_t *bits, float *v_out) {
    if (!c) return fail(ARA_EINVAL, "ctx is NULL");
    if (n == 0) return ARA_OK;
    if (!bits || !v_out) return fail(ARA_EINVAL, "NULL argument");
    CU(enter_device(c->device));
    uint32_t *d_bits = nullptr;
    float *d_out = nullptr;
    int code = ARA_OK;
    if (dalloc(&d_bits, n) || dalloc(&d_out, n)) {
        cudaGetLastError();
        code = fail(ARA_ENOMEM, "device allocation failed");
    } else {
        cudaError_t e = cudaMemcpyAsync(d_bits, bits, n * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream);
        if (!e) e = launch_normal_quantiles(d_bits, n, d_out, c->stream);
        if (!e) e = cudaMemcpyAsync(v_out, d_out, n * sizeof(float), cudaMemcpyDeviceToHost, c->stream);
        if (!e) e = cudaStreamSynchronize(c->stream);
        if (e) code = fail(ARA_ECUDA, "ara_normal_quantiles: %s", cudaGetErrorString(e));
    }
    cudaFree(d_bits); cudaFree(d_out);
    return code;
}

}  // extern "C"
