// ara_internal.cuh -- device data layout shared by the host planner
// (ara_api.cu) and the kernels.  See DESIGN.md "Data layout in HBM".
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ara.h"

namespace ara {

// Per (layer, XELT) "slot": slots are numbered layer-major, in each layer's
// XELT order, so the present pairs of one occurrence, enumerated in slot
// order, are grouped by layer.
struct SlotInfo {
    uint32_t elt;       // XELT id j (keys z_(E), reading G2)
    uint32_t prog;      // program of the slot's layer (keys z_(Prog,E))
    uint32_t layer;     // layer index
    uint32_t has_terms; // 1 if XELT terms apply (G7)
    float ret, lim, share, pad;
};

struct LayerInfo {
    double occ_r, occ_l, agg_r, agg_l;
};

// Per-record sampler constants, derived on the device in fp64 from the
// record and stored fp32: 32 B, one L2 sector.
//   a, b      : alpha, beta, capped per G9
//   wi, wc    : sigma_I/sigma, sigma_C/sigma divided by sqrt(sum of squares)
//               (steps 3-4 of section 3.2 folded into two weights)
//   scale     : max_l; for degenerate records (G10) the loss itself
//   mu_l, sd_l: mean and sd of logit(X), X ~ Beta(a,b) (psi(a)-psi(b),
//               sqrt(psi1(a)+psi1(b))): initial guess of the fp64 solve
//   mode      : kModeTable (quantile table), kModeExact (per-sample fp64
//               solve), kModeDegenerate (loss = scale)
// quantile tables: lambda(v) = logit I^-1(Phi(v); a, b) at v = -7.75 + 0.5 j,
// j = 0..31 (|v| <= 7.48 for the draws of U's grid), 256 B per record in one
// array whose first node sits 64 B past a 128-B boundary: each record's
// central nodes j = 8..23 (v in [-3.75, 3.75], 99.98 % of samples) fill
// exactly one 128-B line -- the part that stays L2-resident -- and the nodes
// of any interval are adjacent (one address computation per sample; round 2's
// separate hot / cold arrays cost a 64-bit select per sample)
constexpr int kTabNodes = 32;
constexpr float kTabV0 = -7.75f, kTabH = 0.5f;
constexpr int kTabPad = 8;    // float2 before node 0 of record 0 (64 B)
constexpr float kTabDegenerate = 88.0f;   // every node of a degenerate record's table (G10): x = 1
struct TablePtr {
    const float2 *nodes;      // [records][kTabNodes], nodes - kTabPad is 128-B aligned
};
// the nodes of interval ti (ti, ti + 1 adjacent) of record rec
__device__ __forceinline__ const float2 *table_row(const TablePtr &T, uint64_t rec, int ti) {
    return (T.nodes + ti) + rec * kTabNodes;
}

// Shared-memory copy of a presence bitmap (words) plus one zero word after it
// (the sentinel event's bit), by bulk asynchronous copies (TMA engine,
// cp.async.bulk) completing on an mbarrier: one thread issues the 16-B
// multiple in 32 KiB pieces, the block writes the remaining <= 3 words and the
// zero word, then every thread waits on the barrier.  smem: the bitmap at
// offset 0 (16-B aligned), the 8-B barrier at bitmap_smem_barrier(words).
// The per-thread load loop it replaced kept one load in flight per thread
// (10 % of the primary kernel's stall samples at cfg2).
__host__ __device__ constexpr uint32_t bitmap_smem_barrier(uint32_t words) { return ((words + 1) * 4u + 15u) & ~15u; }
__host__ __device__ constexpr uint32_t bitmap_smem_bytes(uint32_t words) { return bitmap_smem_barrier(words) + 16u; }
__device__ __forceinline__ void load_bitmap_smem(unsigned char *smem, const uint32_t *__restrict__ g, uint32_t words) {
    uint32_t *bm = reinterpret_cast<uint32_t *>(smem);
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(smem + bitmap_smem_barrier(words));
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t bulk = (words * 4u) & ~15u;                  // bytes by the copy engine
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bulk) : "memory");
        for (uint32_t o = 0; o < bulk; o += 32768u) {
            const uint32_t n = bulk - o < 32768u ? bulk - o : 32768u;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(dst + o), "l"(reinterpret_cast<const unsigned char *>(g) + o), "r"(n), "r"(bar)
                         : "memory");
        }
    }
    for (uint32_t t = bulk / 4u + threadIdx.x; t <= words; t += blockDim.x) bm[t] = t < words ? g[t] : 0u;
    __syncthreads();                                            // (the barrier is initialised; the tail written)
    uint32_t done = 0;
    while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(bar) : "memory");
}

constexpr uint32_t kModeTable = 0, kModeExact = 1, kModeDegenerate = 2;
struct __align__(16) BetaRec {
    float a, b, wi, wc;
    float scale, mu_l, sd_l;
    uint32_t mode;
};

// Per device record ((layer, XELT) slot, record) constants of the split
// sampler (32 B, one L2 sector): the beta parameters and weights of the
// record's BetaRec plus the draw keys, so a pair is sampled from this one
// load.  meta: slot | run_end << 8 | layer << 16 | mode << 28 (run_end: last
// record of its (event, layer) run); tab: the input record (its quantile
// table, shared by every slot of the XELT); key: XELT id | program << 24
// (ARA_MAX_XELTS, ARA_MAX_PROGRAMS).
struct __align__(32) SplitRec {    // 32 B: one 256-bit load
    float a, b, wi, wc;
    float scale;
    uint32_t meta;
    uint32_t tab, key;
};

// ARA_DEVICE_CHECKS builds (tools/build_variant.sh chk -DARA_DEVICE_CHECKS=1)
// trap on a failed bounds check in the hot kernels: the GPU test suite runs
// against such a build as a bounds-checked pass (compute-sanitizer is not
// available on every pool)
#ifndef ARA_DEVICE_CHECKS
#define ARA_DEVICE_CHECKS 0
#endif
#define ARA_CHECK(cond)                                   \
    do {                                                  \
        if (ARA_DEVICE_CHECKS && !(cond)) __trap();       \
    } while (0)

struct PortfolioDev {
    uint32_t catalog;
    uint32_t n_slots, n_layers;
    uint32_t bitmap_shift;    // event e -> presence bit e >> shift
    uint32_t bitmap_words;
    uint32_t sentinel_event;  // an id whose presence bit is 0 (bit index bitmap_words * 32: the zero word
                              // appended in shared memory, or a zero bit of the bitmap)
    uint32_t sentinel_ok;     // 0: no such id fits in 32 bits (per-event length test instead)
    uint64_t n_dev_records;
    uint32_t n_exact_records; // records without a quantile table (fp64 per-sample solve)
    uint64_t n_tables;        // input records in the record store (quantile tables)
    const uint32_t *bitmap;   // [bitmap_words]
    const BetaRec *recs;      // [input records] (the record store, shared by the groups)
    TablePtr tables;          // [input records] (lambda, lambda') nodes
    const float *rec_mu;      // [input records] mean loss (primary uncertainty)
    const uint32_t *rec_orig; // [n_dev_records] record index within its XELT
    const uint2 *cidx;        // [catalog] (first device record, record count) of each event
    const uint32_t *cidx4;    // [catalog] the same packed as first | count << 24, or null (>= 2^24 device records)
    const SplitRec *srecs;    // [n_dev_records]
    const uint2 *mu_meta;     // [n_dev_records] (mean loss bits, meta = slot | run_end << 8 | layer << 16):
                              // one 8 B gather per pair with SU off
    uint32_t any_terms;       // some slot has XELT terms (G7)
    uint32_t all_sigma_zero;  // every record has sigma_I = sigma_C = 0 (no draw is ever taken, G10)
    uint32_t occ_lp;          // occurrence losses per event in occ (n_layers rounded up to 1, 2, 4, 8)
    const float *occ;         // [catalog][occ_lp] occurrence loss of each (event, layer) without draws
                              // (lines 6-11 at the mean losses; the primary-uncertainty fast path)
    const uint32_t *occ_bitmap; // [bitmap_words] as bitmap, but bit set only if some event of the bit has a
                              // nonzero occurrence loss in some layer (the primary path's filter; a subset
                              // of the presence bits, so the sentinel event's bit is 0 here too)
    const SlotInfo *slots;    // [n_slots]
    const LayerInfo *layers;  // [n_layers]
};

struct YetDev {
    uint64_t n_trials, first_trial;
    uint32_t fixed_len;       // 0 => CSR
    const uint64_t *offsets;  // device [n_trials+1] or null
    const uint32_t *events;   // allocation padded by 16 B (bulk copies round up)
    uint64_t n_events;
    const uint32_t *max_event;  // device word: largest event id (set at every upload)
};

// device-side status words: the per-run counters first (zeroed by every
// run), then the error counters (zeroed by a synchronous run, accumulated
// across ARA_ASYNC runs until ara_ctx_synchronize reads them)
struct RunStatus {
    unsigned long long next_trial;   // dynamic trial scheduler of the fused kernel
    unsigned int n_redo;             // trials touching a table-less record (fp64 kernel)
    unsigned int n_ovf;              // trials whose pairs overflowed their batch region
    unsigned int n_ovf_fit;          // ARA_ASYNC: overflow trials that fit the pre-sized pool
    unsigned int pad0;
    unsigned long long pad1;
    unsigned int nonconverged;       // fp64 solves that did not converge
    unsigned int bad_event;          // != 0: some event id >= catalog (count on the error path)
    unsigned int pool_short;         // ARA_ASYNC: overflow trials that did not fit (YLT not written)
    unsigned int pad2;
};
constexpr size_t kRunCounters = 32;  // bytes of RunStatus zeroed by every run

// The split (two-kernel) scan, run batch by batch on two streams:
// compact_kernel writes each trial's present pairs {device record, k} to its
// region of the batch's slot (cap pairs) and their count to counts[t]
// (kOverflow if more than cap: the trial is listed in ovf / ovf_n with its
// exact count and compacted again by the overflow pass into an exactly
// sized region of the overflow pool); sample_kernel samples them.
constexpr uint32_t kOverflow = 0xffffffffu;
constexpr uint32_t kSplitMaxLayers = 8;   // larger portfolios run in groups of layers
struct SplitArgs {
    PortfolioDev pf;
    YetDev yet;
    uint64_t seed;
    uint32_t flags;
    float *ylt;
    uint32_t *dbg_count;
    uint64_t *dbg_hash;
    RunStatus *status;
    // work items of this launch: trial t0 + i (batch), or list[i] (overflow pass)
    uint32_t t0, n_items;
    const unsigned int *n_items_dev;   // non-null: the item count is read on the device (ARA_ASYNC)
    const uint32_t *list;
    const uint64_t *pool_off;     // overflow pass: region of item i in the pool (pair units)
    unsigned long long *sched;    // this launch's dynamic-scheduler counter (zeroed)
    uint2 *pairs;                 // the batch's slot, or the overflow pool
    uint32_t cap;                 // pairs per batch region
    uint32_t *counts;             // [n_trials]
    uint32_t *ovf, *ovf_n;        // overflowing trials and their exact pair counts (status->n_ovf)
    uint32_t *redo;               // trials with a table-less record (fp64 kernel)
    uint32_t pkey[20];            // Philox key schedule of the seed (round r: pkey[2r], pkey[2r+1])
    uint32_t kbits;               // > 0: pairs packed in 4 B as device record << kbits | k
    uint32_t kmask;               // (1 << kbits) - 1
    float *occ_max;               // null, or [n_layers][n_trials] largest occurrence loss (G29)
    uint32_t rng_mode;            // 0: reading G2; 1: ARA_RNG_RECORD; 2: ARA_RNG_OCCURRENCE; 3: ARA_RNG_SUPPLIED
    const float *zp_sup;          // mode 3: z_(Prog,E) per YET occurrence, [program][zp_stride]
    uint64_t zp_stride;           // occurrences of the YET
    const float *ze_sup;          // mode 3: z_(E) per device record
    uint32_t ze_mask, ze_tag;     // z_(E) counter (trial, k, elt & ze_mask, ze_tag) in modes 0 and 2
};
size_t sample_smem_bytes(uint32_t n_layers, bool occ_max);
// cached attribute / occupancy set-up of a kernel launch (per device)
cudaError_t prepare_launch(const void *kern, size_t smem, int threads, int &per_sm);

// the primary-uncertainty fast path (ara_primary.cu)
struct PrimaryArgs {
    PortfolioDev pf;
    YetDev yet;
    float *ylt;
    float *occ_max;
    RunStatus *status;
    unsigned long long *sched;
    const float *occ;
    uint32_t lp;
};
cudaError_t launch_primary(const PrimaryArgs &A, cudaStream_t s, int num_sms);
void launch_occ_table(const uint2 *cidx, const uint2 *mu_meta, const double *slot_terms,
                      const LayerInfo *layers, uint32_t n_layers, uint32_t lp, uint32_t catalog, float *out,
                      cudaStream_t s);
void launch_occ_bitmap(const float *occ, uint32_t lp, uint32_t catalog, uint32_t shift, uint32_t words,
                       uint32_t *out, cudaStream_t s);
cudaError_t launch_compact(const SplitArgs &A, cudaStream_t s, int num_sms);
// ARA_ASYNC overflow plan: exclusive scan of the listed trials' pair counts
// into pool offsets, as many as fit pool_pairs (status->n_ovf_fit; the rest
// counted in status->pool_short)
cudaError_t launch_ovf_plan(RunStatus *status, const uint32_t *ovf_n, uint64_t *pool_off, uint64_t pool_pairs,
                            cudaStream_t s);
cudaError_t launch_sample(const SplitArgs &A, cudaStream_t s, int num_sms);
cudaError_t launch_unpack_yet(const uint32_t *packed, uint64_t n, uint32_t bits, uint32_t *out, cudaStream_t s,
                              int num_sms);
cudaError_t launch_yet_max(const uint32_t *ev, uint64_t n, uint32_t *out, cudaStream_t s, int num_sms);
cudaError_t launch_count_bad(const uint32_t *ev, uint64_t n, uint32_t C, unsigned int *out, cudaStream_t s,
                             int num_sms);

// kernels
void launch_split_recs(const BetaRec *recs, const uint32_t *rec_src, const uint32_t *rec_meta,
                       const SlotInfo *slots, const float *mu, uint64_t n, SplitRec *out, uint2 *mu_meta,
                       cudaStream_t s);
void launch_prep_records(const ara_record *raw, const uint32_t *rec_src, uint64_t n,
                         BetaRec *out, float *out_mu, float2 *nodes,
                         unsigned int *n_exact, cudaStream_t s);
// Scan every trial of `yet`, or (trial_list != null) only the n_list listed
// trials.  Without ARA_EXACT the table-only kernel runs and appends to
// `redo` every trial that met a table-less record; the caller re-runs those
// with exact = true (the fp64 per-sample kernel).
cudaError_t launch_scan(const PortfolioDev &pf, const YetDev &yet, uint64_t seed, uint32_t flags,
                        float *ylt, uint32_t *dbg_count, uint64_t *dbg_hash, RunStatus *status,
                        const uint32_t *trial_list, uint64_t n_list, uint32_t *redo, bool exact_kernel,
                        cudaStream_t s, int num_sms, float *occ_max = nullptr, const float *zp_sup = nullptr,
                        uint64_t zp_stride = 0, const float *ze_sup = nullptr,
                        const unsigned int *n_list_dev = nullptr);
cudaError_t launch_sample_losses(const BetaRec *recs, TablePtr tables,
                                 const float *zp,
                                 const float *ze, uint64_t n, bool exact, float *out,
                                 RunStatus *status, cudaStream_t s);
cudaError_t launch_normal_quantiles(const uint32_t *bits, uint64_t n, float *out, cudaStream_t s);
cudaError_t launch_beta_quantiles(const double *a, const double *b, const double *v, uint64_t n, double *x_out,
                                  double *y_out, RunStatus *status, cudaStream_t s);
cudaError_t launch_draw_uniforms(uint64_t seed, const uint4 *ctr, uint64_t n, float *out,
                                 cudaStream_t s);

}  // namespace ara
