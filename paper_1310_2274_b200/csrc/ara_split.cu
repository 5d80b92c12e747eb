// ara_split.cu -- the two-kernel form of the YET scan (Algorithm 1,
// P:134-170), the default path of ara_run:
//
//   compact_kernel : YET stream (line 4) + direct-access lookup (line 6):
//                    presence bitmap, then the event index entry of each hit;
//                    per trial, the present (occurrence, slot) pairs
//                    {device record, k} written to a fixed-capacity region
//                    of HBM
//   sample_kernel  : per trial, dense 64-pair rounds of draws (line 7,
//                    section 3) and XELT terms (line 8), the per-occurrence
//                    sums (line 9) by segmented warp scans in registers,
//                    occurrence terms (line 11), trial sums, aggregate terms
//                    (line 12) -> YLT (line 17).  Bound by the ALU pipes.
//
// A trial whose pairs overflow its region, or that meets a table-less record,
// is listed for the fused fp64-capable kernel (ara_kernels.cu).
#include <algorithm>
#include <mutex>
#include <vector>
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"
#include "ara_sampler.cuh"

namespace ara {

namespace {

// One CTA of 32 warps per SM for each kernel, <= 64 registers per thread.
// (16 + 16 warps, so that a batch's compaction could share the SMs with the
// previous batch's sampling on a second stream, measured slower: both
// kernels load the L1/LSU pipe.)
#ifndef ARA_COMPACT_WARPS
#define ARA_COMPACT_WARPS 32
#endif
constexpr int kCompactThreads = ARA_COMPACT_WARPS * 32;   // compaction (bitmap in shared memory)
#ifndef ARA_SAMPLE_WARPS
#define ARA_SAMPLE_WARPS 32
#endif
constexpr int kSampleWarps = ARA_SAMPLE_WARPS;            // sampling
#ifndef ARA_SAMPLE_U
#define ARA_SAMPLE_U 2                // pairs per lane in flight per sampler round
#endif
constexpr int kU = ARA_SAMPLE_U;
#ifndef ARA_XCAP
#define ARA_XCAP 512
#endif
constexpr uint32_t kXCap = ARA_XCAP;    // pairs per sampler segment (a multiple of 32 kU, >= ARA_MAX_SLOTS; the
                                        // shared memory left to L1 serves the record and table gathers)
#ifndef ARA_RED_UNROLL
#define ARA_RED_UNROLL 4
#endif
constexpr int kRedUnroll = ARA_RED_UNROLL;   // the run reduction's unroll
static_assert(kXCap % (32 * kU) == 0 && kXCap >= ARA_MAX_SLOTS, "segment must hold one occurrence");

__device__ __forceinline__ uint64_t splitmix64_(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// Philox4x32-10 lane 0 with the seed's key schedule precomputed (ks[2r],
// ks[2r+1] = round r's keys): the XORs take the keys from the constant bank
__device__ __forceinline__ uint32_t philox_lane0_k(uint32_t i, uint32_t k, uint32_t id, uint32_t tag,
                                                   const uint32_t (&ks)[20]) {
    uint4 c = make_uint4(i, k, id, tag);
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ ks[2 * r], lo1, hi0 ^ c.w ^ ks[2 * r + 1], lo0);
    }
    return c.x;
}

// min(max(d, 0), lim) for finite or +inf d, lim (G5) by comparisons and
// selects: fmin/fmax would add NaN handling to the sampler's run loop
__device__ __forceinline__ double xl_clip_(double d, double lim) {
    return d > 0.0 ? (d < lim ? d : lim) : 0.0;
}
template <class T>
__device__ __forceinline__ T xl_clip_t_(T d, T lim) {
    return d > (T)0 ? (d < lim ? d : lim) : (T)0;
}
// p ? a : 0 in one SEL the optimiser keeps on the fp32 value (written plainly,
// the select is moved past the widening conversion and doubled)
__device__ __forceinline__ float sel_f32_(bool p, float a) {
    float r;
    asm("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n selp.f32 %0, %1, 0f00000000, q;\n}" : "=f"(r) : "f"(a), "r"((uint32_t)p));
    return r;
}
__device__ __forceinline__ double warp_sum_f64_(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace

// ---------------------------------------------------------------------------
// compact_kernel: one warp per trial (dynamic scheduler), persistent, one CTA
// per SM (the bitmap, <= 128 KiB, in shared memory).  A launch covers the
// work items of one batch of trials (item i = trial t0 + i) or of a list
// (item i = trial list[i]: the overflow pass).  The warp walks the flat
// sequence of 128-event chunks of its items as a register pipeline:
//   fetch   : one uint4 per lane (evict-first), two chunks in flight
//   stage A : presence bitmap (branch-free) and, for the hits, the event's
//             index entry (first device record, record count) from L2: loads
//             issued
//   stage B : one chunk later, so the entry loads overlap stage A of the next
//             chunk: the present pairs {device record, k} written in
//             (occurrence, slot) order to the item's region (an event's
//             records are consecutive, event-major in slot order, so its
//             pairs are first .. first + count - 1)
// Batch items: region i of the batch's slot, cap pairs; counts[t] = pairs of
// trial t, or kOverflow -- then (t, exact count) is appended to the overflow
// list and the overflow pass compacts t again into an exactly sized region
// of the overflow pool, for the same sampler.
// ---------------------------------------------------------------------------
struct RawChunk {
    uint4 v;                        // this lane's 4 event ids
    uint32_t t, c, len;             // item (kNoItem: none), chunk, trial length
};

// stage A output of one chunk: the index entries of this lane's 4 events (0 if
// absent).  IX4: packed 4-byte entries first | count << 24 (cidx4: half the
// gathered bytes and fewer L1 data-pipe wavefronts); else (first, count)
template <bool IX4>
struct ChunkA;
template <>
struct ChunkA<false> {
    uint2 ci[4];
    uint32_t t, c, len;
    __device__ __forceinline__ uint32_t first(int q) const { return ci[q].x; }
    __device__ __forceinline__ uint32_t cnt(int q) const { return ci[q].y; }
};
template <>
struct ChunkA<true> {
    uint32_t ci[4];
    uint32_t t, c, len;
    __device__ __forceinline__ uint32_t first(int q) const { return ci[q] & 0xffffffu; }
    __device__ __forceinline__ uint32_t cnt(int q) const { return ci[q] >> 24; }
};
constexpr uint32_t kNoItem = 0xffffffffu;

// predicated 4-byte store to a global address (no branch)
__device__ __forceinline__ void st_u32_if(bool p, uint64_t addr, uint32_t a) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.global.u32 [%1], %2;\n}" ::"r"((uint32_t)p),
                 "l"(addr), "r"(a)
                 : "memory");
}

// predicated 8-byte store {a, b} to a global address (no branch)
__device__ __forceinline__ void st_pair_if(bool p, uint64_t addr, uint32_t a, uint32_t b) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %0, 0;\n @q st.global.v2.u32 [%1], {%2, %3};\n}" ::"r"((uint32_t)p),
                 "l"(addr), "r"(a), "r"(b)
                 : "memory");
}

// trial of work item i
__device__ __forceinline__ uint32_t item_trial(const SplitArgs &A, uint32_t i) {
    return A.list ? __ldg(A.list + i) : A.t0 + i;
}

// The compaction pipeline of one warp over the items it claims from the
// launch's scheduler.  Sink: begin(i) -> the region of item i's pairs
// (warp-uniform), end(i, n) after its last chunk (n > cap: overflow).
// BM: 0 = bitmap shift 0 and a sentinel event (lanes past a trial's end hold
// an id whose presence bit is 0, so no length test per event), 1 = any shift
// with the sentinel, 2 = any shift, length test per event.
// VEC: fixed-length trials with K % 4 == 0 (every chunk 16-B aligned): one
// uint4 per lane from a per-item pointer, no per-id length tests.
template <bool PK, int BM, bool VEC, bool IX4, class Sink>
__device__ __forceinline__ void produce_pairs(const SplitArgs &A, const uint32_t *bitmap, Sink &sink) {
    using CA = ChunkA<IX4>;
    const int lane = threadIdx.x & 31;
    const uint32_t shift = A.pf.bitmap_shift, cap = A.cap;
    const uint32_t n_items = A.n_items_dev ? *A.n_items_dev : A.n_items;
    const uint32_t *events = A.yet.events;
    const uint64_t *offsets = A.yet.offsets;
    const uint2 *__restrict__ cidx = A.pf.cidx;
    const uint32_t *__restrict__ cidx4 = A.pf.cidx4;
    const uint32_t K = A.yet.fixed_len;
    const uint32_t mul = 1u << A.kbits;
    const uint32_t sent = BM == 2 ? 0u : A.pf.sentinel_event;

    // fetch side: the item being fetched and the chunk within it (warp-uniform)
    uint32_t pt = kNoItem;
    uint32_t pc = 0, plen = 0;                        // (plen = 0 when there is no item)
    uint64_t pbase = 0;
    const uint4 *psrc = nullptr;                      // VEC: this lane's uint4 of the item's chunk 0
    // items are claimed one ahead (lane 0's atomic for the next item in flight
    // while this one streams); a claimed item is always the claiming warp's next
    uint32_t claim = 0;
    if (lane == 0) claim = (uint32_t)atomicAdd(A.sched, 1ull);
    auto next_item = [&]() {                          // start the claimed item, claim the next
        const uint32_t i = __shfl_sync(0xffffffffu, claim, 0);
        if (lane == 0 && i < n_items) claim = (uint32_t)atomicAdd(A.sched, 1ull);
        pt = i < n_items ? i : kNoItem;
        pc = 0;
        plen = 0;
        if (pt != kNoItem) {
            const uint32_t t = item_trial(A, pt);
            if (VEC) { pbase = (uint64_t)t * K; plen = K; }
            else if (offsets) { pbase = offsets[t]; plen = (uint32_t)(offsets[t + 1] - pbase); }
            else { pbase = (uint64_t)t * K; plen = K; }
            if (VEC) psrc = reinterpret_cast<const uint4 *>(events + pbase) + lane;
        }
    };
    auto fetch = [&](RawChunk &r) {
        r.t = pt; r.c = pc; r.len = plen;
        r.v = make_uint4(sent, sent, sent, sent);
        const uint32_t k = pc * 128u + 4u * lane;
        if (VEC) {
            if (k < plen) r.v = __ldcs(psrc + pc * 32u);
        } else if (pt != kNoItem) {
            const uint32_t *src = events + pbase + k;
            if (k < plen) r.v.x = __ldcs(src);
            if (k + 1 < plen) r.v.y = __ldcs(src + 1);
            if (k + 2 < plen) r.v.z = __ldcs(src + 2);
            if (k + 3 < plen) r.v.w = __ldcs(src + 3);
        }
        if (pt != kNoItem) {
            if ((pc + 1) * 128u >= plen) next_item();
            else ++pc;
        }
    };
    auto stage_a = [&](const RawChunk &r, CA &S) {
        S.t = r.t; S.c = r.c; S.len = r.len;
        const uint32_t k0 = r.c * 128u + 4u * lane;
        const uint32_t ee[4] = {r.v.x, r.v.y, r.v.z, r.v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t bit = BM == 0 ? ee[q] : ee[q] >> shift;
            const uint32_t w = bitmap[bit >> 5];
            bool hit = __funnelshift_r(w, 0u, bit) & 1u;      // w >> (bit & 31)
            if (BM == 2) hit = hit && k0 + q < r.len;
            ARA_CHECK(!hit || ee[q] < A.pf.catalog);
            if constexpr (IX4) {
                S.ci[q] = 0u;
                asm volatile(                             // predicated load through L2, no branch
                    "{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n @p ld.global.cg.u32 %0, [%2];\n}"
                    : "+r"(S.ci[q])
                    : "r"((uint32_t)hit), "l"(cidx4 + ee[q]));
            } else {
                S.ci[q] = make_uint2(0u, 0u);
                asm volatile(
                    "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p ld.global.cg.v2.u32 {%0, %1}, [%3];\n}"
                    : "+r"(S.ci[q].x), "+r"(S.ci[q].y)
                    : "r"((uint32_t)hit), "l"(cidx + ee[q]));
            }
        }
    };
    // stage B: pairs out.  One warp prefix sum of the pair counts; a present
    // event has one pair in ~87 % of cases (cfg3), so the first pairs are
    // predicated stores and the rest one warp-uniform loop over the extra
    // pairs (usually one pass).
    uint32_t n = 0;                                   // pairs of the current item (warp-uniform)
    uint2 *out = nullptr;                             // the current item's pair region
    auto stage_b = [&](const CA &S) {
        if (S.c == 0) n = 0;
        const uint32_t k0 = S.c * 128u + 4u * lane;
        const uint32_t np = S.cnt(0) + S.cnt(1) + S.cnt(2) + S.cnt(3);
        // exclusive warp prefix of np, bit-sliced over ballots (votes, no
        // shuffles through the shared-memory pipe): 3 slices unless some
        // lane has >= 8 pairs in the chunk; np <= 4 * ARA_MAX_SLOTS = 896
        // < 2^10, so 10 slices cover every case
        static_assert(4 * ARA_MAX_SLOTS < (1 << 10), "pair count of a lane's 4 events must fit 10 bits");
        uint32_t excl = 0;
        const uint32_t tot = __reduce_add_sync(0xffffffffu, np);   // the chunk's pairs (one REDUX)
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const uint32_t m = __ballot_sync(0xffffffffu, (np >> b) & 1u);
            excl += (uint32_t)__popc(m & lt) << b;
        }
        if (__any_sync(0xffffffffu, np > 7u)) {
#pragma unroll 1
            for (int b = 3; b < 10; ++b) {
                const uint32_t m = __ballot_sync(0xffffffffu, (np >> b) & 1u);
                excl += (uint32_t)__popc(m & lt) << b;
            }
        }
        if (S.c == 0) out = sink.begin(S.t);
        uint32_t pos = n + excl;
        if (n + tot <= cap) {                         // the chunk fits (warp-uniform)
            ARA_CHECK(pos + np <= cap);
            // one 64-bit address per event, predicated stores (no branches)
            uint32_t pq[4], mx = 0, o = pos;
            if (PK) {                                 // pair = record * 2^kbits + k (one IMAD)
                uint32_t *const out32 = reinterpret_cast<uint32_t *>(out);
                uint32_t pv[4];
                // the first two pairs of each event in this pass (a chunk of
                // cfg3 almost always holds an event with two records), the
                // rest in a warp-uniform loop (a third pair: ~1/3 of chunks)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    pq[q] = o;
                    pv[q] = S.first(q) * mul + (k0 + q);
                    st_u32_if(S.cnt(q) != 0u, reinterpret_cast<uint64_t>(out32 + o), pv[q]);
                    st_u32_if(S.cnt(q) > 1u, reinterpret_cast<uint64_t>(out32 + o + 1), pv[q] + mul);
                    o += S.cnt(q);
                    mx = max(mx, S.cnt(q));
                }
#pragma unroll 1
                for (uint32_t j = 2; __any_sync(0xffffffffu, j < mx); ++j)   // events with three or more pairs
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        st_u32_if(j < S.cnt(q), reinterpret_cast<uint64_t>(out32 + (pq[q] + j)), pv[q] + j * mul);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    pq[q] = o;
                    st_pair_if(S.cnt(q) != 0u, reinterpret_cast<uint64_t>(out + o), S.first(q), k0 + q);
                    o += S.cnt(q);
                    mx = max(mx, S.cnt(q));
                }
#pragma unroll 1
                for (uint32_t j = 1; __any_sync(0xffffffffu, j < mx); ++j)
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        st_pair_if(j < S.cnt(q), reinterpret_cast<uint64_t>(out + (pq[q] + j)), S.first(q) + j, k0 + q);
            }
        }
        // (a chunk that does not fit: nothing is stored, the count goes on --
        // the overflow pass compacts the trial again into an exact region)
        n += tot;
        if ((S.c + 1) * 128u >= S.len) sink.end(S.t, n);           // last chunk of the item
    };

    // ping-pong: while chunk X is in stage B, chunk X+1 is in stage A and
    // chunks X+2, X+3 are in flight from HBM
    next_item();
    RawChunk ra, rb;
    CA ca, cb;
    fetch(ra);
    fetch(rb);
    stage_a(ra, ca);
    fetch(ra);
    while (ca.t != kNoItem) {
        stage_a(rb, cb);
        fetch(rb);
        stage_b(ca);
        if (cb.t == kNoItem) break;
        stage_a(ra, ca);
        fetch(ra);
        stage_b(cb);
    }
}

// batch items: region i of the batch's slot; counts[t] = pairs or kOverflow,
// an overflowing trial listed with its exact pair count
struct SlotSink {
    const SplitArgs &A;
    __device__ uint2 *begin(uint32_t i) const {     // (packed pairs: 4-byte regions)
        return A.kbits ? reinterpret_cast<uint2 *>(reinterpret_cast<uint32_t *>(A.pairs) + (uint64_t)i * A.cap)
                       : A.pairs + (uint64_t)i * A.cap;
    }
    __device__ void end(uint32_t i, uint32_t n) const {
        if ((threadIdx.x & 31) == 0) {
            const uint32_t t = A.t0 + i;
            A.counts[t] = n <= A.cap ? n : kOverflow;
            if (n > A.cap) {
                const uint32_t j = atomicAdd(&A.status->n_ovf, 1u);
                A.ovf[j] = t;
                A.ovf_n[j] = n;
            }
        }
    }
};

// overflow items: region at pool_off[i] (pair units), sized exactly
struct PoolSink {
    const SplitArgs &A;
    __device__ uint2 *begin(uint32_t i) const {
        const uint64_t off = __ldg(A.pool_off + i);
        return A.kbits ? reinterpret_cast<uint2 *>(reinterpret_cast<uint32_t *>(A.pairs) + off) : A.pairs + off;
    }
    __device__ void end(uint32_t, uint32_t) const {}
};

template <bool PK, int BM, bool VEC, bool IX4>
__global__ void __launch_bounds__(kCompactThreads, 32 / ARA_COMPACT_WARPS) compact_kernel(const __grid_constant__ SplitArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem);
    if (A.n_items_dev && *A.n_items_dev == 0) return; // a device-sized pass with nothing to do
    if (*A.yet.max_event >= A.pf.catalog) {           // out-of-range ids: nothing is read
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&A.status->bad_event, 1u);
        return;
    }
    load_bitmap_smem(smem, A.pf.bitmap, A.pf.bitmap_words);      // (+ one zero word: the sentinel's bit)
    if (A.list) {
        PoolSink sink{A};
        produce_pairs<PK, BM, VEC, IX4>(A, bitmap, sink);
    } else {
        SlotSink sink{A};
        produce_pairs<PK, BM, VEC, IX4>(A, bitmap, sink);
    }
}

// ---------------------------------------------------------------------------
// sample_kernel: one warp per trial (dynamic scheduler).  The trial's present
// pairs {device record, k} (dense, (occurrence, slot) order, from
// compact_kernel) are processed in rounds of 32 kU pairs, pair p of the
// round on lane p mod 32 (the next round's pairs prefetched):
//   draw   : one SplitRec load, Philox draws keyed (trial, k, program /
//            XELT), steps 2-4, quantile table (line 7), XELT terms (line 8)
//   runs   : the pairs of one (occurrence, layer) run are consecutive, so
//            each 32-pair group is reduced in registers by a segmented warp
//            scan (fp32, reading G28; the run boundaries from one ballot of
//            the records' run-end flags), the open run carried into the next
//            group (line 9); the lane holding a run's last pair applies the
//            occurrence terms (line 11) and adds the result to its fp64 share
//            of the layer's trial sum
// At the trial's end one fixed-tree warp sum per layer -> aggregate terms
// (line 12) -> YLT (line 17).  Every sum runs in an order fixed by the pair
// positions alone, so the YLT is a pure function of (portfolio, YET, seed).
// ---------------------------------------------------------------------------
// Per-warp shared-memory workspace of the sampler.
struct SampleWs {
    const SlotInfo *slots;
    const LayerInfo *layers;
    double *accs;                 // multi-layer: this lane's column of [nl][32]
    unsigned int *dc;             // [nl]
    unsigned long long *dhs;      // [nl]
    float *mos;                   // OM, multi-layer: this lane's column of [nl][32] (largest occurrence loss)
    uint32_t *xs;                 // [xcap] loss bits | run end << 31
    uint8_t *fl;                  // [xcap] layer (multi-layer portfolios)
};

// The sampler on trial t's n present pairs at `in` (CG: read them through L2 only).
using RunT = float;                            // in-stretch run sums and occurrence clips (G28)
template <bool SU, bool SL, bool DBG, bool CG, bool PK = false, bool OM = false, int RS = 0>
__device__ __forceinline__ void sample_trial(const SplitArgs &A, const SampleWs &W, uint64_t t, uint32_t n,
                                             const uint2 *in) {
    const int lane = threadIdx.x & 31;
    const uint32_t nl = A.pf.n_layers;
    const uint64_t n_trials = A.yet.n_trials;
    const bool terms = A.pf.any_terms != 0;
    const SlotInfo *slots = W.slots;
    const LayerInfo *layers = W.layers;
    uint32_t *xs = W.xs;
    uint8_t *fl = W.fl;
    double *accs = W.accs;
    unsigned int *dc = W.dc;
    unsigned long long *dhs = W.dhs;
    const SplitRec *__restrict__ srecs = A.pf.srecs;
    const TablePtr tables = A.pf.tables;
    auto ldpair = [&](const uint2 *q) -> uint2 {    // {device record, k}
        if (PK) {                                     // packed: record << kbits | k (operands from the
            const uint32_t w = __ldcs(reinterpret_cast<const uint32_t *>(in) + (q - in));   // constant bank)
            return make_uint2(w >> A.kbits, w & A.kmask);
        }
        return CG ? __ldcg(q) : __ldcs(q);
    };
    const uint32_t trial_g = (uint32_t)(A.yet.first_trial + t);
    // RS 2: index of the trial's first occurrence in the YET (supplied z_(Prog,E))
    const uint64_t occ_base = RS != 2 ? 0 : A.yet.offsets ? A.yet.offsets[t] : t * (uint64_t)A.yet.fixed_len;
    if (!SL)
        for (uint32_t l = 0; l < nl; ++l) accs[l * 32] = 0.0;
    if (OM && !SL)
        for (uint32_t l = 0; l < nl; ++l) W.mos[l * 32] = 0.0f;
    float mo = 0.0f;                               // OM, SL: this lane's largest occurrence loss
    if (DBG)
        for (uint32_t l = lane; l < nl; l += 32) { dc[l] = 0u; dhs[l] = 0ull; }
    double acc = 0.0;                              // SL: this lane's share of the trial sum
    double carry = 0.0;                            // run open at the previous segment's end
    uint32_t modes = 0;                            // OR of the live pairs' meta: bit 28 = a table-less record
                                                   // (mode exact: the trial is redone in fp64)
    uint2 pn[kU];                                   // next round's pairs, prefetched
#pragma unroll
    for (int u = 0; u < kU; ++u) pn[u] = 32u * u + lane < n ? ldpair(in + 32u * u + lane) : make_uint2(0u, 0u);
    for (uint32_t off = 0; off < n; off += kXCap) {
        const uint32_t ns = min(n - off, kXCap);
        // ---- rounds: x and run flags of every pair of the segment; U = 2
        // pairs per lane, or 1 for a last round of <= 32 pairs
        auto round = [&](auto UC, uint32_t b) {
            constexpr int U = decltype(UC)::value;
            uint2 e[kU];
            bool live[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                e[u] = pn[u];
                live[u] = b + 32u * u + lane < ns;
                const uint32_t q = off + b + 32u * kU + 32u * u + lane;
                pn[u] = q < n ? ldpair(in + q) : make_uint2(0u, 0u);
            }
            uint32_t meta[kU];
            float x[kU];
            if (SU) {
                SplitRec r[kU];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    r[u] = srecs[e[u].x];                 // (idle lanes: record 0, result unused)
                    meta[u] = r[u].meta;
                }
                float v[kU];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint2 key = make_uint2(r[u].key & 0xffffffu, r[u].key >> 24);   // draw keys (XELT, program)
                    if (RS == 2) {                        // supplied with the inputs
                        const float zp = __ldg(A.zp_sup + (uint64_t)key.y * A.zp_stride + occ_base + e[u].y);
                        const float ze = __ldg(A.ze_sup + e[u].x);
                        v[u] = fmaf(r[u].wi, norm_quantile_f(zp), r[u].wc * norm_quantile_f(ze));
                    } else {
                        const uint32_t bp = philox_lane0_k(trial_g, e[u].y, key.y, 1u, A.pkey);       // z_(Prog,E)
                        const uint32_t be =                                                           // z_(E)
                            RS == 1 ? philox_lane0_k(__ldg(A.pf.rec_orig + e[u].x), key.x, 0u, 6u, A.pkey)  // (A)
                                    : philox_lane0_k(trial_g, e[u].y, key.x & A.ze_mask, A.ze_tag, A.pkey); // G2, (B)
                        v[u] = fmaf(r[u].wi, norm_quantile_from_bits(bp), r[u].wc * norm_quantile_from_bits(be));
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    // every record has a table: degenerate records (G10) a constant
                    // one whose value is exactly scale (prep_records_kernel); a
                    // table-less record (mode exact) reads zeros and its trial is
                    // redone in fp64 -- no branch per sample
                    const float uu = (fminf(fmaxf(v[u], kTabV0), -kTabV0) - kTabV0) * (1.0f / kTabH);
                    const int ti = min((int)uu, kTabNodes - 2);
                    const float tt = uu - (float)ti;
                    ARA_CHECK(!(live[u]) || (e[u].x < A.pf.n_dev_records && r[u].tab < A.pf.n_tables &&
                                             ti >= 0 && ti <= kTabNodes - 2));
                    const float2 *row = table_row(tables, r[u].tab, ti);
                    x[u] = r[u].scale * sigmoidf_(quintic_from_nodes(__ldg(row), __ldg(row + 1), ti, tt,
                                                                     r[u].a, r[u].b));
                    modes |= live[u] ? meta[u] : 0u;             // (a select and an OR: no predicated test)
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint2 mm = live[u] ? __ldg(A.pf.mu_meta + e[u].x) : make_uint2(0u, 0u);
                    meta[u] = mm.y;                   // primary uncertainty: the mean loss (one 8 B gather)
                    x[u] = __uint_as_float(mm.x);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t layer = (meta[u] >> 16) & 63u;
                if (terms) {                                          // line 8 (G7)
                    const SlotInfo &si = slots[meta[u] & 0xffu];
                    if (si.has_terms) x[u] = si.share * fminf(fmaxf(x[u] - si.ret, 0.0f), si.lim);
                }
                if (DBG && live[u]) {
                    atomicAdd(&dc[layer], 1u);
                    const uint64_t hv = splitmix64_(splitmix64_(splitmix64_((uint64_t)e[u].y) ^
                                                                slots[meta[u] & 0xffu].elt) ^
                                                    A.pf.rec_orig[e[u].x]);
                    atomicAdd(&dhs[layer], (unsigned long long)hv);
                }
                if (live[u]) {                                // (losses are >= 0)
                    const uint32_t p = b + 32u * u + lane;
                    ARA_CHECK(p < kXCap);
                    xs[p] = __float_as_uint(x[u]) | ((meta[u] & 0x100u) << 23);   // (x >= +0: bit 31 free)
                    if (!SL) fl[p] = (uint8_t)layer;
                }
            }
        };
        for (uint32_t b = 0; b < ns; b += 32u * kU) {
            if (kU >= 3 && ns - b > 64u) round(std::integral_constant<int, kU>{}, b);
            else if (ns - b > 32u) round(std::integral_constant<int, 2>{}, b);
            else round(std::integral_constant<int, 1>{}, b);
        }
        __syncwarp();
        // ---- reduce: runs (line 9) and occurrence terms (line 11)
        // (an odd stretch length keeps the lanes' reads on distinct banks)
#ifndef ARA_ODD_STRETCH
#define ARA_ODD_STRETCH 1
#endif
        const uint32_t per = ((ns + 31) / 32) | (ARA_ODD_STRETCH ? 1u : 0u), i0 = min(lane * per, ns),
                       i1 = min(i0 + per, ns);
        RunT o = 0, head = 0;                          // (RunT: the in-stretch run sums)
        bool has_end = false;
        uint32_t head_layer = 0;
        const RunT occ_r0 = (RunT)layers[0].occ_r, occ_l0 = (RunT)layers[0].occ_l;
#pragma unroll kRedUnroll
        for (uint32_t i = i0; i < i1; ++i) {           // branch-free
            const uint32_t q = xs[i];                  // loss bits | run end << 31
            o += (RunT)__uint_as_float(q & 0x7fffffffu);
            const bool end = (q >> 31) != 0u;
            const uint32_t lay = SL ? 0u : (uint32_t)fl[i];
            const RunT orr = SL ? occ_r0 : (RunT)layers[lay].occ_r, oll = SL ? occ_l0 : (RunT)layers[lay].occ_l;
            const RunT gr = xl_clip_t_(o - orr, oll);   // (fp32: the run's clip, G28)
            const bool first = end && !has_end, inner = end && has_end;
            head = first ? o : head;
            head_layer = first ? lay : head_layer;
            // (the select on the fp32 value, then one widening add: acc + 0.0 = acc)
            if (SL) acc += (double)sel_f32_(inner, gr);
            else if (inner) accs[lay * 32] += (double)gr;
            if (OM) {                                  // OEP basis (G29); fp32 rounding is monotone
                if (SL) mo = fmaxf(mo, inner ? (float)gr : 0.0f);
                else if (inner) W.mos[lay * 32] = fmaxf(W.mos[lay * 32], (float)gr);
            }
            has_end = has_end || end;
            o = end ? (RunT)0 : o;
        }
        // join the runs that cross stretches: exclusive segmented sum over
        // lanes of the open tails (a lane with a run end starts a segment)
        double v = o;                              // this lane's contribution to the run it leaves open
        bool seg = has_end;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, v, d);
            const bool ys = __shfl_up_sync(0xffffffffu, seg, d);
            if (lane >= d && !seg) v += y;
            if (lane >= d) seg = seg || ys;
        }
        // v = inclusive segmented sum; the run entering lane l is lane l-1's v (+ carry)
        double in_run = __shfl_up_sync(0xffffffffu, v, 1);
        const bool prev_seg = __shfl_up_sync(0xffffffffu, seg, 1);
        if (lane == 0) in_run = 0.0;
        if (lane == 0 || !prev_seg) in_run += carry;   // no run end before me in this segment
        if (has_end) {
            const LayerInfo &L = layers[head_layer];
            const double g = xl_clip_(head + in_run - L.occ_r, L.occ_l);
            if (SL) acc += g; else accs[head_layer * 32] += g;
            if (OM) {
                if (SL) mo = fmaxf(mo, (float)g);
                else W.mos[head_layer * 32] = fmaxf(W.mos[head_layer * 32], (float)g);
            }
        }
        // run left open at the segment's end (continues in the next segment)
        const double last = has_end ? o : o + in_run;
        carry = __shfl_sync(0xffffffffu, last, 31);
        __syncwarp();
    }
    static_assert(kModeExact == 1u, "the table-less flag is meta bit 28");
    const bool redo = __any_sync(0xffffffffu, (modes >> 28) & 1u);
    if (redo) {
        if (lane == 0) A.redo[atomicAdd(&A.status->n_redo, 1u)] = (uint32_t)t;
        return;
    }
    // aggregate terms (line 12, G6) -> YLT (line 17)
    for (uint32_t l = 0; l < nl; ++l) {
        const double S = warp_sum_f64_(SL ? acc : accs[l * 32]);   // fixed tree
        if (lane == 0) {
            const LayerInfo &L = layers[l];
            A.ylt[(uint64_t)l * n_trials + t] = (float)xl_clip_(S - L.agg_r, L.agg_l);   // line 12 (G5, G6)
            if (DBG) {
                if (A.dbg_count) A.dbg_count[(uint64_t)l * n_trials + t] = dc[l];
                if (A.dbg_hash) A.dbg_hash[(uint64_t)l * n_trials + t] = dhs[l];
            }
        }
        if (OM) {
            const unsigned mb = __reduce_max_sync(0xffffffffu, __float_as_uint(SL ? mo : W.mos[l * 32]));
            if (lane == 0) A.occ_max[(uint64_t)l * n_trials + t] = __uint_as_float(mb);
        }
    }
}


// RS: the random source -- 0: Philox, reading G2 and ARA_RNG_OCCURRENCE
// (through A.ze_mask / A.ze_tag); 1: Philox z_(E) per XELT record
// (ARA_RNG_RECORD); 2: z_(Prog,E) / z_(E) supplied with the YET and the
// records (ARA_RNG_SUPPLIED, the paper's data model).  A.list set: the items
// of the overflow pass (pairs in the overflow pool).
template <bool SU, bool SL, bool DBG, bool PK, bool OM, int RS = 0>
__global__ void __launch_bounds__(kSampleWarps * 32, 32 / kSampleWarps)   // <= 64 registers
    sample_kernel(const __grid_constant__ SplitArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t nl = A.pf.n_layers;
    // carved by byte offsets from the shared base (no integer round trip), so
    // every pointer below stays in the shared address space (LDS / STS)
    size_t o = 0;
    SlotInfo *slots = reinterpret_cast<SlotInfo *>(smem);
    o += ARA_MAX_SLOTS * sizeof(SlotInfo);
    LayerInfo *layers = reinterpret_cast<LayerInfo *>(smem + o);
    o += ARA_MAX_LAYERS * sizeof(LayerInfo);
    double *accw = reinterpret_cast<double *>(smem + o);                        // [warps][nl][32]
    o += kSampleWarps * nl * 32 * sizeof(double);
    unsigned int *cw = reinterpret_cast<unsigned int *>(smem + o);              // [warps][nl]
    o += (kSampleWarps * nl * sizeof(unsigned int) + 7) & ~(size_t)7;
    unsigned long long *hw = reinterpret_cast<unsigned long long *>(smem + o);  // [warps][nl]
    o += kSampleWarps * nl * sizeof(unsigned long long);
    float *mow = reinterpret_cast<float *>(smem + o);                           // OM && !SL: [warps][nl][32]
    if (A.n_items_dev && *A.n_items_dev == 0) return; // a device-sized pass with nothing to do
    for (uint32_t t = threadIdx.x; t < A.pf.n_slots; t += blockDim.x) slots[t] = A.pf.slots[t];
    for (uint32_t t = threadIdx.x; t < nl; t += blockDim.x) layers[t] = A.pf.layers[t];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (*A.yet.max_event >= A.pf.catalog) return;   // compact_kernel wrote no pairs
    uint32_t *xsw = reinterpret_cast<uint32_t *>(mow + ((OM && !SL) ? kSampleWarps * nl * 32 : 0));
    uint8_t *flw = reinterpret_cast<uint8_t *>(xsw + kSampleWarps * kXCap);
    const SampleWs W{slots, layers, accw + warp * nl * 32 + lane, cw + warp * nl, hw + warp * nl,
                     (OM && !SL) ? mow + warp * nl * 32 + lane : nullptr, xsw + warp * kXCap, flw + warp * kXCap};
    const uint32_t n_items = A.n_items_dev ? *A.n_items_dev : A.n_items;
    while (true) {
        unsigned long long i = 0;
        if (lane == 0) i = atomicAdd(A.sched, 1ull);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= n_items) break;
        uint32_t t, n;
        uint64_t off;                                 // the item's pairs: offset in pair units
        if (A.list) {
            t = __ldg(A.list + i);
            n = __ldg(A.ovf_n + i);
            off = __ldg(A.pool_off + i);
        } else {
            t = A.t0 + (uint32_t)i;
            n = __ldg(A.counts + t);
            if (n == kOverflow) continue;             // sampled in the overflow pass
            off = i * (uint64_t)A.cap;
        }
        sample_trial<SU, SL, DBG, false, PK, OM, RS>(A, W, t, n, PK ? reinterpret_cast<const uint2 *>(
                                                                reinterpret_cast<const uint32_t *>(A.pairs) + off)
                                                            : A.pairs + off);
        __syncwarp();
    }
}

__global__ void split_recs_kernel(const BetaRec *__restrict__ recs, const uint32_t *__restrict__ rec_src,
                                  const uint32_t *__restrict__ rec_meta, const SlotInfo *__restrict__ slots,
                                  const float *__restrict__ mu, uint64_t n, SplitRec *__restrict__ out,
                                  uint2 *__restrict__ mu_meta) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t src = rec_src[t];
        const BetaRec r = recs[src];
        const uint32_t m = rec_meta[t];
        const SlotInfo &s = slots[m & 0xffu];
        out[t] = SplitRec{r.a, r.b, r.wi, r.wc, r.scale, m | (r.mode << 28), src, s.elt | (s.prog << 24)};
        mu_meta[t] = make_uint2(__float_as_uint(mu[src]), m);
    }
}

void launch_split_recs(const BetaRec *recs, const uint32_t *rec_src, const uint32_t *rec_meta,
                       const SlotInfo *slots, const float *mu, uint64_t n, SplitRec *out, uint2 *mu_meta,
                       cudaStream_t s) {
    if (n == 0) return;
    const uint64_t blocks = (n + 255) / 256;
    split_recs_kernel<<<(unsigned)(blocks < 65535u * 16u ? blocks : 65535u * 16u), 256, 0, s>>>(
        recs, rec_src, rec_meta, slots, mu, n, out, mu_meta);
}

// ARA_ASYNC overflow plan (one CTA): pool offsets of the listed trials in
// list order, an exclusive scan in chunks of 1024; the trials that do not fit
// the pre-sized pool are counted (reported at the next synchronisation)
__global__ void ovf_plan_kernel(RunStatus *status, const uint32_t *__restrict__ ovf_n, uint64_t *__restrict__ pool_off,
                                uint64_t pool_pairs) {
    __shared__ unsigned long long part[32];
    __shared__ unsigned long long base_s;
    __shared__ unsigned int fit_s;
    const uint32_t n = status->n_ovf;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) { base_s = 0; fit_s = n; }
    __syncthreads();
    for (uint32_t c0 = 0; c0 < n; c0 += blockDim.x) {
        const uint32_t i = c0 + threadIdx.x;
        const unsigned long long v = i < n ? ovf_n[i] : 0ull;
        unsigned long long x = v;                                  // inclusive warp scan
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) part[warp] = x;
        __syncthreads();
        if (warp == 0) {
            unsigned long long w = lane < (int)(blockDim.x >> 5) ? part[lane] : 0ull;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += y;
            }
            part[lane] = w;                                        // inclusive over warps
        }
        __syncthreads();
        const unsigned long long excl = base_s + (warp ? part[warp - 1] : 0ull) + x - v;
        if (i < n) {
            pool_off[i] = excl;
            if (excl + v > pool_pairs) atomicMin(&fit_s, i);        // the first trial that does not fit
        }
        __syncthreads();
        if (threadIdx.x == 0) base_s += part[(blockDim.x >> 5) - 1];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        status->n_ovf_fit = fit_s;
        status->pool_short += n - fit_s;
    }
}

cudaError_t launch_ovf_plan(RunStatus *status, const uint32_t *ovf_n, uint64_t *pool_off, uint64_t pool_pairs,
                            cudaStream_t s) {
    ovf_plan_kernel<<<1, 1024, 0, s>>>(status, ovf_n, pool_off, pool_pairs);
    return cudaGetLastError();
}

// Packed YET upload (ara_yet_refill_packed): ids bit-packed LSB-first, `bits`
// per id -> uint32 event ids.  Four ids per thread, one 16 B store; the
// packed words are read through L1 (each word serves ~32/bits ids).
__global__ void unpack_yet_kernel(const uint32_t *__restrict__ packed, uint64_t n, uint32_t bits,
                                  uint64_t words, uint32_t *__restrict__ out) {
    const uint32_t mask = bits == 32u ? 0xffffffffu : (1u << bits) - 1u;
    const uint64_t n4 = (n + 3) / 4;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n4; q += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t x = 4 * q + j, bit = x * (uint64_t)bits, w = bit >> 5;
            const uint32_t sh = (uint32_t)(bit & 31u);
            uint32_t lo = 0u, hi = 0u;
            if (x < n) {                                 // (no read past the packed words)
                lo = __ldg(packed + w);
                hi = w + 1 < words ? __ldg(packed + w + 1) : 0u;
            }
            v[j] = __funnelshift_r(lo, hi, sh) & mask;
        }
        reinterpret_cast<uint4 *>(out)[q] = make_uint4(v[0], v[1], v[2], v[3]);   // (+4 words of padding)
    }
}

cudaError_t launch_unpack_yet(const uint32_t *packed, uint64_t n, uint32_t bits, uint32_t *out, cudaStream_t s,
                              int num_sms) {
    if (n == 0) return cudaSuccess;
    const uint64_t words = (n * (uint64_t)bits + 31) / 32;
    unpack_yet_kernel<<<num_sms * 8, 256, 0, s>>>(packed, n, bits, words, out);
    return cudaGetLastError();
}

// largest event id of a YET (run after every upload): ara_run checks it
// against the catalog before any table is indexed
__global__ void yet_max_kernel(const uint32_t *__restrict__ ev, uint64_t n, uint32_t *out) {
    uint32_t m = 0;
    const uint64_t n4 = n / 4;
    const uint4 *v = reinterpret_cast<const uint4 *>(ev);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 q = __ldcs(v + i);
        m = max(m, max(max(q.x, q.y), max(q.z, q.w)));
    }
    for (uint64_t i = n4 * 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, ev[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void count_bad_kernel(const uint32_t *__restrict__ ev, uint64_t n, uint32_t C, unsigned int *out) {
    unsigned int c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        c += ev[i] >= C;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

cudaError_t launch_yet_max(const uint32_t *ev, uint64_t n, uint32_t *out, cudaStream_t s, int num_sms) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess || n == 0) return e;
    yet_max_kernel<<<num_sms * 4, 512, 0, s>>>(ev, n, out);
    return cudaGetLastError();
}

cudaError_t launch_count_bad(const uint32_t *ev, uint64_t n, uint32_t C, unsigned int *out, cudaStream_t s,
                             int num_sms) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess || n == 0) return e;
    count_bad_kernel<<<num_sms * 4, 512, 0, s>>>(ev, n, C, out);
    return cudaGetLastError();
}

// Launch preparation cached per (device, kernel, dynamic shared memory): the
// attribute call and the occupancy query cost microseconds of host time
// that would otherwise sit between the kernels of every ara_run.
cudaError_t prepare_launch(const void *kern, size_t smem, int threads, int &per_sm) {
    struct Entry { int dev; const void *k; size_t smem; int threads, per_sm; };
    struct Attr { int dev; const void *k; size_t max_smem; };
    static std::mutex mu;
    static std::vector<Entry> cache;
    static std::vector<Attr> attrs;                   // the largest size each kernel was opened for
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    std::lock_guard<std::mutex> lock(mu);
    for (const Entry &e : cache)
        if (e.dev == dev && e.k == kern && e.smem == smem && e.threads == threads) { per_sm = e.per_sm; return cudaSuccess; }
    Attr *a = nullptr;
    for (Attr &x : attrs)
        if (x.dev == dev && x.k == kern) a = &x;
    if (!a || a->max_smem < smem) {
        err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
        if (a) a->max_smem = smem; else attrs.push_back(Attr{dev, kern, smem});
    }
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (err != cudaSuccess) return err;
    cache.push_back(Entry{dev, kern, smem, threads, per_sm});
    return cudaSuccess;
}

static bool env_compact_ix4() {                 // (test aid: ARA_COMPACT_IX4=0 selects 8-byte entries)
    static const bool on = [] {
        const char *e = getenv("ARA_COMPACT_IX4");
        return !(e && *e == '0');
    }();
    return on;
}

cudaError_t launch_compact(const SplitArgs &A, cudaStream_t s, int num_sms) {
    const size_t smem = bitmap_smem_bytes(A.pf.bitmap_words);
    using K = void (*)(SplitArgs);
    const int bm = !A.pf.sentinel_ok ? 2 : A.pf.bitmap_shift == 0 ? 0 : 1;
    const bool vec = A.yet.offsets == nullptr && (A.yet.fixed_len & 3u) == 0;   // every chunk 16-B aligned
    // packed pairs of fixed-length trials read 4-byte index entries (< 2^24 device records)
    const bool ix4 = A.kbits && vec && A.pf.cidx4 && env_compact_ix4();
#define ARA_CK(PK_, V_, I_) (bm == 0 ? (K)compact_kernel<PK_, 0, V_, I_> : bm == 1 ? (K)compact_kernel<PK_, 1, V_, I_> \
                                                                             : (K)compact_kernel<PK_, 2, V_, I_>)
    const K kern = ix4 ? ARA_CK(true, true, true)
                 : A.kbits ? (vec ? ARA_CK(true, true, false) : ARA_CK(true, false, false))
                           : (vec ? ARA_CK(false, true, false) : ARA_CK(false, false, false));
#undef ARA_CK
    int per_sm = 0;
    cudaError_t err = prepare_launch((const void *)kern, smem, kCompactThreads, per_sm);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint32_t blocks = A.n_items_dev ? (uint32_t)num_sms
                                          : std::max(1u, std::min<uint32_t>((uint32_t)num_sms,
                                                                            (A.n_items + ARA_COMPACT_WARPS - 1) /
                                                                                ARA_COMPACT_WARPS));
    kern<<<blocks, kCompactThreads, smem, s>>>(A);      // one CTA per SM (persistent)
    return cudaGetLastError();
}

size_t sample_smem_bytes(uint32_t n_layers, bool occ_max) {
    // slot and layer tables plus the per-warp layer accumulators; the rest of
    // the SM's shared memory is the compaction's bitmap and L1 data cache for
    // the record and table gathers
    const bool sl = n_layers == 1;
    return sizeof(SlotInfo) * ARA_MAX_SLOTS + sizeof(LayerInfo) * ARA_MAX_LAYERS +
           sizeof(double) * kSampleWarps * n_layers * 32 +
           kSampleWarps * n_layers * (sizeof(unsigned int) + sizeof(unsigned long long)) + 16 +
           (occ_max && !sl ? sizeof(float) * kSampleWarps * n_layers * 32 : 0) +
           (sizeof(uint32_t) + sizeof(uint8_t)) * kSampleWarps * kXCap + 16;
}

cudaError_t launch_sample(const SplitArgs &A, cudaStream_t s, int num_sms) {
    const bool dbg = (A.flags & ARA_DEBUG_LOOKUP) != 0, su = (A.flags & ARA_SU) != 0;
    const bool sl = A.pf.n_layers == 1;
    if (A.pf.n_layers > kSplitMaxLayers) return cudaErrorInvalidValue;
    const size_t smem = sample_smem_bytes(A.pf.n_layers, A.occ_max != nullptr);
    using K = void (*)(SplitArgs);
#define ARA_SK(P, O)                                                                                            \
    (su ? (sl ? (dbg ? (K)sample_kernel<true, true, true, P, O> : (K)sample_kernel<true, true, false, P, O>)     \
            : (dbg ? (K)sample_kernel<true, false, true, P, O> : (K)sample_kernel<true, false, false, P, O>))   \
        : (sl ? (dbg ? (K)sample_kernel<false, true, true, P, O> : (K)sample_kernel<false, true, false, P, O>)   \
              : (dbg ? (K)sample_kernel<false, false, true, P, O> : (K)sample_kernel<false, false, false, P, O>)))
    // ARA_RNG_RECORD / ARA_RNG_SUPPLIED: their own instantiations (SU on, no occ_max: ara_run
    // sends those cases to the fp64-capable kernel)
#define ARA_SR(RS_)                                                                                                 \
    (A.kbits ? (sl ? (dbg ? (K)sample_kernel<true, true, true, true, false, RS_>                                   \
                          : (K)sample_kernel<true, true, false, true, false, RS_>)                                 \
                   : (dbg ? (K)sample_kernel<true, false, true, true, false, RS_>                                  \
                          : (K)sample_kernel<true, false, false, true, false, RS_>))                               \
             : (sl ? (dbg ? (K)sample_kernel<true, true, true, false, false, RS_>                                  \
                          : (K)sample_kernel<true, true, false, false, false, RS_>)                                \
                   : (dbg ? (K)sample_kernel<true, false, true, false, false, RS_>                                 \
                          : (K)sample_kernel<true, false, false, false, false, RS_>)))
    const uint32_t rs = su && (A.rng_mode == 1 || A.rng_mode == 3) ? (A.rng_mode == 1 ? 1u : 2u) : 0u;
    if (rs && A.occ_max) return cudaErrorInvalidValue;
    const K kern = rs == 1 ? ARA_SR(1) : rs == 2 ? ARA_SR(2)
                 : A.occ_max ? (A.kbits ? ARA_SK(true, true) : ARA_SK(false, true))
                             : (A.kbits ? ARA_SK(true, false) : ARA_SK(false, false));
#undef ARA_SR
#undef ARA_SK
    int per_sm = 0;
    cudaError_t err = prepare_launch((const void *)kern, smem, kSampleWarps * 32, per_sm);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint32_t blocks = A.n_items_dev ? (uint32_t)num_sms
                                          : std::max(1u, std::min<uint32_t>((uint32_t)num_sms,
                                                                            (A.n_items + kSampleWarps - 1) / kSampleWarps));
    kern<<<blocks, kSampleWarps * 32, smem, s>>>(A);    // one CTA per SM (persistent)
    return cudaGetLastError();
}

}  // namespace ara
