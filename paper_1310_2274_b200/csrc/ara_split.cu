// ara_split.cu -- the two-kernel form of the YET scan (Algorithm 1,
// P:134-170), the default path of ara_run:
//
//   compact_kernel : YET stream (line 4) + presence bitmap (first level of
//                    the direct-access lookup, line 6): per trial, the list
//                    of hits {event id, occurrence k} written to a
//                    fixed-capacity per-trial region of HBM.  Streams the
//                    YET at HBM speed with a few instructions per event.
//   sample_kernel  : per trial, the index entries of its hits (second level
//                    of line 6) expanded into present (occurrence, slot)
//                    pairs in a shared-memory ring, then dense 64-pair
//                    rounds: draws (line 7, section 3), XELT terms (line 8),
//                    a segmented warp scan for the per-occurrence sums
//                    (line 9), occurrence terms (line 11), fp64 trial sums,
//                    aggregate terms (line 12) -> YLT (line 17).  ALU-bound.
//
// A trial whose hits overflow the region, or that meets a table-less
// record, is listed for the fused fp64-capable kernel (ara_kernels.cu).
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"
#include "ara_sampler.cuh"

#ifndef ARA_SEG_EARLY_EXIT
#define ARA_SEG_EARLY_EXIT 0
#endif

namespace ara {

namespace {

constexpr int kCompactThreads = 1024;   // compaction: 1 CTA per SM (bitmap in shared memory)
#ifndef ARA_SAMPLE_WARPS
#define ARA_SAMPLE_WARPS 16
#endif
#ifndef ARA_SAMPLE_MINB
#define ARA_SAMPLE_MINB 2
#endif
constexpr int kSampleWarps = ARA_SAMPLE_WARPS;   // sampling: 2 CTAs of 512 threads per SM

__device__ __forceinline__ uint64_t splitmix64_(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double warp_sum_f64_(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace

// ---------------------------------------------------------------------------
// compact_kernel: YET stream (Alg.1 line 4) + the first level of the
// direct-access lookup (line 6): the presence bitmap.  One warp per trial
// (static interleave: trial = global warp + r * warps in the grid),
// persistent, one CTA per SM (the bitmap, <= 128 KiB, lives in shared
// memory).  The warp walks the flat sequence of 128-event chunks of its
// trials with two chunks in flight (one uint4 per lane, evict-first); per
// chunk a branch-free bitmap test of each lane's 4 events, one warp prefix
// sum of the hit counts, and the hits {event id, occurrence index k} written
// in occurrence order to the trial's region of HBM.
// counts[t] = hits of trial t, or kOverflow (then t is appended to redo).  A
// hit past the region is clamped onto its last entry: the region of an
// overflowing trial is never read.
// ---------------------------------------------------------------------------
struct RawChunk {
    uint4 v;                        // this lane's 4 event ids
    uint32_t t, c, len;             // trial (>= n_trials: none), chunk, trial length
};

__global__ void __launch_bounds__(kCompactThreads, 1) compact_kernel(const __grid_constant__ SplitArgs A) {
    constexpr int kWarps = kCompactThreads / 32;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem);
    const uint32_t C = A.pf.catalog, shift = A.pf.bitmap_shift, cap = A.cap;
    if (*A.yet.max_event >= C) {                      // out-of-range ids: nothing is read
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&A.status->bad_event, 1u);
        return;
    }
    for (uint32_t t = threadIdx.x; t < A.pf.bitmap_words; t += blockDim.x) bitmap[t] = A.pf.bitmap[t];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint32_t n_trials = (uint32_t)A.yet.n_trials;    // <= 2^32 - 1 (ara_load_yet)
    const uint32_t nw = gridDim.x * kWarps;
    const uint32_t *events = A.yet.events;
    const uint64_t *offsets = A.yet.offsets;
    const uint32_t K = A.yet.fixed_len;
    const bool vec = offsets == nullptr && (K & 3u) == 0;   // every chunk 16 B aligned

    // fetch side: position in the flat chunk sequence (warp-uniform)
    uint32_t pt = blockIdx.x * kWarps + (threadIdx.x >> 5);
    uint32_t pc = 0, plen = 0;
    uint64_t pbase = 0;
    auto set_trial = [&]() {
        if (pt < n_trials) {
            if (offsets) { pbase = offsets[pt]; plen = (uint32_t)(offsets[pt + 1] - pbase); }
            else { pbase = (uint64_t)pt * K; plen = K; }
        }
    };
    auto fetch = [&](RawChunk &r) {
        r.t = pt; r.c = pc; r.len = plen;
        r.v = make_uint4(0u, 0u, 0u, 0u);
        if (pt < n_trials) {
            const uint32_t k = pc * 128u + 4u * lane;
            const uint32_t *src = events + pbase + k;
            if (vec) {
                if (k < plen) r.v = __ldcs(reinterpret_cast<const uint4 *>(src));
            } else {
                if (k < plen) r.v.x = __ldcs(src);
                if (k + 1 < plen) r.v.y = __ldcs(src + 1);
                if (k + 2 < plen) r.v.z = __ldcs(src + 2);
                if (k + 3 < plen) r.v.w = __ldcs(src + 3);
            }
            if ((pc + 1) * 128u >= plen) { pt = pt + nw < pt ? n_trials : pt + nw; pc = 0; set_trial(); }
            else ++pc;
        }
    };

    uint32_t n = 0;                                   // hits of the current trial (warp-uniform)
    auto process = [&](const RawChunk &r) {
        if (r.c == 0) n = 0;
        const uint32_t k0 = r.c * 128u + 4u * lane;
        const uint32_t ee[4] = {r.v.x, r.v.y, r.v.z, r.v.w};
        bool hit[4];
        uint32_t hc = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t bit = ee[q] >> shift;
            const uint32_t w = bitmap[bit >> 5];
            hit[q] = k0 + q < r.len && ((w >> (bit & 31)) & 1u);
            hc += hit[q];
        }
        uint32_t incl = hc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint2 *out = A.hits + (uint64_t)r.t * cap;
        uint32_t pos = n + incl - hc;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            if (hit[q]) out[min(pos, cap - 1u)] = make_uint2(ee[q], k0 + q);
            pos += hit[q];
        }
        n += __shfl_sync(0xffffffffu, incl, 31);
        if ((r.c + 1) * 128u >= r.len && lane == 0) {           // last chunk of the trial
            A.counts[r.t] = n <= cap ? n : kOverflow;
            if (n > cap) A.redo[atomicAdd(&A.status->n_redo, 1u)] = r.t;
        }
    };

    set_trial();
    RawChunk ra, rb;                                  // ping-pong: one in use, one in flight
    fetch(ra);
    fetch(rb);
    while (ra.t < n_trials) {
        const RawChunk cur = ra;
        fetch(ra);
        process(cur);
        if (rb.t >= n_trials) break;
        const RawChunk cur2 = rb;
        fetch(rb);
        process(cur2);
    }
}

// ---------------------------------------------------------------------------
// sample_kernel: persistent warps; each warp runs 64 virtual lanes (two per
// thread, so two independent samples are in flight per thread) over a
// continuous queue of hits that spans its trials (claimed dynamically, at
// most two in flight per warp, so no lane idles at a trial boundary).  A
// virtual lane works through one hit at a time: the hit's present pairs are
// the consecutive device records [first, first + n) (event-major, slot
// order), one per round.  Lanes whose hit is done take the next hits, in
// order, from a 32-entry shared-memory batch refilled from the event index
// (second level of Alg.1 line 6), hits prefetched one batch ahead.
// Per pair: one SplitRec load, Philox draws keyed (trial, k, program / XELT),
// steps 2-4, quantile table (line 7), XELT terms (line 8), and the running
// fp64 occurrence sum of the (occurrence, layer) run in slot order (line 9);
// at the run's last record the occurrence terms (line 11) go into the lane's
// trial sum.  Trial sums are 64-bit fixed point (LayerInfo::fx_scale), so
// integer adds make them independent of which lane took which hit: the YLT
// is bit-identical across runs, launch shapes and shardings.  When a trial's
// hits are all handed out and no lane holds one, a warp sum gives the trial
// sum per layer -> aggregate terms (line 12) -> YLT (line 17).
// SL: single-layer portfolio (trial sums in registers); otherwise per-lane,
// per-layer sums in shared memory (n_layers <= kSplitMaxLayers).
// ---------------------------------------------------------------------------
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

__device__ __forceinline__ long long warp_sum_i64_(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// warp-uniform state of a warp's hit queue (shared memory, not registers)
struct WarpQueue {
    uint32_t nc, s0;          // trials claimed; oldest trial not retired (trial s -> parity s & 1)
    uint32_t tid[2];          // local trial index of each parity
    uint32_t rem[2];          // hits of that trial not yet handed out
    uint32_t fdone;           // no trials left to claim
    uint32_t fnh, fh;         // fetch trial (number nc - 1): hit count, next hit to batch
    uint32_t bn, bq, bpar;    // batch: size, handed out, parity
    uint64_t hoff;            // fetch trial's hit region
};

template <bool SU, bool SL, bool DBG>
__global__ void __launch_bounds__(kSampleWarps * 32, ARA_SAMPLE_MINB)   // 2 CTAs/SM: <= 64 registers
    sample_kernel(const __grid_constant__ SplitArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t nl = A.pf.n_layers;
    SlotInfo *slots = reinterpret_cast<SlotInfo *>(smem);
    LayerInfo *layers = reinterpret_cast<LayerInfo *>(slots + ARA_MAX_SLOTS);
    uint4 *hbufs = reinterpret_cast<uint4 *>(layers + ARA_MAX_LAYERS);           // [warps][32]
    WarpQueue *wqs = reinterpret_cast<WarpQueue *>(hbufs + kSampleWarps * 32);    // [warps]
    long long *accw = reinterpret_cast<long long *>(wqs + kSampleWarps);          // [warps][2][nl][32]
    unsigned int *cw = reinterpret_cast<unsigned int *>(accw + kSampleWarps * 2 * nl * 32);
    unsigned long long *hw = reinterpret_cast<unsigned long long *>(
        ((uintptr_t)(cw + kSampleWarps * 2 * nl) + 7) & ~(uintptr_t)7);        // [warps][2][nl]
    for (uint32_t t = threadIdx.x; t < A.pf.n_slots; t += blockDim.x) slots[t] = A.pf.slots[t];
    for (uint32_t t = threadIdx.x; t < nl; t += blockDim.x) layers[t] = A.pf.layers[t];
    for (uint32_t t = threadIdx.x; t < kSampleWarps * 2 * nl * 32; t += blockDim.x) accw[t] = 0;
    if (threadIdx.x < kSampleWarps) wqs[threadIdx.x] = WarpQueue{};
    if (DBG)
        for (uint32_t t = threadIdx.x; t < kSampleWarps * 2 * nl; t += blockDim.x) { cw[t] = 0u; hw[t] = 0ull; }
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (*A.yet.max_event >= A.pf.catalog) return;   // compact_kernel wrote no hits
    const uint32_t lt = (1u << lane) - 1u;
    uint4 *hbuf = hbufs + warp * 32;
    WarpQueue &Q = wqs[warp];
    long long *accs = accw + warp * 2 * nl * 32 + lane;   // this lane's column: accs[(par * nl + l) * 32]
    unsigned int *dc = cw + warp * 2 * nl;
    unsigned long long *dhs = hw + warp * 2 * nl;
    const uint32_t n_trials = (uint32_t)A.yet.n_trials;   // <= 2^32 - 1 (ara_load_yet)
    const uint32_t first_trial = (uint32_t)A.yet.first_trial;
    const uint32_t cap = A.cap;
    const bool terms = A.pf.any_terms != 0;
    const SplitRec *__restrict__ srecs = A.pf.srecs;
    const float2 *__restrict__ hot = A.pf.hot;
    const float2 *__restrict__ tables = A.pf.tables;
    const uint32_t *__restrict__ rmeta = A.pf.rec_meta;
    const uint2 *__restrict__ cidx = A.pf.cidx;

    // per-lane state; the warp-uniform queue state lives in Q (shared memory)
    uint2 nx = make_uint2(0u, 0u);                    // hits [Q.fh, Q.fh + 32) of the fetch trial
    int redo = 0;                                     // bit p: a table-less record in parity p's trial
    // virtual lanes: current record, end of the hit's records, k | parity << 31
    uint32_t cur[2] = {0u, 0u}, end[2] = {0u, 0u}, kk[2] = {0u, 0u};
    double osum[2] = {0.0, 0.0};

    auto claim = [&]() {
        for (;;) {
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(&A.status->next_trial2, 1ull);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= n_trials) { Q.fdone = 1u; return; }
            const uint32_t cnt = __ldg(A.counts + t);
            if (cnt == kOverflow) continue;           // redone by the fused kernel
            const uint32_t par = Q.nc & 1u;
            Q.tid[par] = (uint32_t)t;
            Q.rem[par] = cnt;
            Q.nc += 1u;
            Q.hoff = t * (uint64_t)cap;
            Q.fnh = cnt;
            Q.fh = 0u;
            nx = lane < cnt ? __ldcs(A.hits + Q.hoff + lane) : make_uint2(0u, 0u);
            return;
        }
    };
    auto retire_ready = [&]() -> bool {
        const uint32_t s0 = Q.s0;
        if (s0 >= Q.nc) return false;
        const uint32_t par = s0 & 1u;
        if (Q.rem[par] != 0u) return false;
        const bool mine = (cur[0] < end[0] && (kk[0] >> 31) == par) || (cur[1] < end[1] && (kk[1] >> 31) == par);
        return !__any_sync(0xffffffffu, mine);
    };
    // trial s0 is complete: aggregate terms (line 12, G6) -> YLT (line 17)
    auto retire = [&]() {
        const uint32_t par = Q.s0 & 1u, t = Q.tid[par];
        const bool rd = __any_sync(0xffffffffu, (redo >> par) & 1);
        if (rd && lane == 0) A.redo[atomicAdd(&A.status->n_redo, 1u)] = t;
        for (uint32_t l = 0; l < nl; ++l) {
            long long &a = accs[(par * nl + l) * 32];
            const long long si = warp_sum_i64_(a);
            a = 0;
            if (lane == 0 && !rd) {
                const LayerInfo &L = layers[l];
                A.ylt[(uint64_t)l * n_trials + t] = (float)fmin(fmax((double)si * L.fx_inv - L.agg_r, 0.0), L.agg_l);
                if (DBG) {
                    if (A.dbg_count) A.dbg_count[(uint64_t)l * n_trials + t] = dc[par * nl + l];
                    if (A.dbg_hash) A.dbg_hash[(uint64_t)l * n_trials + t] = dhs[par * nl + l];
                }
            }
        }
        __syncwarp();
        if (DBG)
            for (uint32_t l = lane; l < nl; l += 32) { dc[par * nl + l] = 0u; dhs[par * nl + l] = 0ull; }
        redo &= ~(1 << par);
        __syncwarp();
        Q.s0 += 1u;
    };
    // hand the next hits, in order, to the virtual lanes whose hit is done
    auto refill = [&]() {
        for (;;) {
            const bool n0 = !(cur[0] < end[0]), n1 = !(cur[1] < end[1]);
            const uint32_t m0 = __ballot_sync(0xffffffffu, n0), m1 = __ballot_sync(0xffffffffu, n1);
            const uint32_t tot = __popc(m0) + __popc(m1);
            if (tot == 0) return;
            const uint32_t bq = Q.bq, bn = Q.bn;
            if (bq < bn) {
                const uint32_t avail = bn - bq, bpar = Q.bpar;
                const uint32_t r0 = __popc(m0 & lt), r1 = __popc(m0) + __popc(m1 & lt);
                if (n0 && r0 < avail) {
                    const uint4 v = hbuf[bq + r0];
                    cur[0] = v.x; end[0] = v.y; kk[0] = v.z | (bpar << 31);
                }
                if (n1 && r1 < avail) {
                    const uint4 v = hbuf[bq + r1];
                    cur[1] = v.x; end[1] = v.y; kk[1] = v.z | (bpar << 31);
                }
                const uint32_t take = min(tot, avail);
                Q.bq = bq + take;
                Q.rem[bpar] -= take;
                __syncwarp();
                if (take == tot) return;
                continue;
            }
            const uint32_t fh = Q.fh, fnh = Q.fnh;
            if (Q.nc == 0u || fh >= fnh) {            // fetch trial exhausted: claim the next
                if (Q.fdone || Q.nc >= Q.s0 + 2u) return;   // none left / window full
                claim();
                continue;
            }
            // next batch of the fetch trial: event index entries (line 6)
            uint2 ci = make_uint2(0u, 0u);
            if (fh + lane < fnh) ci = __ldg(cidx + nx.x);
            const bool ok = ci.y != 0u;               // a shared presence bit may cover an absent event
            const uint32_t om = __ballot_sync(0xffffffffu, ok);
            if (ok) hbuf[__popc(om & lt)] = make_uint4(ci.x, ci.x + ci.y, nx.y, 0u);
            const uint32_t nb = __popc(om), bpar = (Q.nc - 1u) & 1u;
            Q.bn = nb;
            Q.bq = 0u;
            Q.bpar = bpar;
            Q.rem[bpar] -= min(32u, fnh - fh) - nb;   // absent events: handed out as nothing
            Q.fh = fh + 32u;
            nx = fh + 32u + lane < fnh ? __ldcs(A.hits + Q.hoff + fh + 32u + lane) : make_uint2(0u, 0u);
            __syncwarp();
        }
    };

    for (;;) {
        bool live[2];
        for (;;) {
            while (retire_ready()) retire();
            refill();
            live[0] = cur[0] < end[0];
            live[1] = cur[1] < end[1];
            if (__any_sync(0xffffffffu, live[0] || live[1])) break;
            if (Q.fdone && Q.s0 >= Q.nc) return;
        }

        // one present pair per live virtual lane (Alg.1 lines 7-9)
        uint32_t rec[2], meta[2];
        float x[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) rec[u] = live[u] ? cur[u] : 0u;
        if (SU) {
            SplitRec r[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                r[u] = live[u] ? srecs[rec[u]] : SplitRec{0, 0, 0, 0, 0, kModeDegenerate << 28, 0, 0};
                meta[u] = r[u].meta;
            }
            float v[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t tg = first_trial + Q.tid[kk[u] >> 31], k = kk[u] & 0x7fffffffu;
                const uint32_t bp = philox_lane0_k(tg, k, r[u].prog, 1u, A.pkey);    // z_(Prog,E)
                const uint32_t be = philox_lane0_k(tg, k, r[u].elt, 2u, A.pkey);     // z_(E)
                v[u] = fmaf(r[u].wi, norm_quantile_from_bits(bp), r[u].wc * norm_quantile_from_bits(be));
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t mode = meta[u] >> 28;
                if (mode == kModeTable) {
                    const float uu = (fminf(fmaxf(v[u], kTabV0), -kTabV0) - kTabV0) * (1.0f / kTabH);
                    const int ti = min((int)uu, kTabNodes - 2);
                    const float tt = uu - (float)ti;
                    const bool in_hot = (unsigned)(ti - kHotJ0) < (unsigned)(kHotN - 1);
                    const float2 *row = in_hot ? hot + (uint64_t)rec[u] * kHotN + (ti - kHotJ0)
                                               : tables + (uint64_t)rec[u] * kTabStride + ti;
                    x[u] = r[u].scale * sigmoidf_(quintic_from_nodes(__ldg(row), __ldg(row + 1), ti, tt,
                                                                     r[u].a, r[u].b));
                } else if (mode == kModeDegenerate) {
                    x[u] = r[u].scale;
                } else {
                    x[u] = 0.0f;                      // table-less record: trial redone in fp64
                    redo |= 1 << (kk[u] >> 31);
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                meta[u] = live[u] ? __ldg(rmeta + rec[u]) : 0u;
                x[u] = live[u] ? __ldg(A.pf.rec_mu + rec[u]) : 0.0f;
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t layer = (meta[u] >> 16) & 63u;
            if (terms) {                                              // line 8 (G7)
                const SlotInfo &si = slots[meta[u] & 0xffu];
                if (si.has_terms) x[u] = si.share * fminf(fmaxf(x[u] - si.ret, 0.0f), si.lim);
            }
            if (DBG && live[u]) {
                const uint32_t elt = slots[meta[u] & 0xffu].elt;
                const uint32_t par = kk[u] >> 31;
                atomicAdd(&dc[par * nl + layer], 1u);
                const uint64_t hv = splitmix64_(splitmix64_(splitmix64_((uint64_t)(kk[u] & 0x7fffffffu)) ^ elt) ^
                                                A.pf.rec_orig[rec[u]]);
                atomicAdd(&dhs[par * nl + layer], (unsigned long long)hv);
            }
            // occurrence sum of the (occurrence, layer) run (line 9); at its
            // last record the occurrence terms (line 11) into the trial sum
            const double o = osum[u] + (double)x[u];
            const bool run_end = live[u] && (meta[u] & 0x100u);
            if (run_end) {
                const LayerInfo &L = layers[layer];
                const long long gi = __double2ll_rn(fmin(fmax(o - L.occ_r, 0.0), L.occ_l) * L.fx_scale);
                accs[((kk[u] >> 31) * nl + layer) * 32] += gi;
            }
            osum[u] = run_end ? 0.0 : (live[u] ? o : osum[u]);
            cur[u] += live[u] ? 1u : 0u;
        }
    }
}

__global__ void split_recs_kernel(const BetaRec *__restrict__ recs, const uint32_t *__restrict__ rec_meta,
                                  const SlotInfo *__restrict__ slots, uint64_t n, SplitRec *__restrict__ out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const BetaRec r = recs[t];
        const uint32_t m = rec_meta[t];
        const SlotInfo &s = slots[m & 0xffu];
        out[t] = SplitRec{r.a, r.b, r.wi, r.wc, r.scale, m | (r.mode << 28), s.elt, s.prog};
    }
}

void launch_split_recs(const BetaRec *recs, const uint32_t *rec_meta, const SlotInfo *slots, uint64_t n,
                       SplitRec *out, cudaStream_t s) {
    if (n == 0) return;
    const uint64_t blocks = (n + 255) / 256;
    split_recs_kernel<<<(unsigned)(blocks < 65535u * 16u ? blocks : 65535u * 16u), 256, 0, s>>>(recs, rec_meta,
                                                                                               slots, n, out);
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

cudaError_t launch_compact(const SplitArgs &A, cudaStream_t s, int num_sms) {
    const size_t smem = (A.pf.bitmap_words * 4u + 15u) & ~15u;
    cudaError_t err = cudaFuncSetAttribute(compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, compact_kernel, kCompactThreads, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    compact_kernel<<<num_sms * per_sm, kCompactThreads, smem, s>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_sample(const SplitArgs &A, cudaStream_t s, int num_sms) {
    const bool dbg = (A.flags & ARA_DEBUG_LOOKUP) != 0, su = (A.flags & ARA_SU) != 0;
    const bool sl = A.pf.n_layers == 1;
    if (A.pf.n_layers > kSplitMaxLayers) return cudaErrorInvalidValue;
    const size_t smem = sizeof(SlotInfo) * ARA_MAX_SLOTS + sizeof(LayerInfo) * ARA_MAX_LAYERS +
                        sizeof(uint4) * kSampleWarps * 32 + sizeof(WarpQueue) * kSampleWarps +
                        sizeof(long long) * kSampleWarps * 2 * A.pf.n_layers * 32 +
                        kSampleWarps * 2 * A.pf.n_layers * (sizeof(unsigned int) + sizeof(unsigned long long)) + 16;
    using K = void (*)(SplitArgs);
    const K kern = su ? (sl ? (dbg ? (K)sample_kernel<true, true, true> : (K)sample_kernel<true, true, false>)
                            : (dbg ? (K)sample_kernel<true, false, true> : (K)sample_kernel<true, false, false>))
                      : (sl ? (dbg ? (K)sample_kernel<false, true, true> : (K)sample_kernel<false, true, false>)
                            : (dbg ? (K)sample_kernel<false, false, true> : (K)sample_kernel<false, false, false>));
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSampleWarps * 32, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    kern<<<num_sms * per_sm, kSampleWarps * 32, smem, s>>>(A);
    return cudaGetLastError();
}

}  // namespace ara
