// ara_split.cu -- the two-kernel form of the YET scan (Algorithm 1,
// P:134-170), the default path of ara_run:
//
//   compact_kernel : YET stream (line 4) + direct-access lookup (line 6):
//                    per trial, the list of present (occurrence, slot) pairs,
//                    written to a fixed-capacity per-trial region of HBM.
//                    Latency-bound (HBM events, L2 index), so it runs 32
//                    warps per SM with a small register budget.
//   sample_kernel  : per trial, its pairs in dense 32-wide rounds: draws
//                    (line 7, section 3), XELT terms (line 8), a segmented
//                    warp scan for the per-occurrence sums (line 9),
//                    occurrence terms (line 11), fp64 trial sums, aggregate
//                    terms (line 12) -> YLT (line 17).  ALU-bound.
//
// A trial whose pairs overflow the region, or that meets a table-less
// record, is listed for the fused fp64-capable kernel (ara_kernels.cu).
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"
#include "ara_sampler.cuh"

#ifndef ARA_COMPACT_COMBINED
#define ARA_COMPACT_COMBINED 0
#endif
#ifndef ARA_SEG_EARLY_EXIT
#define ARA_SEG_EARLY_EXIT 0
#endif

namespace ara {

namespace {

constexpr int kCompactWarps = 32;   // 1024 threads, <= 64 registers
constexpr int kSampleWarps = 16;    // 512 threads

__device__ __forceinline__ uint64_t splitmix64_(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <int MW>
__device__ __forceinline__ void load_index_(const uint32_t *index, uint32_t stride, uint32_t e, uint32_t &first,
                                            uint32_t (&mask)[MW]) {
    const uint32_t *ix = index + (uint64_t)e * stride;
    if (MW == 1) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(ix));
        first = v.x; mask[0] = v.y;
    } else {
        const uint4 v0 = __ldg(reinterpret_cast<const uint4 *>(ix));
        first = v0.x; mask[0] = v0.y;
        if (MW > 1) mask[1] = v0.z;
        if (MW > 2) mask[2] = v0.w;
        if (MW > 3) {
            const uint4 v1 = __ldg(reinterpret_cast<const uint4 *>(ix) + 1);
            mask[3] = v1.x;
            if (MW > 4) mask[4] = v1.y;
            if (MW > 5) mask[5] = v1.z;
            if (MW > 6) mask[6] = v1.w;
        }
    }
}

__device__ __forceinline__ double warp_sum_f64_(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace

// ---------------------------------------------------------------------------
// compact_kernel: one warp per trial (dynamic scheduler).  Per 128-event
// chunk: uint4 event loads (evict-first, next chunk prefetched), presence
// bitmap in shared memory, index entries of the hits (L2), one warp prefix sum
// of the pair counts, pairs written in (occurrence, slot) order.
// counts[t] = pairs of trial t, or kOverflow (then t is appended to redo).
// ---------------------------------------------------------------------------
template <int MW>
__global__ void __launch_bounds__(kCompactWarps * 32, 1)
    compact_kernel(const __grid_constant__ SplitArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem);
    for (uint32_t t = threadIdx.x; t < A.pf.bitmap_words; t += blockDim.x) bitmap[t] = A.pf.bitmap[t];
    __syncthreads();

    const int lane = threadIdx.x & 31;
    const uint64_t n_trials = A.yet.n_trials;
    const uint32_t C = A.pf.catalog, shift = A.pf.bitmap_shift, cap = A.cap;
    const uint32_t *index = A.pf.index;
    const uint32_t stride = A.pf.idx_stride;

    while (true) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&A.status->next_trial, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n_trials) break;
        const uint64_t base = A.yet.fixed_len ? t * (uint64_t)A.yet.fixed_len : A.yet.offsets[t];
        const uint32_t len = A.yet.fixed_len ? A.yet.fixed_len : (uint32_t)(A.yet.offsets[t + 1] - base);
        const uint32_t *ev = A.yet.events + base;
        const bool vec = (base & 3u) == 0;
        uint2 *out = A.pairs + t * (uint64_t)cap;
        uint32_t n = 0;                                  // pairs so far (warp-uniform)
        auto load4 = [&](uint32_t k) -> uint4 {
            uint4 r = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
            if (vec && k + 3 < len) return __ldcs(reinterpret_cast<const uint4 *>(ev + k));
            if (k < len) r.x = __ldcs(ev + k);
            if (k + 1 < len) r.y = __ldcs(ev + k + 1);
            if (k + 2 < len) r.z = __ldcs(ev + k + 2);
            if (k + 3 < len) r.w = __ldcs(ev + k + 3);
            return r;
        };
        uint4 nxt = load4(4u * lane);
        for (uint32_t c = 0; c < len; c += 128) {                   // Alg.1 line 4
            const uint4 cur = nxt;
            nxt = load4(c + 128 + 4u * lane);
            const uint32_t k0 = c + 4u * lane;
            const uint32_t ee[4] = {cur.x, cur.y, cur.z, cur.w};
            uint32_t first[4], mask[4][MW], np = 0;
#pragma unroll
            for (int qd = 0; qd < 4; ++qd) {
                const uint32_t e = ee[qd];
                first[qd] = 0;
#pragma unroll
                for (int w = 0; w < MW; ++w) mask[qd][w] = 0u;
                if (k0 + qd < len) {
                    if (e >= C) {
                        atomicAdd(&A.status->bad_event, 1u);
                    } else {
                        const uint32_t bit = e >> shift;
                        if ((bitmap[bit >> 5] >> (bit & 31)) & 1u)
                            load_index_<MW>(index, stride, e, first[qd], mask[qd]);   // line 6
                    }
                }
            }
#pragma unroll
            for (int qd = 0; qd < 4; ++qd)
#pragma unroll
                for (int w = 0; w < MW; ++w) np += __popc(mask[qd][w]);
            uint32_t incl = np;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t pos = n + incl - np;
            if (MW == 1 && ARA_COMPACT_COMBINED) {
                // one loop over the set bits of all four occurrences, in
                // (occurrence, slot) order: trip count = this lane's pairs
                uint32_t m0 = mask[0][0], m1 = mask[1][0], m2 = mask[2][0], m3 = mask[3][0];
                uint32_t r0 = first[0], r1 = first[1], r2 = first[2], r3 = first[3];
                while (m0 | m1 | m2 | m3) {
                    const int qd = m0 ? 0 : (m1 ? 1 : (m2 ? 2 : 3));
                    const uint32_t mw = qd == 0 ? m0 : (qd == 1 ? m1 : (qd == 2 ? m2 : m3));
                    const uint32_t rec = qd == 0 ? r0 : (qd == 1 ? r1 : (qd == 2 ? r2 : r3));
                    const uint32_t slot = (uint32_t)(__ffs(mw) - 1);
                    if (pos < cap) out[pos] = make_uint2(rec, ((k0 + qd) << 8) | slot);
                    ++pos;
                    const uint32_t mn = mw & (mw - 1);
                    if (qd == 0) { m0 = mn; ++r0; } else if (qd == 1) { m1 = mn; ++r1; }
                    else if (qd == 2) { m2 = mn; ++r2; } else { m3 = mn; ++r3; }
                }
            } else {
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                    uint32_t rec = first[qd];
#pragma unroll
                    for (int w = 0; w < MW; ++w) {
                        uint32_t mw = mask[qd][w];
                        while (mw) {
                            const uint32_t slot = (uint32_t)(w * 32 + __ffs(mw) - 1);
                            mw &= mw - 1;
                            if (pos < cap) out[pos] = make_uint2(rec, ((k0 + qd) << 8) | slot);
                            ++pos;
                            ++rec;
                        }
                    }
                }
            }
            n += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) {
            A.counts[t] = n <= cap ? n : kOverflow;
            if (n > cap) A.redo[atomicAdd(&A.status->n_redo, 1u)] = (uint32_t)t;
        }
    }
}

// ---------------------------------------------------------------------------
// sample_kernel: one warp per trial (dynamic scheduler); the trial's pairs in
// rounds of 64 (two per lane in flight).  Per round: record + table loads,
// Philox draws, steps 2-4, quantile table, XELT terms; then a segmented
// inclusive scan (fp64, keyed by occurrence and layer) carried across rounds;
// segment tails apply the occurrence terms and accumulate the trial sum.
// SL: single-layer portfolio (per-lane fp64 accumulators, one warp sum at the
// end); otherwise per-layer sums in shared memory via fixed-tree reductions.
// ---------------------------------------------------------------------------
template <bool SU, bool SL, bool DBG>
__global__ void __launch_bounds__(kSampleWarps * 32, 2)   // 2 CTAs/SM: <= 64 registers
    sample_kernel(const __grid_constant__ SplitArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    SlotInfo *slots = reinterpret_cast<SlotInfo *>(smem);
    LayerInfo *layers = reinterpret_cast<LayerInfo *>(slots + ARA_MAX_SLOTS);
    double *Sw = reinterpret_cast<double *>(layers + ARA_MAX_LAYERS);   // [warps][n_layers]
    unsigned int *cw = reinterpret_cast<unsigned int *>(Sw + kSampleWarps * A.pf.n_layers);
    unsigned long long *hw = reinterpret_cast<unsigned long long *>(
        ((uintptr_t)(cw + kSampleWarps * A.pf.n_layers) + 7) & ~(uintptr_t)7);
    for (uint32_t t = threadIdx.x; t < A.pf.n_slots; t += blockDim.x) slots[t] = A.pf.slots[t];
    for (uint32_t t = threadIdx.x; t < A.pf.n_layers; t += blockDim.x) layers[t] = A.pf.layers[t];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t nl = A.pf.n_layers;
    double *S = Sw + warp * nl;
    unsigned int *dc = cw + warp * nl;
    unsigned long long *dhs = hw + warp * nl;
    const uint64_t n_trials = A.yet.n_trials;
    const uint64_t seed = A.seed;
    const BetaRec *__restrict__ recs = A.pf.recs;
    const float2 *__restrict__ hot = A.pf.hot;
    const float2 *__restrict__ tables = A.pf.tables;

    while (true) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&A.status->next_trial2, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n_trials) break;
        const uint32_t n = __ldg(A.counts + t);
        if (n == kOverflow) continue;                 // redone by the fused kernel
        const uint32_t trial_g = (uint32_t)(A.yet.first_trial + t);
        const uint2 *in = A.pairs + t * (uint64_t)A.cap;
        if (!SL || DBG)
            for (uint32_t l = lane; l < nl; l += 32) { S[l] = 0.0; dc[l] = 0u; dhs[l] = 0ull; }
        __syncwarp();
        double acc = 0.0;                              // SL: this lane's share of the trial sum
        uint32_t ckey = 0xffffffffu;                   // segment carried from the previous round
        double csum = 0.0;
        int redo = 0;
        for (uint32_t b = 0; b < n; b += 64) {
            uint2 e[2];
            float x[2];
            bool live[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t p = b + 32u * u + lane;
                live[u] = p < n;
                e[u] = live[u] ? __ldcs(in + p) : make_uint2(0u, 0xffffffffu);
            }
            if (SU) {
                BetaRec r[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) r[u] = live[u] ? recs[e[u].x] : BetaRec{0, 0, 0, 0, 0, 0, 0, kModeDegenerate};
                float v[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const SlotInfo &si = slots[live[u] ? (e[u].y & 0xffu) : 0u];
                    const uint32_t k = e[u].y >> 8;
                    const uint32_t bp = philox_lane0(trial_g, k, si.prog, 1u, seed);    // z_(Prog,E)
                    const uint32_t be = philox_lane0(trial_g, k, si.elt, 2u, seed);     // z_(E)
                    v[u] = combine_v(r[u], norm_quantile_from_bits(bp), norm_quantile_from_bits(be));
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (r[u].mode == kModeTable) {
                        const float uu = (fminf(fmaxf(v[u], kTabV0), -kTabV0) - kTabV0) * (1.0f / kTabH);
                        const int ti = min((int)uu, kTabNodes - 2);
                        const float tt = uu - (float)ti;
                        const bool in_hot = (unsigned)(ti - kHotJ0) < (unsigned)(kHotN - 1);
                        const float2 *row = in_hot ? hot + (uint64_t)e[u].x * kHotN + (ti - kHotJ0)
                                                   : tables + (uint64_t)e[u].x * kTabStride + ti;
                        x[u] = r[u].scale * sigmoidf_(quintic_from_nodes(__ldg(row), __ldg(row + 1), ti, tt,
                                                                         r[u].a, r[u].b));
                    } else if (r[u].mode == kModeDegenerate) {
                        x[u] = r[u].scale;
                    } else {
                        x[u] = 0.0f;                  // table-less record: trial redone in fp64
                        redo = 1;
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < 2; ++u) x[u] = live[u] ? __ldg(A.pf.rec_mu + e[u].x) : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const uint32_t slot = e[u].y & 0xffu;
                const SlotInfo &si = slots[live[u] ? slot : 0u];
                if (live[u] && si.has_terms) x[u] = si.share * fminf(fmaxf(x[u] - si.ret, 0.0f), si.lim);
                const uint32_t layer = live[u] ? si.layer : 0u;
                if (DBG && live[u]) {
                    atomicAdd(&dc[layer], 1u);
                    const uint64_t hv = splitmix64_(splitmix64_(splitmix64_((uint64_t)(e[u].y >> 8)) ^ si.elt) ^
                                                    A.pf.rec_orig[e[u].x]);
                    atomicAdd(&dhs[layer], (unsigned long long)hv);
                }
                // segmented inclusive scan over (occurrence, layer) keys (line 9);
                // a segment open at the end of the previous sub-round is carried
                const uint32_t key = live[u] ? ((e[u].y & 0xffffff00u) | layer) : 0xfffffffeu;
                const uint32_t key0 = __shfl_sync(0xffffffffu, key, 0);
                if (ckey != 0xffffffffu && key0 != ckey) {          // the carried segment ended
                    if (lane == 0) {
                        const LayerInfo &L = layers[ckey & 0xffu];
                        const double g = fmin(fmax(csum - L.occ_r, 0.0), L.occ_l);   // line 11
                        if (SL) acc += g; else S[ckey & 0xffu] += g;
                    }
                    ckey = 0xffffffffu;
                }
                // fp32 within an occurrence (<= one value per slot); the carry and
                // the trial sums stay fp64.  Segments are short, so the scan stops
                // as soon as no lane's segment reaches further back.
                float val = live[u] ? x[u] : 0.0f;
                double carry = (lane == 0 && key == ckey) ? csum : 0.0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float y = __shfl_up_sync(0xffffffffu, val, o);
                    const uint32_t ky = __shfl_up_sync(0xffffffffu, key, o);
                    const bool same = lane >= o && ky == key;
                    if (same) val += y;
                    if (ARA_SEG_EARLY_EXIT && !__any_sync(0xffffffffu, same)) break;
                }
                // the carried part reaches every lane of the first segment
                carry = __shfl_sync(0xffffffffu, carry, 0);
                const bool in_first = key == key0 && key0 == ckey;
                const double full = (double)val + (in_first ? carry : 0.0);
                const uint32_t nextkey = __shfl_down_sync(0xffffffffu, key, 1);
                // lane 31's segment may continue into the next sub-round: carry it
                const bool tail = live[u] && lane != 31 && nextkey != key;
                const bool l31 = __shfl_sync(0xffffffffu, (int)live[u], 31) != 0;
                ckey = l31 ? __shfl_sync(0xffffffffu, key, 31) : 0xffffffffu;
                csum = __shfl_sync(0xffffffffu, full, 31);
                double g = 0.0;
                if (tail) {                                           // occurrence terms (line 11)
                    const LayerInfo &L = layers[layer];
                    g = fmin(fmax(full - L.occ_r, 0.0), L.occ_l);
                    if (SL) acc += g;
                }
                if (!SL) {
                    // per-layer trial sums: one fixed-tree warp sum per distinct layer
                    unsigned pending = __ballot_sync(0xffffffffu, tail);
                    while (pending) {
                        const int leader = __ffs(pending) - 1;
                        const uint32_t lay = __shfl_sync(0xffffffffu, layer, leader);
                        const bool mine = tail && layer == lay;
                        const double sm = warp_sum_f64_(mine ? g : 0.0);
                        if (lane == 0) S[lay] += sm;
                        pending &= ~__ballot_sync(0xffffffffu, mine);
                    }
                }
            }
        }
        // the last segment, carried out of the final sub-round
        if (ckey != 0xffffffffu && lane == 0) {
            const LayerInfo &L = layers[ckey & 0xffu];
            const double g = fmin(fmax(csum - L.occ_r, 0.0), L.occ_l);
            if (SL) acc += g; else S[ckey & 0xffu] += g;
        }
        redo = __any_sync(0xffffffffu, redo);
        if (redo) {
            if (lane == 0) A.redo[atomicAdd(&A.status->n_redo, 1u)] = (uint32_t)t;
            continue;
        }
        // aggregate terms (line 12, G6) -> YLT (line 17)
        if (SL) {
            const double Sum = warp_sum_f64_(acc);
            if (lane == 0) {
                const LayerInfo &L = layers[0];
                A.ylt[t] = (float)fmin(fmax(Sum - L.agg_r, 0.0), L.agg_l);
                if (DBG) {
                    if (A.dbg_count) A.dbg_count[t] = dc[0];
                    if (A.dbg_hash) A.dbg_hash[t] = dhs[0];
                }
            }
        } else {
            __syncwarp();
            for (uint32_t l = lane; l < nl; l += 32) {
                const LayerInfo &L = layers[l];
                A.ylt[(uint64_t)l * n_trials + t] = (float)fmin(fmax(S[l] - L.agg_r, 0.0), L.agg_l);
                if (DBG) {
                    if (A.dbg_count) A.dbg_count[(uint64_t)l * n_trials + t] = dc[l];
                    if (A.dbg_hash) A.dbg_hash[(uint64_t)l * n_trials + t] = dhs[l];
                }
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
template <int MW>
static cudaError_t launch_compact_mw(const SplitArgs &A, cudaStream_t s, int num_sms) {
    const size_t smem = (A.pf.bitmap_words * 4u + 15u) & ~15u;
    auto kern = compact_kernel<MW>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCompactWarps * 32, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    kern<<<num_sms * per_sm, kCompactWarps * 32, smem, s>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_compact(const SplitArgs &A, cudaStream_t s, int num_sms) {
    if (A.pf.mask_words == 1) return launch_compact_mw<1>(A, s, num_sms);
    if (A.pf.mask_words <= 3) return launch_compact_mw<3>(A, s, num_sms);
    if (A.pf.mask_words == 4) return launch_compact_mw<4>(A, s, num_sms);
    return launch_compact_mw<7>(A, s, num_sms);
}

cudaError_t launch_sample(const SplitArgs &A, cudaStream_t s, int num_sms) {
    const bool dbg = (A.flags & ARA_DEBUG_LOOKUP) != 0, su = (A.flags & ARA_SU) != 0;
    const bool sl = A.pf.n_layers == 1;
    const size_t smem = sizeof(SlotInfo) * ARA_MAX_SLOTS + sizeof(LayerInfo) * ARA_MAX_LAYERS +
                        kSampleWarps * A.pf.n_layers * (sizeof(double) + sizeof(unsigned int) +
                                                     sizeof(unsigned long long)) + 16;
    auto pick = [&]() {
        if (su) {
            if (sl) return dbg ? sample_kernel<true, true, true> : sample_kernel<true, true, false>;
            return dbg ? sample_kernel<true, false, true> : sample_kernel<true, false, false>;
        }
        if (sl) return dbg ? sample_kernel<false, true, true> : sample_kernel<false, true, false>;
        return dbg ? sample_kernel<false, false, true> : sample_kernel<false, false, false>;
    };
    auto kern = pick();
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
