// ara_primary.cu -- the YET scan when no draw is taken: primary uncertainty
// only (ara_run without ARA_SU), or a portfolio whose every record has
// sigma_I = sigma_C = 0 (reading G10: the loss is the mean).  Then lines 6-11
// of Algorithm 1 -- lookup, loss, XELT terms, the per-event sum
// over a layer's XELTs and the occurrence terms -- depend on the event alone,
// so they are evaluated ONCE per (event, layer) at ara_create_portfolio
// (occ_table_kernel, fp64) and the run is a single streaming pass:
//
//   primary_kernel : per trial, stream the event ids (line 4), test the
//                    shared-memory presence bitmap, gather the event's
//                    occurrence losses (one 32-B sector for <= 8 layers),
//                    add them to per-lane fp64 sums (line 12's S), fixed-tree
//                    warp sum, aggregate terms -> YLT (lines 12, 17).
//
// The trial sum runs in an order fixed by the occurrence positions (per lane,
// then a fixed tree), so the YLT is a pure function of (portfolio, YET).
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"

namespace ara {

namespace {

constexpr int kPrimaryWarps = 32;

__device__ __forceinline__ double clip64(double d, double lim) {   // min(max(d, 0), lim) (G5)
    return d > 0.0 ? (d < lim ? d : lim) : 0.0;
}

}  // namespace

// ---------------------------------------------------------------------------
// occ_table[e * LP + l] = g_occ(sum over layer l's records of event e of the
// record's (XELT-termed) mean loss), 0 if the layer holds no record of e.
// One thread per event; the records of an event are consecutive, in slot
// (= layer, then XELT) order, so each layer's sum runs in the layer's XELT
// order, as Algorithm 1's line 5 loop does.
// ---------------------------------------------------------------------------
__global__ void occ_table_kernel(const uint2 *__restrict__ cidx, const uint2 *__restrict__ mu_meta,
                                 const double *__restrict__ slot_terms,
                                 const LayerInfo *__restrict__ layers, uint32_t n_layers, uint32_t lp,
                                 uint32_t catalog, float *__restrict__ out) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < catalog;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 ci = cidx[e];
        uint32_t r = ci.x;
        const uint32_t r1 = ci.x + ci.y;
        for (uint32_t l = 0; l < lp; ++l) {
            double sum = 0.0;
            bool any = false;
            while (r < r1 && ((mu_meta[r].y >> 16) & 63u) == l) {   // layer l's records of e
                const uint32_t slot = mu_meta[r].y & 0xffu;
                double x = (double)__uint_as_float(mu_meta[r].x);   // the loss (G10 / SU off)
                const double *T = slot_terms + 4 * slot;            // XELT terms (line 8, G7)
                if (T[3] != 0.0) x = T[2] * clip64(x - T[0], T[1]);
                sum += x;                                           // line 9
                any = true;
                ++r;
            }
            float g = 0.0f;
            if (any && l < n_layers) g = (float)clip64(sum - layers[l].occ_r, layers[l].occ_l);   // line 11
            out[e * lp + l] = g;
        }
    }
}

void launch_occ_table(const uint2 *cidx, const uint2 *mu_meta, const double *slot_terms,
                      const LayerInfo *layers, uint32_t n_layers, uint32_t lp, uint32_t catalog, float *out,
                      cudaStream_t s) {
    if (catalog == 0) return;
    const uint64_t blocks = (catalog + 255) / 256;
    occ_table_kernel<<<(unsigned)(blocks < 65535u * 16u ? blocks : 65535u * 16u), 256, 0, s>>>(
        cidx, mu_meta, slot_terms, layers, n_layers, lp, catalog, out);
}

// occ_bitmap bit b = some event e of the bit (e >> shift == b, e < catalog) has
// a nonzero occurrence loss in some layer.  An event whose occurrence losses
// are all 0 adds exactly 0 to every trial sum (and to no occurrence maximum),
// so the primary path may skip it like an absent one: the YLT is unchanged
// bit for bit, and the gathers drop to the events that carry a loss (cfg2:
// the occurrence retention zeroes ~40 % of the present events).
__global__ void occ_bitmap_kernel(const float *__restrict__ occ, uint32_t lp, uint32_t catalog, uint32_t shift,
                                  uint32_t words, uint32_t *__restrict__ out) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
        uint32_t m = 0;
        for (uint32_t b = 0; b < 32; ++b) {
            const uint64_t e0 = ((uint64_t)w * 32 + b) << shift, e1 = (((uint64_t)w * 32 + b + 1) << shift);
            bool nz = false;
            for (uint64_t e = e0; e < e1 && e < catalog && !nz; ++e)
                for (uint32_t l = 0; l < lp; ++l) nz = nz || occ[e * lp + l] != 0.0f;
            m |= (nz ? 1u : 0u) << b;
        }
        out[w] = m;
    }
}

void launch_occ_bitmap(const float *occ, uint32_t lp, uint32_t catalog, uint32_t shift, uint32_t words,
                       uint32_t *out, cudaStream_t s) {
    if (words == 0) return;
    occ_bitmap_kernel<<<(words + 255) / 256, 256, 0, s>>>(occ, lp, catalog, shift, words, out);
}

// ---------------------------------------------------------------------------
// primary_kernel: one warp per trial (dynamic scheduler), one CTA of 32 warps
// per SM with the presence bitmap in shared memory.  Per 128-event chunk one
// uint4 of ids per lane (evict-first); the next chunk is in flight while
// this one's occurrence losses are gathered (predicated, through L2).
// LP: occurrence losses per event (1, 2, 4 or 8 layers, padded).
// BM: as compact_kernel (0: shift 0 + sentinel, 1: any shift + sentinel,
// 2: any shift, per-event length test).
// ---------------------------------------------------------------------------
template <int LP>
__device__ __forceinline__ void load_occ(bool p, const float *src, float (&g)[LP]) {
#pragma unroll
    for (int l = 0; l < LP; ++l) g[l] = 0.0f;
    if constexpr (LP == 1) {                      // predicated gathers, no branch
        asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %1, 0;\n @q ld.global.nc.f32 %0, [%2];\n}"
                     : "+f"(g[0]) : "r"((uint32_t)p), "l"(src));
    } else if constexpr (LP == 2) {
        asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.global.nc.v2.f32 {%0, %1}, [%3];\n}"
                     : "+f"(g[0]), "+f"(g[1]) : "r"((uint32_t)p), "l"(src));
    } else {
#pragma unroll
        for (int h = 0; h < LP; h += 4)
            asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %4, 0;\n @q ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%5];\n}"
                         : "+f"(g[h]), "+f"(g[h + 1]), "+f"(g[h + 2]), "+f"(g[h + 3])
                         : "r"((uint32_t)p), "l"(src + h));
    }
}

// One or two layers: the warp walks the flat sequence of 128-event chunks of
// the trials it claims as a register pipeline (as compact_kernel does), so the
// loss gathers of chunk c+1 and the id loads of chunks c+2, c+3 are in flight
// while chunk c is summed; a trial's sums are reduced and written after its
// last chunk.  (The per-trial loop below keeps one chunk of ids and no gathers
// in flight: it waited on L2 latency once per chunk.)
struct PrimRaw {
    uint4 v;
    uint32_t t, c, len;             // trial (kNoTrial: none), chunk, trial length
};
template <int LP>
struct PrimG {
    float g[4][LP];
    uint32_t t, c, len;
};
constexpr uint32_t kNoTrial = 0xffffffffu;

// VEC: fixed-length trials, K % 4 == 0, K > 0: trials assigned to the warps
// round-robin (equal work per trial; a claim's atomic round trip at every
// trial start stalled the warp: 18 % of the stall samples), one uint4 per lane
// from a per-trial pointer.  Else the dynamic scheduler and per-id loads.
template <int LP, int BM, bool OM, bool VEC>
__device__ __forceinline__ void primary_flat(const PrimaryArgs &A, const uint32_t *bitmap) {
    const int lane = threadIdx.x & 31;
    const uint32_t shift = A.pf.bitmap_shift, nl = A.pf.n_layers;
    const uint64_t n_trials = A.yet.n_trials;
    const uint32_t *events = A.yet.events;
    const uint64_t *offsets = A.yet.offsets;
    const uint32_t K = A.yet.fixed_len;
    const uint32_t sent = BM == 2 ? 0u : A.pf.sentinel_event;
    const float *__restrict__ occ = A.occ;

    uint32_t pt = kNoTrial, pc = 0, plen = 0;       // fetch side (warp-uniform; plen 0 without a trial)
    uint64_t pbase = 0;
    const uint4 *psrc = nullptr;                    // VEC: this lane's uint4 of the trial's chunk 0
    // VEC: this warp's next trial (round-robin over the grid's warps)
    uint64_t next_t = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint64_t n_warps = gridDim.x * (uint64_t)(blockDim.x >> 5);
    // (dynamic: claiming the next trial one ahead measured slower -- 0.139 ->
    // 0.143 ms at cfg2, the end-of-launch imbalance it adds)
    auto next_trial = [&]() {
        unsigned long long t = 0;
        if (VEC) {
            t = next_t;
            next_t += n_warps;
        } else {
            if (lane == 0) t = atomicAdd(A.sched, 1ull);
            t = __shfl_sync(0xffffffffu, t, 0);
        }
        pt = t < n_trials ? (uint32_t)t : kNoTrial;
        pc = 0;
        plen = 0;
        if (pt != kNoTrial) {
            if (VEC) { pbase = (uint64_t)pt * K; plen = K; psrc = reinterpret_cast<const uint4 *>(events + pbase) + lane; }
            else if (offsets) { pbase = offsets[pt]; plen = (uint32_t)(offsets[pt + 1] - pbase); }
            else { pbase = (uint64_t)pt * K; plen = K; }
            if (!VEC && plen == 0) {                          // empty trial: S = 0 (YLT = the clip of 0)
                if (lane == 0)
                    for (uint32_t l = 0; l < nl; ++l) {
                        const LayerInfo &L = A.pf.layers[l];
                        A.ylt[(uint64_t)l * n_trials + pt] = (float)clip64(0.0 - L.agg_r, L.agg_l);
                        if (OM) A.occ_max[(uint64_t)l * n_trials + pt] = 0.0f;
                    }
            }
        }
    };
    auto fetch = [&](PrimRaw &r) {
        if (!VEC)
            while (pt != kNoTrial && plen == 0) next_trial();
        r.t = pt; r.c = pc; r.len = plen;
        r.v = make_uint4(sent, sent, sent, sent);
        const uint32_t k = pc * 128u + 4u * lane;
        if (VEC) {
            if (k < plen) r.v = __ldcs(psrc + pc * 32u);
        } else if (pt != kNoTrial) {
            const uint32_t *src = events + pbase + k;
            if (k < plen) r.v.x = __ldcs(src);
            if (k + 1 < plen) r.v.y = __ldcs(src + 1);
            if (k + 2 < plen) r.v.z = __ldcs(src + 2);
            if (k + 3 < plen) r.v.w = __ldcs(src + 3);
        }
        if (pt != kNoTrial) {
            if ((pc + 1) * 128u >= plen) next_trial();
            else ++pc;
        }
    };
    auto stage_a = [&](const PrimRaw &r, PrimG<LP> &G) {      // bitmap, gathers issued
        G.t = r.t; G.c = r.c; G.len = r.len;
        const uint32_t k0 = r.c * 128u + 4u * lane;
        const uint32_t ee[4] = {r.v.x, r.v.y, r.v.z, r.v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t bit = BM == 0 ? ee[q] : ee[q] >> shift;
            bool hit = __funnelshift_r(bitmap[bit >> 5], 0u, bit) & 1u;
            if (BM == 2) hit = hit && k0 + q < r.len;
            ARA_CHECK(!hit || ee[q] < A.pf.catalog);
            load_occ<LP>(hit, occ + (uint64_t)ee[q] * LP, G.g[q]);
        }
    };
    double S[LP];
    float M[LP];
    auto stage_b = [&](const PrimG<LP> &G) {                 // sums; the trial's end -> YLT
        if (G.c == 0) {
#pragma unroll
            for (int l = 0; l < LP; ++l) { S[l] = 0.0; M[l] = 0.0f; }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int l = 0; l < LP; ++l) {
                S[l] += (double)G.g[q][l];               // line 12's trial sum, occurrence order per lane
                if (OM) M[l] = fmaxf(M[l], G.g[q][l]);
            }
        if ((G.c + 1) * 128u >= (VEC ? K : G.len)) {     // (VEC: every trial has K ids)
#pragma unroll
            for (int l = 0; l < LP; ++l) {
                double s = S[l];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                unsigned mb = 0;
                if (OM) mb = __reduce_max_sync(0xffffffffu, __float_as_uint(M[l]));
                if (lane == 0 && (uint32_t)l < nl) {
                    const LayerInfo &L = A.pf.layers[l];
                    A.ylt[(uint64_t)l * n_trials + G.t] = (float)clip64(s - L.agg_r, L.agg_l);
                    if (OM) A.occ_max[(uint64_t)l * n_trials + G.t] = __uint_as_float(mb);
                }
            }
        }
    };
    next_trial();
    PrimRaw ra, rb;
    PrimG<LP> ga, gb;
    fetch(ra);
    fetch(rb);
    stage_a(ra, ga);
    fetch(ra);
    while (ga.t != kNoTrial) {
        stage_a(rb, gb);
        fetch(rb);
        stage_b(ga);
        if (gb.t == kNoTrial) break;
        stage_a(ra, ga);
        fetch(ra);
        stage_b(gb);
    }
}

template <int LP, int BM, bool OM>
__global__ void __launch_bounds__(kPrimaryWarps * 32, 1) primary_kernel(const __grid_constant__ PrimaryArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(smem);
    if (*A.yet.max_event >= A.pf.catalog) {           // out-of-range ids: nothing is read
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&A.status->bad_event, 1u);
        return;
    }
    load_bitmap_smem(smem, A.pf.occ_bitmap, A.pf.bitmap_words);   // nonzero losses only (+ the zero word)
    if constexpr (LP == 1 || (LP == 2 && !OM)) {      // (registers: LP 2 with occ_max would spill)
        if (A.yet.offsets == nullptr && A.yet.fixed_len > 0 && (A.yet.fixed_len & 3u) == 0)
            primary_flat<LP, BM, OM, true>(A, bitmap);
        else
            primary_flat<LP, BM, OM, false>(A, bitmap);
        return;
    }
    const int lane = threadIdx.x & 31;
    const uint32_t shift = A.pf.bitmap_shift, nl = A.pf.n_layers;
    const uint64_t n_trials = A.yet.n_trials;
    const uint32_t *events = A.yet.events;
    const uint64_t *offsets = A.yet.offsets;
    const uint32_t K = A.yet.fixed_len;
    const bool vec = offsets == nullptr && (K & 3u) == 0;
    const uint32_t sent = BM == 2 ? 0u : A.pf.sentinel_event;
    const float *__restrict__ occ = A.occ;
    while (true) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(A.sched, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n_trials) break;
        uint64_t base;
        uint32_t len;
        if (offsets) { base = offsets[t]; len = (uint32_t)(offsets[t + 1] - base); }
        else { base = t * (uint64_t)K; len = K; }
        double S[LP];
        float M[LP];
#pragma unroll
        for (int l = 0; l < LP; ++l) { S[l] = 0.0; M[l] = 0.0f; }
        auto fetch = [&](uint32_t c) {
            uint4 v = make_uint4(sent, sent, sent, sent);
            const uint32_t k = c * 128u + 4u * lane;
            const uint32_t *src = events + base + k;
            if (vec) {
                if (k < len) v = __ldcs(reinterpret_cast<const uint4 *>(src));
            } else {
                if (k < len) v.x = __ldcs(src);
                if (k + 1 < len) v.y = __ldcs(src + 1);
                if (k + 2 < len) v.z = __ldcs(src + 2);
                if (k + 3 < len) v.w = __ldcs(src + 3);
            }
            return v;
        };
        uint4 nxt = fetch(0);
        for (uint32_t c = 0; c * 128u < len; ++c) {
            const uint4 cur = nxt;
            if ((c + 1) * 128u < len) nxt = fetch(c + 1);
            const uint32_t k0 = c * 128u + 4u * lane;
            const uint32_t ee[4] = {cur.x, cur.y, cur.z, cur.w};
            float g[4][LP];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t bit = BM == 0 ? ee[q] : ee[q] >> shift;
                bool hit = __funnelshift_r(bitmap[bit >> 5], 0u, bit) & 1u;
                if (BM == 2) hit = hit && k0 + q < len;
                load_occ<LP>(hit, occ + (uint64_t)ee[q] * LP, g[q]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int l = 0; l < LP; ++l) {
                    S[l] += (double)g[q][l];               // line 12's trial sum, occurrence order per lane
                    if (OM) M[l] = fmaxf(M[l], g[q][l]);
                }
        }
        // fixed-tree warp sums -> aggregate terms (line 12, G6) -> YLT (line 17)
#pragma unroll
        for (int l = 0; l < LP; ++l) {
            double s = S[l];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            unsigned mb = 0;
            if (OM) mb = __reduce_max_sync(0xffffffffu, __float_as_uint(M[l]));
            if (lane == 0 && (uint32_t)l < nl) {
                const LayerInfo &L = A.pf.layers[l];
                A.ylt[(uint64_t)l * n_trials + t] = (float)clip64(s - L.agg_r, L.agg_l);
                if (OM) A.occ_max[(uint64_t)l * n_trials + t] = __uint_as_float(mb);
            }
        }
    }
}

cudaError_t launch_primary(const PrimaryArgs &A, cudaStream_t s, int num_sms) {
    const size_t smem = bitmap_smem_bytes(A.pf.bitmap_words);
    const int bm = !A.pf.sentinel_ok ? 2 : A.pf.bitmap_shift == 0 ? 0 : 1;
    using K = void (*)(PrimaryArgs);
    K kern = nullptr;
#define ARA_PK(LP)                                                                                             \
    (A.occ_max ? (bm == 0 ? (K)primary_kernel<LP, 0, true> : bm == 1 ? (K)primary_kernel<LP, 1, true>          \
                                                                     : (K)primary_kernel<LP, 2, true>)         \
               : (bm == 0 ? (K)primary_kernel<LP, 0, false> : bm == 1 ? (K)primary_kernel<LP, 1, false>        \
                                                                      : (K)primary_kernel<LP, 2, false>))
    switch (A.lp) {
        case 1: kern = ARA_PK(1); break;
        case 2: kern = ARA_PK(2); break;
        case 4: kern = ARA_PK(4); break;
        case 8: kern = ARA_PK(8); break;
        default: return cudaErrorInvalidValue;
    }
#undef ARA_PK
    int per_sm = 0;
    cudaError_t e = prepare_launch((const void *)kern, smem, kPrimaryWarps * 32, per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    kern<<<num_sms, kPrimaryWarps * 32, smem, s>>>(A);
    return cudaGetLastError();
}

}  // namespace ara
