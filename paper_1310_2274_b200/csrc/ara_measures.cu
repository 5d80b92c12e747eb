// ara_measures.cu -- PML / TVaR from the YLT on the device (reading
// G17 with SPEC's conventions S:345-387).  A 4-pass, 8-bit MSB-first radix
// select over order-preserving uint32 keys of the fp32 losses finds the
// threshold T = the K-th largest loss (K = the deepest rank any return
// period needs); the losses above T are compacted and bitonic-sorted in one
// CTA; ties at T are counted, never materialised.  PML interpolates the
// descending order statistics at r = (N+1)/RP; TVaR is the mean of all
// losses >= VaR = L(ceil(N/RP)).
#include <algorithm>
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_measures.cuh"

namespace ara {

constexpr int kMaxDevices = 64;

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t okey(float v) {
    const uint32_t b = __float_as_uint(v == 0.0f ? 0.0f : v);   // -0 -> +0
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// vals[t] for the requested layer, or the roll-up (sum over layers, G16),
// from a [n_shards][n_layers][per] layout.
__global__ void gather_kernel(const float *ylt, uint32_t n_layers, uint64_t per, uint32_t n_shards,
                              int32_t layer, float *vals) {
    const uint64_t n = per * n_shards;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = t / per, i = t - s * per;
        const float *base = ylt + s * (uint64_t)n_layers * per + i;
        float v;
        if (layer >= 0) {
            v = base[(uint64_t)layer * per];
        } else {
            v = 0.0f;
            for (uint32_t l = 0; l < n_layers; ++l) v += base[(uint64_t)l * per];
        }
        vals[t] = v;
    }
}

__global__ void hist_kernel(const float *vals, uint64_t n, const SelectState *st, int shift,
                            unsigned int *hist) {
    __shared__ unsigned int h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint32_t prefix = st->prefix, pmask = st->pmask;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = okey(vals[t]);
        if ((k & pmask) == prefix) atomicAdd(&h[(k >> shift) & 0xffu], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// pick the digit holding the K_rem-th largest key among those matching
__global__ void select_digit_kernel(SelectState *st, const unsigned int *hist, int shift) {
    if (threadIdx.x != 0) return;
    uint64_t need = st->k_rem;
    int d = 255;
    for (; d > 0; --d) {
        if (hist[d] >= need) break;
        need -= hist[d];
    }
    st->k_rem = need;
    st->prefix |= (uint32_t)d << shift;
    st->pmask |= 0xffu << shift;
}

// The whole select in one cooperative launch: gather (or roll-up) -> 4 radix
// passes (block histograms in shared memory, warp-aggregated with
// match.any -> one global histogram per pass -> every block picks the digit
// itself with a warp-parallel suffix count) -> tail compaction
// (warp-aggregated slots), with one grid-wide barrier per pass.
__device__ __forceinline__ void pick_digit(const unsigned int *hist, int shift, uint64_t &need,
                                           uint32_t &prefix, uint32_t &pmask) {
    // one warp: lane L holds digits 255 - 8L .. 248 - 8L (descending)
    const int lane = threadIdx.x & 31;
    uint32_t c[8], tot = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) { c[r] = __ldcg(&hist[255 - 8 * lane - r]); tot += c[r]; }
    uint64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint64_t before = incl - tot;               // keys in higher digits
    const unsigned hit = __ballot_sync(0xffffffffu, before < need && need <= incl);
    int d = 0;
    uint64_t rem = need;
    if (hit) {                                        // the lane holding the K_rem-th largest
        const int L = __ffs(hit) - 1;
        if (lane == L) {
            rem = need - before;
            d = 255 - 8 * lane;
#pragma unroll
            for (int r = 0; r < 7; ++r)
                if (rem > c[r]) { rem -= c[r]; --d; } else break;
        }
        d = __shfl_sync(0xffffffffu, d, L);
        rem = __shfl_sync(0xffffffffu, rem, L);
    } else {                                          // fewer keys than K: the lowest digit
        const uint64_t all = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t h0 = __shfl_sync(0xffffffffu, c[7], 31);
        rem = need - (all - h0);
    }
    need = rem;
    prefix |= (uint32_t)d << shift;
    pmask |= 0xffu << shift;
}

__global__ void __launch_bounds__(256) select_coop_kernel(const float *ylt, uint32_t n_layers, uint64_t per,
                                                          uint32_t n_shards, int32_t layer, float *vals,
                                                          uint64_t k_need, SelectState *st, unsigned int *hist4,
                                                          float *buf, uint32_t cap) {
    cg::grid_group grid = cg::this_grid();
    __shared__ unsigned int h[256];
    __shared__ uint64_t s_need;
    __shared__ uint32_t s_prefix, s_pmask;
    const uint64_t n = per * n_shards;
    const int lane = threadIdx.x & 31;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t wbase = gtid - lane;               // warp-uniform loop base
    if (gtid == 0) *st = SelectState{k_need, 0u, 0u, 0ull, 0ull};
    for (uint64_t i = gtid; i < 4 * 256; i += gstride) hist4[i] = 0u;
    uint64_t need = k_need;
    uint32_t prefix = 0u, pmask = 0u;
    grid.sync();
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        unsigned int *hist = hist4 + 256 * pass;
        for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
        __syncthreads();
        for (uint64_t b = wbase; b < n; b += gstride) {
            const uint64_t t = b + lane;
            float v = 0.0f;
            if (t < n) {
                if (pass == 0) {                      // gather / roll-up (G16)
                    const uint64_t sh = t / per, i = t - sh * per;
                    const float *base = ylt + sh * (uint64_t)n_layers * per + i;
                    if (layer >= 0) {
                        v = base[(uint64_t)layer * per];
                    } else {
                        for (uint32_t l = 0; l < n_layers; ++l) v += base[(uint64_t)l * per];
                    }
                    vals[t] = v;
                } else {
                    v = vals[t];
                }
            }
            const uint32_t k = okey(v);
            const uint32_t d = (t < n && (k & pmask) == prefix) ? (k >> shift) & 0xffu : 256u;
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            if (d < 256u && lane == __ffs(peers) - 1) atomicAdd(&h[d], (unsigned)__popc(peers));
        }
        __syncthreads();
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
            if (h[i]) atomicAdd(&hist[i], h[i]);
        grid.sync();
        if (threadIdx.x < 32) {                       // every block: the digit of the K_rem-th largest
            pick_digit(hist, shift, need, prefix, pmask);
            if (threadIdx.x == 0) { s_need = need; s_prefix = prefix; s_pmask = pmask; }
        }
        __syncthreads();
        need = s_need; prefix = s_prefix; pmask = s_pmask;
    }
    if (gtid == 0) { st->k_rem = need; st->prefix = prefix; st->pmask = pmask; }
    const uint32_t T = prefix;
    unsigned long long n_eq = 0;
    for (uint64_t b = wbase; b < n; b += gstride) {
        const uint64_t t = b + lane;
        const float v = t < n ? vals[t] : 0.0f;
        const uint32_t k = okey(v);
        const unsigned gt = __ballot_sync(0xffffffffu, t < n && k > T);
        n_eq += __popc(__ballot_sync(0xffffffffu, t < n && k == T));
        if (gt) {
            unsigned long long p0 = 0;
            if (lane == 0) p0 = atomicAdd(&st->n_gt, (unsigned long long)__popc(gt));
            p0 = __shfl_sync(0xffffffffu, p0, 0);
            if ((gt >> lane) & 1u) {
                const unsigned long long p = p0 + __popc(gt & ((1u << lane) - 1u));
                if (p < cap) buf[p] = v;
            }
        }
    }
    if (lane == 0 && n_eq) atomicAdd(&st->n_eq, n_eq);
}

// ---- every needed order statistic in one cooperative launch (n_rp <= 4) ----
// The host plans the ranks (PML's L(fl), L(fl+1), VaR = L(m) per return
// period, L(1), L(N); G13b); three radix passes (digits of 12, 10 and 10
// bits: one 4096-bin histogram for every rank, then 1024 bins per group of
// ranks that share a key prefix) select all of them at once, and a last pass
// forms the TVaR tail sums as int64 fixed-point sums (order-independent, so
// exact and deterministic under atomics).  No tail buffer, no sort, no rank
// limit (deep return periods take the same path).
#ifndef ARA_MULTI_THREADS
#define ARA_MULTI_THREADS 1024
#endif
constexpr int kMultiThreads = ARA_MULTI_THREADS;     // one block per SM: cheap grid barriers
constexpr uint32_t kMultiSmemWords = kMaxPlanRanks * 1024u;   // >= 4096 (pass 0)

struct __align__(8) MeasPlan {
    uint64_t rank[kMaxPlanRanks];                  // distinct ranks (1-based, descending order)
    uint64_t fl[4];
    double frac[4];
    int8_t i_one, i_n, i_fl[4], i_fl1[4], i_m[4];
    uint32_t nr, nq;
};

// one warp: the digit of the need-th largest key among a group's nb bins
// (nb = 1024 or 4096; global, complete after the pass's grid barrier) from the
// group's chunk sums (32 bins per chunk, summed by the blocks with their
// histograms): the lanes scan the chunk sums (nb/1024 per lane, descending),
// then the 32 bins of the chunk holding the rank (one per lane).  As
// pick_digit: a group with fewer than need keys takes the lowest digit.
__device__ __forceinline__ void pick_digit_2l(const unsigned int *gh, const unsigned int *gc, uint32_t nb,
                                              int shift, uint64_t &need, uint32_t &prefix) {
    const int lane = threadIdx.x & 31;
    const uint32_t nch = nb >> 5, k = nch >> 5;       // chunks; chunks per lane (4 or 1)
    const uint32_t top = nch - 1u - k * (uint32_t)lane;   // this lane's highest chunk
    uint32_t c[4], tot = 0;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        c[r] = (uint32_t)r < k ? __ldcg(&gc[top - (uint32_t)r]) : 0u;
        tot += c[r];
    }
    uint64_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint64_t before = incl - tot;               // keys in higher chunks
    const unsigned hit = __ballot_sync(0xffffffffu, before < need && need <= incl);
    uint32_t d = 0;
    uint64_t rem;
    if (hit) {
        const int L = __ffs(hit) - 1;
        uint32_t ch = 0;
        rem = need;
        if (lane == L) {                              // the chunk within the lane's k
            rem = need - before;
            ch = top;
#pragma unroll
            for (int r = 0; r < 3; ++r)
                if ((uint32_t)r + 1u < k && rem > c[r]) { rem -= c[r]; --ch; } else break;
        }
        ch = __shfl_sync(0xffffffffu, ch, L);
        rem = __shfl_sync(0xffffffffu, rem, L);       // 1 <= rem <= the chunk's keys
        const uint32_t bin = ch * 32u + 31u - (uint32_t)lane;   // lane 0: the chunk's highest bin
        const uint32_t cb = __ldcg(&gh[bin]);
        uint64_t incl2 = cb;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, incl2, o);
            if (lane >= o) incl2 += y;
        }
        const uint64_t before2 = incl2 - cb;
        const int L2 = __ffs(__ballot_sync(0xffffffffu, before2 < rem && rem <= incl2)) - 1;
        d = __shfl_sync(0xffffffffu, bin, L2);
        rem -= __shfl_sync(0xffffffffu, before2, L2);
    } else {                                          // fewer keys than need: the lowest digit
        const uint64_t all = __shfl_sync(0xffffffffu, incl, 31);
        rem = need - (all - __ldcg(&gh[0]));
    }
    need = rem;
    prefix |= d << shift;
}

__global__ void __launch_bounds__(kMultiThreads) select_multi_kernel(const float *ylt, uint32_t n_layers, uint64_t per,
                                                           uint32_t n_shards, int32_t layer, float *vals,
                                                           const __grid_constant__ MeasPlan M,
                                                           unsigned int *ghist, unsigned long long *gacc,
                                                           uint64_t n_total, double *out) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ unsigned int h[];               // kMultiSmemWords: a pass's block histograms
    __shared__ uint64_t s_need[kMaxPlanRanks];
    __shared__ uint32_t s_prefix[kMaxPlanRanks];
    __shared__ int s_grp[kMaxPlanRanks];
    __shared__ long long s_a[kMultiThreads / 32][4];
    __shared__ unsigned long long s_c[kMultiThreads / 32][4];
    const uint64_t n = per * n_shards;
    const int nr = (int)M.nr, nq = (int)M.nq;
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + tid, gstride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t wbase = gtid - lane;               // warp-uniform loop base
    // (ghist and gacc arrive zeroed: ara_ctx_create, then the end of every launch)
    if (tid < kMaxPlanRanks) { s_need[tid] = M.rank[tid]; s_prefix[tid] = 0u; }
    __syncthreads();
    uint32_t pmask = 0u;
    for (int pass = 0; pass < 3; ++pass) {             // digits of 12, 10, 10 bits
        const int width = pass == 0 ? 12 : 10, shift = pass == 0 ? 20 : pass == 1 ? 10 : 0;
        const uint32_t nb = 1u << width;
        const uint32_t ng = pass == 0 ? 1u : (uint32_t)nr;   // (pass 0: every rank in group 0)
        unsigned int *hist = ghist + (pass == 0 ? 0u : 4096u + (uint32_t)(pass - 1) * kMaxPlanRanks * 1024u);
        unsigned int *chist = ghist + kMultiBinWords + (pass == 0 ? 0u : 128u + (uint32_t)(pass - 1) * kMaxPlanRanks * 32u);
        if (tid < kMaxPlanRanks) {                     // group = first rank with the same prefix
            int g = (int)tid;
            for (int i = 0; i < (int)tid; ++i)
                if (s_prefix[i] == s_prefix[tid]) { g = i; break; }
            s_grp[tid] = g;
        }
        for (uint32_t i = tid; i < ng * nb; i += blockDim.x) h[i] = 0u;
        __syncthreads();
        uint32_t gp[kMaxPlanRanks];                    // group leaders' prefixes in registers
#pragma unroll
        for (int g = 0; g < kMaxPlanRanks; ++g) gp[g] = (g < nr && s_grp[g] == g) ? s_prefix[g] : 0xffffffffu;
        for (uint64_t b = wbase; b < n; b += gstride) {
            const uint64_t t = b + lane;
            uint32_t gd = 0xffffffffu;                 // (group, digit) of this element, or none
            if (t < n) {
                float v;
                if (pass == 0) {                       // gather / roll-up (G16)
                    const uint64_t sh = t / per, i = t - sh * per;
                    const float *base = ylt + sh * (uint64_t)n_layers * per + i;
                    if (layer >= 0) {
                        v = base[(uint64_t)layer * per];
                    } else {
                        v = 0.0f;
                        for (uint32_t l = 0; l < n_layers; ++l) v += base[(uint64_t)l * per];
                    }
                    vals[t] = v;
                } else {
                    v = vals[t];
                }
                const uint32_t k = okey(v), kp = k & pmask;
#pragma unroll
                for (int g = kMaxPlanRanks - 1; g >= 0; --g)   // groups are disjoint
                    if (kp == gp[g]) gd = (uint32_t)g << 12 | ((k >> shift) & (nb - 1u));
            }
            const unsigned peers = __match_any_sync(0xffffffffu, gd);
            if (gd != 0xffffffffu && lane == (uint32_t)(__ffs(peers) - 1))
                atomicAdd(&h[(gd >> 12) * nb + (gd & 0xfffu)], (unsigned)__popc(peers));
        }
        __syncthreads();
        for (uint32_t i = tid; i < ng * nb; i += blockDim.x)
            if (h[i]) atomicAdd(&hist[i], h[i]);
        for (uint32_t ci = tid; ci < ng * (nb >> 5); ci += blockDim.x) {   // chunk sums (32 bins; the
            uint32_t cs = 0;                                                 // rotated reads: distinct banks)
            for (uint32_t j = 0; j < 32u; ++j) cs += h[ci * 32u + ((j + ci) & 31u)];
            if (cs) atomicAdd(&chist[ci], cs);
        }
        grid.sync();
        for (int r = (int)warp; r < nr; r += (int)(blockDim.x >> 5)) {   // every block: its ranks' digits
            uint64_t need = s_need[r];
            uint32_t prefix = s_prefix[r];
            const uint32_t g = pass == 0 ? 0u : (uint32_t)s_grp[r];
            pick_digit_2l(hist + g * nb, chist + g * (nb >> 5), nb, shift, need, prefix);
            if (lane == 0) { s_need[r] = need; s_prefix[r] = prefix; }
        }
        pmask |= (nb - 1u) << shift;
        __syncthreads();
    }
    // TVaR tail sums: entries >= VaR (ties included), fixed point v * 2^E
    uint32_t vk[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) vk[q] = q < nq ? s_prefix[M.i_m[q]] : 0xffffffffu;
    const float vmax = fmaxf(fabsf(okey_inv(s_prefix[M.i_one])), fabsf(okey_inv(s_prefix[M.i_n])));
    int ex = 0;
    frexpf(vmax > 0.0f && vmax < INFINITY ? vmax : 1.0f, &ex);   // |v| < 2^ex
    const int lg = 64 - __clzll((long long)(n + 1));             // n + 1 <= 2^lg
    const double scale = ldexp(1.0, 62 - ex - lg);
    long long a[4] = {0, 0, 0, 0};
    unsigned long long c[4] = {0, 0, 0, 0};
    for (uint64_t t = gtid; t < n; t += gstride) {
        const float v = vals[t];
        const uint32_t k = okey(v);
        const long long fx = __double2ll_rn((double)v * scale);  // exact scaling by a power of 2
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < nq && k >= vk[q]) { a[q] += fx; ++c[q]; }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a[q] += __shfl_xor_sync(0xffffffffu, a[q], o);
            c[q] += __shfl_xor_sync(0xffffffffu, c[q], o);
        }
        if (lane == 0) { s_a[warp][q] = a[q]; s_c[warp][q] = c[q]; }
    }
    __syncthreads();
    if (tid < (uint32_t)nq) {
        long long sa = 0;
        unsigned long long sc = 0;
        for (uint32_t w = 0; w < (blockDim.x >> 5); ++w) { sa += s_a[w][tid]; sc += s_c[w][tid]; }
        if (sa) atomicAdd(&gacc[tid], (unsigned long long)sa);     // two's complement: signed sums
        if (sc) atomicAdd(&gacc[4 + tid], sc);
    }
    grid.sync();
    // every block is past its last histogram read: zero them for the next launch
    for (uint64_t i = gtid; i < kMultiHistWords; i += gstride) ghist[i] = 0u;
    if (blockIdx.x == 0 && tid < (uint32_t)nq) {
        const int q = (int)tid;
        auto L = [&](int i) -> double { return (double)okey_inv(s_prefix[i]); };
        const uint64_t fl = M.fl[q], N = n_total;
        const double frac = M.frac[q];
        double pml;
        if (fl < 1 || (fl == 1 && frac == 0.0)) pml = L(M.i_one);
        else if (fl >= N) pml = L(M.i_n);
        else pml = L(M.i_fl[q]) + frac * (L(M.i_fl1[q]) - L(M.i_fl[q]));
        const double sum = (double)(long long)__ldcg(&gacc[q]) / scale;
        out[3 * q] = pml;
        out[3 * q + 1] = sum / (double)__ldcg(&gacc[4 + q]);
        out[3 * q + 2] = L(M.i_m[q]);
    }
    if (blockIdx.x == 0) {                            // (block 0 alone read the tail sums)
        __syncthreads();
        if (tid < 8) gacc[tid] = 0ull;
    }
}

cudaError_t launch_measures_multi(const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                                  int32_t layer, const double *rps, uint32_t n_rp, MeasuresScratch &S,
                                  double *d_out, cudaStream_t s) {
    MeasPlan M{};
    const uint64_t N = n_total;
    auto idx = [&](uint64_t r) -> int8_t {            // index of rank r in the plan (added if new)
        if (r < 1) r = 1;
        if (r > N) r = N;
        for (uint32_t i = 0; i < M.nr; ++i) if (M.rank[i] == r) return (int8_t)i;
        M.rank[M.nr] = r;
        return (int8_t)M.nr++;
    };
    M.i_one = idx(1);
    M.i_n = idx(N);
    for (uint32_t q = 0; q < n_rp; ++q) {             // (G13b; as sort_measures_kernel)
        const double rp = rps[q];
        uint64_t fl, m;
        double frac;
        if (rp == floor(rp) && rp < 1.8e19) {
            const uint64_t R = (uint64_t)rp;
            fl = (N + 1) / R; frac = (double)((N + 1) % R) / rp; m = (N + R - 1) / R;
        } else {
            const double r = (double)(N + 1) / rp;
            fl = (uint64_t)floor(r); frac = r - (double)fl;
            const uint64_t a = (uint64_t)floor((1.0 - 1.0 / rp) * (double)N) + 1;
            m = N - (a < N ? a : N) + 1;
        }
        if (m < 1) m = 1;
        if (m > N) m = N;
        M.fl[q] = fl; M.frac[q] = frac;
        M.i_fl[q] = idx(fl); M.i_fl1[q] = idx(fl + 1); M.i_m[q] = idx(m);
    }
    M.nq = n_rp;
    static int blocks_by_dev[kMaxDevices] = {};      // co-resident blocks of the cooperative launch, per device
    int dev = 0;
    cudaGetDevice(&dev);
    int &blocks = blocks_by_dev[dev % kMaxDevices];
    if (!blocks) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(select_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kMultiSmemWords * sizeof(unsigned int)));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_multi_kernel, kMultiThreads,
                                                      kMultiSmemWords * sizeof(unsigned int));
        blocks = sms * std::min(per_sm, 1);           // one block per SM (0 if it cannot be resident)
        if (!blocks) return cudaErrorCooperativeLaunchTooLarge;
    }
    const uint64_t per = n_total / n_shards;
    float *vals = S.vals;
    unsigned int *hist = S.mhist;
    unsigned long long *acc = S.macc;
    uint64_t nt = n_total;
    void *args[] = {(void *)&ylt, (void *)&n_layers, (void *)&per, (void *)&n_shards, (void *)&layer,
                    (void *)&vals, (void *)&M, (void *)&hist, (void *)&acc, (void *)&nt, (void *)&d_out};
    return cudaLaunchCooperativeKernel((void *)select_multi_kernel, dim3(blocks), dim3(kMultiThreads), args,
                                       kMultiSmemWords * sizeof(unsigned int), s);
}

// one CTA of 1024 threads: bitonic sort (descending) of P = 1024 E values,
// then the measures.  Thread t holds elements t E .. t E + E - 1 in registers:
// a compare-exchange partner at distance j < E is in the same thread, at
// E <= j < 32 E in the same warp (shuffle), and only j >= 32 E goes through
// shared memory (stored transposed, [r][t], so the exchange is conflict-free).
template <int E>
__global__ void __launch_bounds__(1024) sort_measures_kernel(const float *buf, SelectState *st,
                                                             const __grid_constant__ RpList R, uint32_t n_rp,
                                                             uint64_t n_total, double *out) {
    const double *rps = R.v;                          // (kernel parameter: no host->device copy)
    extern __shared__ float sv[];
    constexpr uint32_t P = 1024u * E;
    const uint32_t ng = (uint32_t)st->n_gt;
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    float v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const uint32_t i = tid * E + r;
        v[r] = i < ng ? buf[i] : -INFINITY;
    }
    auto keep = [](bool lower_desc, float a, float b) {   // value kept by the element
        return lower_desc ? fmaxf(a, b) : fminf(a, b);
    };
    for (uint32_t k = 2; k <= P; k <<= 1) {
        uint32_t j = k >> 1;
        for (; j >= 32u * E; j >>= 1) {               // across warps: shared memory
            __syncthreads();
#pragma unroll
            for (int r = 0; r < E; ++r) sv[r * 1024 + tid] = v[r];
            __syncthreads();
            const uint32_t m = j / E;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const uint32_t i = tid * E + r;
                const float w = sv[r * 1024 + (tid ^ m)];
                v[r] = keep(((i & k) == 0) == ((tid & m) == 0), v[r], w);
            }
        }
        for (; j >= (uint32_t)E; j >>= 1) {           // across lanes: shuffles
            const uint32_t m = j / E;
#pragma unroll
            for (int r = 0; r < E; ++r) {
                const uint32_t i = tid * E + r;
                const float w = __shfl_xor_sync(0xffffffffu, v[r], m);
                v[r] = keep(((i & k) == 0) == ((lane & m) == 0), v[r], w);
            }
        }
#pragma unroll
        for (int jj = E / 2; jj >= 1; jj >>= 1) {     // within the thread: registers
            if ((uint32_t)jj < k) {
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    if ((r & jj) == 0) {
                        const uint32_t i = tid * E + r;
                        const float a = v[r], b = v[r + jj];
                        const bool desc = (i & k) == 0;
                        v[r] = desc ? fmaxf(a, b) : fminf(a, b);
                        v[r + jj] = desc ? fminf(a, b) : fmaxf(a, b);
                    }
                }
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < E; ++r) sv[tid * E + r] = v[r];
    __syncthreads();
    const float T = okey_inv(st->prefix);
    const uint64_t neq = st->n_eq, N = n_total;
    auto L = [&](uint64_t r) -> double {         // descending order statistic, 1-based
        return r <= ng ? (double)sv[r - 1] : (double)T;
    };
    __shared__ double red_s[1024];
    __shared__ unsigned int red_c[1024];
    for (uint32_t q = 0; q < n_rp; ++q) {
        const double rp = rps[q];
        uint64_t fl, m;
        double frac;
        if (rp == floor(rp) && rp < 1.8e19) {
            const uint64_t R = (uint64_t)rp;
            fl = (N + 1) / R;
            frac = (double)((N + 1) % R) / rp;
            m = (N + R - 1) / R;
        } else {
            const double r = (double)(N + 1) / rp;
            fl = (uint64_t)floor(r);
            frac = r - (double)fl;
            const uint64_t a = (uint64_t)floor((1.0 - 1.0 / rp) * (double)N) + 1;
            m = N - (a < N ? a : N) + 1;
        }
        if (m < 1) m = 1;
        if (m > N) m = N;
        const double var = L(m);
        // tail sum over the sorted values >= VaR: fixed per-thread strides and a
        // fixed tree, so the result does not depend on timing
        double acc = 0.0;
        unsigned int cnt = 0;
        for (uint32_t i = threadIdx.x; i < ng; i += blockDim.x)
            if ((double)sv[i] >= var) { acc += (double)sv[i]; ++cnt; }
        red_s[threadIdx.x] = acc;
        red_c[threadIdx.x] = cnt;
        __syncthreads();
        for (uint32_t o = blockDim.x / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) {
                red_s[threadIdx.x] += red_s[threadIdx.x + o];
                red_c[threadIdx.x] += red_c[threadIdx.x + o];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            double pml;
            if (fl < 1 || (fl == 1 && frac == 0.0)) pml = L(1);
            else if (fl >= N) pml = L(N);
            else pml = L(fl) + frac * (L(fl + 1) - L(fl));
            double sum = red_s[0];
            uint64_t c = red_c[0];
            if (var == (double)T) { sum += (double)neq * (double)T; c += neq; }
            out[3 * q] = pml;
            out[3 * q + 1] = sum / (double)c;
            out[3 * q + 2] = var;
        }
        __syncthreads();
    }
}

// ---- deep ranks (K > kSortCap): one radix select per needed rank ----------
__global__ void tail_sum_kernel(const float *vals, uint64_t n, const SelectState *st, double *part_sum,
                                unsigned long long *part_cnt) {
    __shared__ double ss[256];
    __shared__ unsigned long long sc[256];
    const uint32_t T = st->prefix;                // key of VaR
    double acc = 0.0;
    unsigned long long c = 0;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const float v = vals[t];
        if (okey(v) >= T) { acc += (double)v; ++c; }
    }
    ss[threadIdx.x] = acc; sc[threadIdx.x] = c;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) { ss[threadIdx.x] += ss[threadIdx.x + o]; sc[threadIdx.x] += sc[threadIdx.x + o]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { part_sum[blockIdx.x] = ss[0]; part_cnt[blockIdx.x] = sc[0]; }
}

struct DeepRp { uint64_t fl, m; double frac; };

__global__ void deep_final_kernel(const SelectState *states, const DeepRp *q, uint32_t rp_index,
                                  uint64_t N, const double *part_sum, const unsigned long long *part_cnt,
                                  int nblocks, double *out) {
    if (threadIdx.x != 0) return;
    const SelectState *st = states + 3 * rp_index;
    const double L1 = okey_inv(st[0].prefix), L2 = okey_inv(st[1].prefix);   // L(fl), L(fl+1)
    const DeepRp r = q[rp_index];
    double pml;
    if (r.fl < 1 || (r.fl == 1 && r.frac == 0.0)) pml = L1;                   // rank clamped to 1
    else if (r.fl >= N) pml = L1;                                             // rank clamped to N
    else pml = L1 + r.frac * (L2 - L1);
    double sum = 0.0;
    unsigned long long cnt = 0;
    for (int b = 0; b < nblocks; ++b) { sum += part_sum[b]; cnt += part_cnt[b]; }
    out[3 * rp_index] = pml;
    out[3 * rp_index + 1] = sum / (double)cnt;
    out[3 * rp_index + 2] = okey_inv(st[2].prefix);                          // VaR = L(m)
}

static cudaError_t select_rank(const float *vals, uint64_t n, SelectState *st, unsigned int *hist,
                               cudaStream_t s) {
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        cudaError_t e = cudaMemsetAsync(hist, 0, 256 * sizeof(unsigned int), s);
        if (e != cudaSuccess) return e;
        hist_kernel<<<148 * 4, 256, 0, s>>>(vals, n, st, shift, hist);
        select_digit_kernel<<<1, 32, 0, s>>>(st, hist, shift);
    }
    return cudaGetLastError();
}

cudaError_t launch_measures_deep(const float *ylt, uint32_t n_layers, uint64_t n_total,
                                 uint32_t n_shards, int32_t layer, const double *rps, uint32_t n_rp,
                                 MeasuresScratch &S, double *d_out, cudaStream_t s) {
    const uint64_t per = n_total / n_shards, N = n_total;
    gather_kernel<<<148 * 4, 256, 0, s>>>(ylt, n_layers, per, n_shards, layer, S.vals);
    static thread_local SelectState init[kMaxRanks];
    static thread_local DeepRp q[64];
    for (uint32_t i = 0; i < n_rp; ++i) {
        const double rp = rps[i];
        uint64_t fl, m;
        double frac;
        if (rp == floor(rp) && rp < 1.8e19) {
            const uint64_t R = (uint64_t)rp;
            fl = (N + 1) / R; frac = (double)((N + 1) % R) / rp; m = (N + R - 1) / R;
        } else {
            const double r = (double)(N + 1) / rp;
            fl = (uint64_t)floor(r); frac = r - (double)fl;
            const uint64_t a = (uint64_t)floor((1.0 - 1.0 / rp) * (double)N) + 1;
            m = N - (a < N ? a : N) + 1;
        }
        if (m < 1) m = 1;
        if (m > N) m = N;
        q[i] = {fl, m, frac};
        const uint64_t r0 = fl < 1 ? 1 : (fl > N ? N : fl);
        const uint64_t r1 = fl + 1 > N ? N : fl + 1;
        init[3 * i] = SelectState{r0, 0u, 0u, 0ull, 0ull};
        init[3 * i + 1] = SelectState{r1, 0u, 0u, 0ull, 0ull};
        init[3 * i + 2] = SelectState{m, 0u, 0u, 0ull, 0ull};
    }
    cudaError_t e = cudaMemcpyAsync(S.states, init, 3 * n_rp * sizeof(SelectState),
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    DeepRp *d_q = reinterpret_cast<DeepRp *>(S.buf);          // reuse the tail buffer
    e = cudaMemcpyAsync(d_q, q, n_rp * sizeof(DeepRp), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    for (uint32_t i = 0; i < 3 * n_rp; ++i) {
        e = select_rank(S.vals, N, S.states + i, S.hist, s);
        if (e != cudaSuccess) return e;
    }
    for (uint32_t i = 0; i < n_rp; ++i) {
        tail_sum_kernel<<<kRedBlocks, 256, 0, s>>>(S.vals, N, S.states + 3 * i + 2, S.part_sum, S.part_cnt);
        deep_final_kernel<<<1, 32, 0, s>>>(S.states, d_q, i, N, S.part_sum, S.part_cnt, kRedBlocks, d_out);
    }
    e = cudaStreamSynchronize(s);          // host staging arrays are reused next call
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_measures(const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                            int32_t layer, const RpList &rps, uint32_t n_rp, uint64_t k_need,
                            MeasuresScratch &S, double *d_out, cudaStream_t s) {
    const uint64_t per = n_total / n_shards;
    {
        static int coop_by_dev[kMaxDevices] = {};    // co-resident blocks of the cooperative select, per device
        int dev = 0;
        cudaGetDevice(&dev);
        int &coop_blocks = coop_by_dev[dev % kMaxDevices];
        if (!coop_blocks) {
            int sms = 0, per_sm = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_coop_kernel, 256, 0);
            coop_blocks = sms * std::min(per_sm, 4);
            if (!coop_blocks) return cudaErrorCooperativeLaunchTooLarge;
        }
        float *vals = S.vals, *buf = S.buf;
        unsigned int *hist = S.hist;
        SelectState *st = S.state;
        uint32_t cap = kSortCap;
        uint64_t kk = k_need;
        void *args[] = {(void *)&ylt, (void *)&n_layers, (void *)&per, (void *)&n_shards, (void *)&layer,
                        (void *)&vals, (void *)&kk, (void *)&st, (void *)&hist, (void *)&buf, (void *)&cap};
        cudaError_t e = cudaLaunchCooperativeKernel((void *)select_coop_kernel, dim3(coop_blocks), dim3(256), args,
                                                    0, s);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaSuccess;
    uint32_t P = 1024;
    while (P < k_need) P <<= 1;
    using K = void (*)(const float *, SelectState *, const RpList, uint32_t, uint64_t, double *);
    const K kern = P <= 1024 ? (K)sort_measures_kernel<1> : P <= 2048 ? (K)sort_measures_kernel<2>
                 : P <= 4096 ? (K)sort_measures_kernel<4> : P <= 8192 ? (K)sort_measures_kernel<8>
                 : P <= 16384 ? (K)sort_measures_kernel<16> : (K)sort_measures_kernel<32>;
    const size_t smem = sizeof(float) * P;
    static bool attr_by_dev[kMaxDevices] = {};       // once per device (all six instantiations)
    int dev = 0;
    cudaGetDevice(&dev);
    bool &attr_set = attr_by_dev[dev % kMaxDevices];
    if (!attr_set) {
        const K all[] = {sort_measures_kernel<1>, sort_measures_kernel<2>, sort_measures_kernel<4>,
                         sort_measures_kernel<8>, sort_measures_kernel<16>, sort_measures_kernel<32>};
        for (K k : all) {
            e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(float) * kSortCap));
            if (e != cudaSuccess) return e;
        }
        attr_set = true;
    }
    kern<<<1, 1024, smem, s>>>(S.buf, S.state, rps, n_rp, n_total, d_out);
    return cudaGetLastError();
}

}  // namespace ara

// ---------------------------------------------------------------------------
// Exceedance curve (SPEC's ExceedanceCurve): the
// YLT (one layer or the roll-up) sorted descending, L(1) >= ... >= L(N), whose
// empirical exceedance probability at rank i is i/(N+1).  A stable LSD radix
// sort of 32-bit keys ~okey(v) (ascending keys = descending losses), four
// 8-bit passes; each pass: per-tile digit counts -> one exclusive scan in
// digit-major order -> a stable scatter (tiles in order; inside a tile,
// chunks of 1024 in order, warps in order, lanes in order via match.any).
// ---------------------------------------------------------------------------
namespace ara {

constexpr int kEpThreads = 1024;

__global__ void ep_keys_kernel(const float *ylt, uint32_t n_layers, uint64_t per, uint32_t n_shards, int32_t layer,
                               uint32_t *keys) {
    const uint64_t n = per * n_shards;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t sh = t / per, i = t - sh * per;
        const float *base = ylt + sh * (uint64_t)n_layers * per + i;
        float v;
        if (layer >= 0) {
            v = base[(uint64_t)layer * per];
        } else {
            v = 0.0f;
            for (uint32_t l = 0; l < n_layers; ++l) v += base[(uint64_t)l * per];
        }
        keys[t] = ~okey(v);
    }
}

__global__ void __launch_bounds__(kEpThreads) ep_count_kernel(const uint32_t *keys, uint64_t n, uint64_t tile,
                                                              int shift, uint32_t *counts) {
    __shared__ unsigned int h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const uint64_t b0 = blockIdx.x * tile, b1 = min(n, b0 + tile);
    for (uint64_t t = b0 + threadIdx.x; t < b1; t += blockDim.x) atomicAdd(&h[(keys[t] >> shift) & 0xffu], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += blockDim.x) counts[(uint64_t)d * gridDim.x + blockIdx.x] = h[d];
}

// exclusive scan of counts[256 * nb] in place (digit-major), one block
__global__ void __launch_bounds__(kEpThreads) ep_scan_kernel(uint32_t *counts, uint32_t total) {
    __shared__ uint32_t part[kEpThreads];
    const uint32_t per = (total + blockDim.x - 1) / blockDim.x;
    const uint32_t a = threadIdx.x * per, b = min(total, a + per);
    uint32_t s = 0;
    for (uint32_t i = a; i < b; ++i) s += counts[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (uint32_t o = 1; o < blockDim.x; o <<= 1) {        // inclusive scan of the parts
        const uint32_t v = threadIdx.x >= o ? part[threadIdx.x - o] : 0u;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0u;
    for (uint32_t i = a; i < b; ++i) { const uint32_t c = counts[i]; counts[i] = run; run += c; }
}

__global__ void __launch_bounds__(kEpThreads) ep_scatter_kernel(const uint32_t *in, uint32_t *out, uint64_t n,
                                                                uint64_t tile, int shift, const uint32_t *offs) {
    __shared__ uint32_t base[256];                // next output slot of each digit for this tile
    __shared__ uint32_t wc[kEpThreads / 32][256];  // per-warp digit counts -> exclusive prefixes
    __shared__ uint32_t tot[256];                 // the chunk's digit totals
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < 256; d += blockDim.x) base[d] = offs[(uint64_t)d * gridDim.x + blockIdx.x];
    const uint64_t b0 = blockIdx.x * tile, b1 = min(n, b0 + tile);
    for (uint64_t c = b0; c < b1; c += blockDim.x) {
        for (int i = threadIdx.x; i < (kEpThreads / 32) * 256; i += blockDim.x) (&wc[0][0])[i] = 0u;
        __syncthreads();
        const uint64_t t = c + threadIdx.x;
        const bool live = t < b1;
        const uint32_t k = live ? in[t] : 0u;
        const uint32_t d = live ? (k >> shift) & 0xffu : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));        // earlier lanes, same digit
        if (live && rank == 0) wc[warp][d] = __popc(peers);
        __syncthreads();
        if (threadIdx.x < 256) {                  // digit: exclusive prefix over the warps, in order
            uint32_t sum = 0;
            for (int w = 0; w < kEpThreads / 32; ++w) { const uint32_t v = wc[w][threadIdx.x]; wc[w][threadIdx.x] = sum; sum += v; }
            tot[threadIdx.x] = sum;
        }
        __syncthreads();
        if (live) out[base[d] + wc[warp][d] + rank] = k;
        __syncthreads();
        if (threadIdx.x < 256) base[threadIdx.x] += tot[threadIdx.x];
    }
}

__global__ void ep_values_kernel(const uint32_t *keys, uint64_t n, float *out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x)
        out[t] = okey_inv(~keys[t]);
}

cudaError_t launch_exceedance_curve(const float *ylt, uint32_t n_layers, uint64_t n_total, uint32_t n_shards,
                                    int32_t layer, uint32_t *scratch /*[2 n + 256 nb]*/, float *out,
                                    cudaStream_t s, int num_sms) {
    const uint64_t per = n_total / n_shards, n = n_total;
    const uint32_t nb = (uint32_t)std::min<uint64_t>((uint64_t)num_sms * 2, (n + kEpThreads - 1) / kEpThreads);
    const uint64_t tile = (n + nb - 1) / nb;
    uint32_t *a = scratch, *b = scratch + n, *counts = scratch + 2 * n;
    ep_keys_kernel<<<num_sms * 4, 256, 0, s>>>(ylt, n_layers, per, n_shards, layer, a);
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 8 * pass;
        ep_count_kernel<<<nb, kEpThreads, 0, s>>>(a, n, tile, shift, counts);
        ep_scan_kernel<<<1, kEpThreads, 0, s>>>(counts, 256u * nb);
        ep_scatter_kernel<<<nb, kEpThreads, 0, s>>>(a, b, n, tile, shift, counts);
        std::swap(a, b);
    }
    ep_values_kernel<<<num_sms * 4, 256, 0, s>>>(a, n, out);     // (4 passes: the keys are back in `scratch`)
    return cudaGetLastError();
}

}  // namespace ara
