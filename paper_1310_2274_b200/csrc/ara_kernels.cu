// ara_kernels.cu -- sm_100a kernels of the ARA hot path (arXiv 1310.2274):
// record preparation + quantile tables, the fused YET scan
// (Algorithm 1), and component kernels used by the row-level
// parity tests.
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"
#include "ara_sampler.cuh"

namespace ara {

// ---------------------------------------------------------------------------
// Record preparation (preprocessing stage), one thread per record, fp64:
// beta parameters with the sigma_beta cap (G9), degenerate records
// (G10), the steps-3/4 weights, and the record's quantile table
// lambda(v) = logit I^-1(Phi(v); a, b) at v = -8, -7.5, ..., 8 with its
// derivative.  The table is accepted only if the quintic Hermite interpolant
// (evaluated from the stored fp32 values, as the sampler will) matches an
// exact solve at every interval midpoint to (1-x)|dlambda| <= 1e-5 (10x
// inside the parity tolerance; typical table error is < 1e-8);
// otherwise the record is marked for the per-sample fp64 solve.
// ---------------------------------------------------------------------------
__device__ double quintic_mid64(float l0, float d0, float l1, float d1, double v0, double a, double b) {
    // the sampler's interpolant at t = 1/2, evaluated in fp64 on the fp32 table values
    auto s2 = [&](double lam, double d, double v) {
        const double x = 1.0 / (1.0 + exp(-lam)), y = 1.0 / (1.0 + exp(lam));
        return d * (-v - (a * y - b * x) * d);
    };
    const double H = kTabH;
    const double s0 = s2(l0, d0, v0), s1 = s2(l1, d1, v0 + H);
    // basis at t = 1/2: h01 = 1/2, h10 = 1/8 * 5/4... computed generically
    const double t = 0.5, omt = 0.5, t2 = t * t, t3 = t2 * t;
    const double h01 = t3 * (10.0 + t * (-15.0 + 6.0 * t));
    const double h10 = t * omt * omt * omt * (1.0 + 3.0 * t);
    const double h11 = -t3 * omt * (4.0 - 3.0 * t);
    const double h20 = 0.5 * t2 * omt * omt * omt, h21 = 0.5 * t3 * omt * omt;
    return l0 + h01 * ((double)l1 - l0) + h10 * H * d0 + h11 * H * d1 + h20 * H * H * s0 + h21 * H * H * s1;
}

__global__ void prep_records_kernel(const ara_record *__restrict__ raw, const uint32_t *__restrict__ src,
                                    uint64_t n, BetaRec *__restrict__ out, float *__restrict__ out_mu,
                                    float2 *__restrict__ nodes, unsigned int *n_exact) {
    const double LN_SQRT_2PI = 0.91893853320467274178;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const ara_record q = raw[src ? src[t] : t];
        const double mu = q.mean_loss, si = q.sigma_i, sc = q.sigma_c, mx = q.max_loss;
        out_mu[t] = q.mean_loss;
        BetaRec r;
        const double sigma = si + sc;                          // step 1
        if (sigma == 0.0 || mu == 0.0 || mu == mx) {           // G10
            r.a = 0.0f; r.b = 0.0f; r.wi = 0.0f; r.wc = 0.0f;
            r.scale = (sigma == 0.0) ? q.mean_loss : (mu == 0.0 ? 0.0f : q.max_loss);
            r.mu_l = 0.0f; r.sd_l = 0.0f; r.mode = kModeDegenerate;
            out[t] = r;
            // a constant table (lambda = 88, lambda' = 0): the split sampler's
            // quintic returns 88 exactly and 1 / (1 + 2^(-88 log2 e)) = 1 in fp32
            // (the power flushes to 0), so its loss is scale * 1 = the loss
            if (nodes)
                for (int j = 0; j < kTabNodes; ++j) nodes[t * kTabNodes + j] = make_float2(kTabDegenerate, 0.0f);
            continue;
        }
        const double mub = mu / mx, sb0 = sigma / mx;
        const double smax = sqrt(mub * (1.0 - mub));
        const double sb = (sb0 >= smax) ? smax * (1.0 - 1e-6) : sb0;
        const double kappa = (smax / sb) * (smax / sb) - 1.0;
        const double a = mub * kappa, b = (1.0 - mub) * kappa;
        const double wi = si / sigma, wc = sc / sigma;
        const double nr = sqrt(wi * wi + wc * wc);
        const double lnB = lgamma(a) + lgamma(b) - lgamma(a + b);
        const double mu_l = digamma_d(a) - digamma_d(b);
        r.a = (float)a; r.b = (float)b;
        r.wi = (float)(wi / nr); r.wc = (float)(wc / nr);
        r.scale = q.max_loss;
        r.mu_l = (float)mu_l;
        r.sd_l = (float)sqrt(trigamma_d(a) + trigamma_d(b));
        r.mode = kModeTable;
        if (nodes) {
            float2 tab[kTabNodes];
            double lam[kTabNodes], d1[kTabNodes], d2[kTabNodes];
            bool good = true;
            auto node = [&](int j, double guess) {
                const double v = kTabV0 + kTabH * j;
                bool ok;
                const double l = lambda_exact64(v, a, b, lnB, guess, ok);
                bool sok;
                const Tail64 e = tail64(l, v <= 0.0, a, b, lnB, sok);
                ok = ok && sok;
                const double lnd = -0.5 * v * v - LN_SQRT_2PI + lnB - a * e.lnx - b * e.lny;
                const double d = exp(lnd);
                lam[j] = l; d1[j] = d;
                d2[j] = d * (-v - (a * e.y - b * e.x) * d);
                if (!ok || !isfinite(l) || !isfinite(d) || !isfinite(d2[j]) || fabs(l) > 1e30 || d > 1e30)
                    good = false;
            };
            const int mid = kTabNodes / 2;
            node(mid, mu_l);
            for (int j = mid + 1; j < kTabNodes && good; ++j)
                node(j, lam[j - 1] + kTabH * d1[j - 1] + 0.5 * kTabH * kTabH * d2[j - 1]);
            for (int j = mid - 1; j >= 0 && good; --j)
                node(j, lam[j + 1] - kTabH * d1[j + 1] + 0.5 * kTabH * kTabH * d2[j + 1]);
            if (good) {
                for (int j = 0; j < kTabNodes; ++j) tab[j] = make_float2((float)lam[j], (float)d1[j]);
                for (int j = 0; j + 1 < kTabNodes && good; ++j) {
                    const double v0 = kTabV0 + kTabH * j;
                    const double li = quintic_mid64(tab[j].x, tab[j].y, tab[j + 1].x, tab[j + 1].y, v0,
                                                    (double)r.a, (double)r.b);
                    bool ok;
                    const double le = lambda_exact64(v0 + 0.5 * kTabH, a, b, lnB, li, ok);
                    const double x = 1.0 / (1.0 + exp(-le));
                    // loss = max_l x: only the relative error of x matters, and
                    // not at all once x < 1e-7 (fp32 cannot hold lambda ~ -100 to 1e-5)
                    if (!ok || !isfinite(li) || (x > 1e-7 && (1.0 - x) * fabs(li - le) > 1e-5)) good = false;
                }
            }
            if (good) {
                for (int j = 0; j < kTabNodes; ++j) nodes[t * kTabNodes + j] = tab[j];
            } else {
                r.mode = kModeExact;
                if (n_exact) atomicAdd(n_exact, 1u);
            }
        }
        out[t] = r;
    }
}

void launch_prep_records(const ara_record *raw, const uint32_t *src, uint64_t n, BetaRec *out,
                         float *out_mu, float2 *nodes, unsigned int *n_exact, cudaStream_t s) {
    if (n == 0) return;
    const int threads = 128;
    const uint64_t blocks = (n + threads - 1) / threads;
    prep_records_kernel<<<(unsigned)(blocks < 65535 * 16 ? blocks : 65535 * 16), threads, 0, s>>>(
        raw, src, n, out, out_mu, nodes, n_exact);
}

// ---------------------------------------------------------------------------
// The fused YET scan.  One warp owns one trial at a time (dynamic trial
// scheduler).  Per trial:
//   1. stream the event ids, 128 per warp-load (uint4 per lane, evict-first,
//      next chunk prefetched), test each against the shared-memory presence
//      bitmap and compact the hits (k, e) into a warp list;
//   2. per 64 hits, fetch the event-major index entries (L2-resident) with
//      all loads in flight, and enqueue every present (occurrence, slot) pair
//      into the warp's shared-memory queue, whole occurrences at a time;
//   3. when the queue is full (and at the end of the trial): sample all
//      queued pairs with all 32 lanes busy (Philox draws, steps 2-4, quantile
//      table), then reduce each (occurrence, layer) segment, apply the
//      occurrence terms and add to the trial's per-layer fp64 sum;
//   4. apply the aggregate terms -> YLT.
// All reductions are fixed trees / fixed orders: the YLT is a pure function
// of the inputs (bit-identical across runs and trial shardings).
// ---------------------------------------------------------------------------
#ifndef ARA_SCAN_WARPS
#define ARA_SCAN_WARPS 16
#endif
constexpr int kWarps = ARA_SCAN_WARPS;  // warps per CTA (1 CTA per SM)
constexpr int kQCap = 256;          // pair queue capacity per warp (>= ARA_MAX_SLOTS)
static_assert(kQCap >= ARA_MAX_SLOTS, "queue must hold one occurrence's pairs");

struct WarpBuf {
    uint2 q[kQCap];                 // {device record, (k << 8) | slot}
    float xs[kQCap];                // sampled loss per queued pair
    uint32_t seg[kQCap];            // (occurrence, layer) segments: start | len << 16 | layer << 24
};
// followed per warp by: double S[L]; unsigned long long hsh[L]; unsigned cnt[L]

struct ScanArgs {
    PortfolioDev pf;
    YetDev yet;
    uint64_t seed;
    uint32_t flags;
    float *ylt;
    uint32_t *dbg_count;
    uint64_t *dbg_hash;
    RunStatus *status;
    const uint32_t *trial_list;     // null: all trials
    uint64_t n_list;
    const unsigned int *n_list_dev; // non-null: the list length is read on the device (ARA_ASYNC)
    uint32_t *redo;                 // trials to re-run with the fp64 kernel
    float *occ_max;                 // null, or [n_layers][n_trials] largest occurrence loss (G29)
    const float *zp_sup;            // ARA_RNG_SUPPLIED: z_(Prog,E) [program][zp_stride]
    uint64_t zp_stride;
    const float *ze_sup;            // ARA_RNG_SUPPLIED: z_(E) per device record
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Dynamic shared memory of the scan kernel.  The out-of-line helpers address
// it through this symbol + byte offsets so every access compiles to LDS/STS.
extern __shared__ __align__(16) unsigned char scan_smem[];

// byte offsets of this warp's pieces and the block's tables in scan_smem
struct WarpMem {
    uint32_t buf, S, hsh, cnt, om, slots, layers;
};
__device__ __forceinline__ WarpBuf &wbuf(const WarpMem &M) { return *reinterpret_cast<WarpBuf *>(scan_smem + M.buf); }
__device__ __forceinline__ double *wS(const WarpMem &M) { return reinterpret_cast<double *>(scan_smem + M.S); }
__device__ __forceinline__ unsigned long long *whsh(const WarpMem &M) {
    return reinterpret_cast<unsigned long long *>(scan_smem + M.hsh);
}
__device__ __forceinline__ unsigned int *wcnt(const WarpMem &M) { return reinterpret_cast<unsigned int *>(scan_smem + M.cnt); }
// largest occurrence loss of the trial per layer (fp32 bits; losses are >= 0)
__device__ __forceinline__ unsigned int *wom(const WarpMem &M) { return reinterpret_cast<unsigned int *>(scan_smem + M.om); }
__device__ __forceinline__ const SlotInfo *wslots(const WarpMem &M) {
    return reinterpret_cast<const SlotInfo *>(scan_smem + M.slots);
}
__device__ __forceinline__ const LayerInfo *wlayers(const WarpMem &M) {
    return reinterpret_cast<const LayerInfo *>(scan_smem + M.layers);
}

// what the sampler needs from the launch arguments (passed by value into the
// out-of-line helpers so they read registers, not the param space)
struct SampleArgs {
    const BetaRec *recs;            // by input record
    TablePtr tables;                // by input record
    const float *rec_mu;            // by input record
    const SplitRec *srecs;          // per device record (.tab: its input record)
    const uint32_t *rec_orig;
    RunStatus *status;
    uint64_t seed;
    bool exact;
    uint32_t rng;                   // 0: reading G2; 1: ARA_RNG_RECORD; 2: ARA_RNG_OCCURRENCE; 3: ARA_RNG_SUPPLIED
    const float *zp_sup;            // rng 3: z_(Prog,E) per YET occurrence, [program][zp_stride]
    uint64_t zp_stride;
    const float *ze_sup;            // rng 3: z_(E) per device record
    uint64_t occ_base;              // rng 3: the current trial's first occurrence in the YET
};

// z_(E) of device record `rec` (XELT si.elt) at occurrence k of trial i (G2 and its alternatives)
__device__ __forceinline__ uint32_t draw_ze(const SampleArgs &G, const SlotInfo &si, uint32_t rec,
                                            uint32_t trial_g, uint32_t k) {
    if (G.rng == 1) return philox_lane0(__ldg(G.rec_orig + rec), si.elt, 0u, 6u, G.seed);
    if (G.rng == 2) return philox_lane0(trial_g, k, 0u, 7u, G.seed);
    return philox_lane0(trial_g, k, si.elt, 2u, G.seed);
}

// Sample every queued pair, reduce the (occurrence, layer) segments, apply the
// occurrence terms, add to the layer sums.  Out of line: a single copy of the
// sampler keeps the instruction working set in the I-cache.  Returns 1 if a
// table-less record was met (the trial must be redone).
template <bool SU, bool EX>
__device__ __noinline__ int flush_queue(const SampleArgs G, const WarpMem M, uint32_t trial_g, int lane,
                                        int qn, int nseg) {
    WarpBuf &B = wbuf(M);
    const SlotInfo *slots = wslots(M);
    int redo = 0;
    // sample, four pairs per lane in flight (Alg.1 lines 7-8): all record loads
    // first, then the draws, then the table loads, then the interpolation
    constexpr int U = 4;
    for (int p0 = lane; p0 < qn; p0 += 32 * U) {
        uint2 e[U];
        bool live[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            live[u] = p0 + 32 * u < qn;
            e[u] = B.q[live[u] ? p0 + 32 * u : p0];
        }
        if (SU) {
            BetaRec r[U];
#pragma unroll
            for (int u = 0; u < U; ++u) r[u] = G.recs[__ldg(&G.srecs[e[u].x].tab)];
            float v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const SlotInfo &si = slots[e[u].y & 0xffu];
                const uint32_t k = e[u].y >> 8;
                if (G.rng == 3) {                    // supplied with the inputs
                    const float zp = __ldg(G.zp_sup + (uint64_t)si.prog * G.zp_stride + G.occ_base + k);
                    v[u] = combine_v(r[u], norm_quantile_f(zp), norm_quantile_f(__ldg(G.ze_sup + e[u].x)));
                } else {
                    const uint32_t bp = philox_lane0(trial_g, k, si.prog, 1u, G.seed);   // z_(Prog,E)
                    const uint32_t be = draw_ze(G, si, e[u].x, trial_g, k);              // z_(E)
                    v[u] = combine_v(r[u], norm_quantile_from_bits(bp), norm_quantile_from_bits(be));
                }
            }
            float2 n0[U], n1[U];
            int ti[U];
            float tt[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {       // table rows
                const float uu = (fminf(fmaxf(v[u], kTabV0), -kTabV0) - kTabV0) * (1.0f / kTabH);
                ti[u] = min((int)uu, kTabNodes - 2);
                tt[u] = uu - (float)ti[u];
                const float2 *row = table_row(G.tables, __ldg(&G.srecs[e[u].x].tab), ti[u]);
                if (r[u].mode == kModeTable) { n0[u] = __ldg(row); n1[u] = __ldg(row + 1); }
                else { n0[u] = make_float2(0.f, 0.f); n1[u] = n0[u]; }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float x;
                if (r[u].mode == kModeDegenerate) {
                    x = r[u].scale;
                } else if (r[u].mode == kModeTable && !(EX && G.exact)) {
                    x = r[u].scale * sigmoidf_(quintic_from_nodes(n0[u], n1[u], ti[u], tt[u], r[u].a, r[u].b));
                } else if (!EX) {
                    x = 0.0f;               // table-less record: this trial is redone by the fp64 kernel
                    redo = 1;
                } else {
                    bool ok;
                    x = sample_exact64(r[u].a, r[u].b, r[u].mu_l, r[u].sd_l, r[u].scale, v[u], ok);
                    if (!ok) atomicAdd(&G.status->nonconverged, 1u);
                }
                const SlotInfo &si = slots[e[u].y & 0xffu];
                if (si.has_terms) x = si.share * fminf(fmaxf(x - si.ret, 0.0f), si.lim);
                if (live[u]) B.xs[p0 + 32 * u] = x;
            }
        } else {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                float x = __ldg(G.rec_mu + __ldg(&G.srecs[e[u].x].tab));
                const SlotInfo &si = slots[e[u].y & 0xffu];
                if (si.has_terms) x = si.share * fminf(fmaxf(x - si.ret, 0.0f), si.lim);
                if (live[u]) B.xs[p0 + 32 * u] = x;
            }
        }
    }
    __syncwarp();
    // segments = (occurrence, layer) runs recorded at enqueue: sum (line 9),
    // occurrence terms (line 11), add to the layer's trial sum
    const LayerInfo *layers = wlayers(M);
    double *S = wS(M);
    for (int base = 0; base < nseg; base += 32) {
        const int sidx = base + lane;
        const bool have = sidx < nseg;
        uint32_t layer = 0;
        double g = 0.0;
        if (have) {
            const uint32_t d = B.seg[sidx];
            const int st = (int)(d & 0xffffu), len = (int)((d >> 16) & 0xffu);
            layer = d >> 24;
            double l = 0.0;
            for (int r = 0; r < len; ++r) l += (double)B.xs[st + r];
            const LayerInfo &L = layers[layer];
            g = fmin(fmax(l - L.occ_r, 0.0), L.occ_l);
        }
        // deterministic per-layer reduction: one fixed-tree warp sum per
        // distinct layer among this round's segments
        unsigned pending = __ballot_sync(0xffffffffu, have);
        while (pending) {
            const int leader = __ffs(pending) - 1;
            const uint32_t lay = __shfl_sync(0xffffffffu, layer, leader);
            const bool mine = have && layer == lay;
            const double sum = warp_sum_f64(mine ? g : 0.0);
            const unsigned mb = __reduce_max_sync(0xffffffffu, mine ? __float_as_uint((float)g) : 0u);
            if (lane == 0) { S[lay] += sum; wom(M)[lay] = max(wom(M)[lay], mb); }
            pending &= ~__ballot_sync(0xffffffffu, mine);
        }
    }
    __syncwarp();
    return __any_sync(0xffffffffu, redo) ? 1 : 0;
}

// The present (occurrence, slot) pairs of one occurrence: the event's device
// records first .. first + count - 1 (event-major, slot order); their slot
// and layer from rec_meta.  count_occ: pairs and (occurrence, layer)
// segments; write_occ: enqueue them.
__device__ __forceinline__ void count_occ(const uint2 *mu_meta, uint32_t first, uint32_t count, uint32_t &np,
                                          uint32_t &ns) {
    np = count;
    ns = 0;
    for (uint32_t r = first; r < first + count; ++r) ns += (__ldg(&mu_meta[r].y) >> 8) & 1u;   // run ends
}

template <bool DBG>
__device__ __forceinline__ void write_occ(const SampleArgs &G, const WarpMem &M, WarpBuf &B,
                                          const SlotInfo *slots, const uint2 *mu_meta, uint32_t k,
                                          uint32_t first, uint32_t count, uint32_t pos, uint32_t spos) {
    uint32_t prev = 0xffffffffu, sstart = pos;
    for (uint32_t rec = first; rec < first + count; ++rec) {
        const uint32_t meta = __ldg(&mu_meta[rec].y);
        const uint32_t slot = meta & 0xffu, lay = (meta >> 16) & 63u;
        if (lay != prev) {
            if (prev != 0xffffffffu) B.seg[spos++] = sstart | ((pos - sstart) << 16) | (prev << 24);
            sstart = pos;
            prev = lay;
        }
        B.q[pos++] = make_uint2(rec, (k << 8) | slot);
        if (DBG) {
            atomicAdd(&wcnt(M)[lay], 1u);
            const uint64_t hv = splitmix64(splitmix64(splitmix64((uint64_t)k) ^ slots[slot].elt) ^ G.rec_orig[rec]);
            atomicAdd(&whsh(M)[lay], (unsigned long long)hv);
        }
    }
    if (prev != 0xffffffffu) B.seg[spos] = sstart | ((pos - sstart) << 16) | (prev << 24);
}

// Enqueue the present (occurrence, slot) pairs of a 128-event chunk: each
// lane holds <= 4 occurrences (index entries already loaded, Alg.1 line 6).
// One packed prefix sum (pairs low, segments high) places every pair and
// (occurrence, layer) segment; if the queue would overflow it is flushed
// first, and a chunk that alone exceeds the queue goes occurrence group by
// group.  q packs (qn, nseg, redo) as qn | nseg << 12 | redo << 24.
template <bool SU, bool EX, bool DBG>
__device__ __forceinline__ int enqueue_chunk(const SampleArgs G, const WarpMem M, uint32_t trial_g, int lane,
                                          int q, uint32_t k0, uint32_t hitbits,
                                          const uint4 first4, const uint4 count4, const uint2 *mu_meta) {
    WarpBuf &B = wbuf(M);
    const SlotInfo *slots = wslots(M);
    int qn = q & 0xfff, nseg = (q >> 12) & 0xfff, redo = q >> 24;
    const uint32_t first[4] = {first4.x, first4.y, first4.z, first4.w};
    const uint32_t count[4] = {count4.x, count4.y, count4.z, count4.w};
    uint32_t np[4], ns[4];
    uint32_t mine = 0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        np[h] = 0; ns[h] = 0;
        if ((hitbits >> h) & 1u) count_occ(mu_meta, first[h], count[h], np[h], ns[h]);
        mine += np[h] | (ns[h] << 16);
    }
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    if ((int)(tot & 0xffffu) > kQCap - qn && (int)(tot & 0xffffu) <= kQCap) {   // make room
        redo |= flush_queue<SU, EX>(G, M, trial_g, lane, qn, nseg);
        qn = 0; nseg = 0;
    }
    if ((int)(tot & 0xffffu) <= kQCap - qn) {                 // common case: the chunk fits
        const uint32_t ex = incl - mine;
        uint32_t pos = (uint32_t)qn + (ex & 0xffffu), spos = (uint32_t)nseg + (ex >> 16);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (np[h]) write_occ<DBG>(G, M, B, slots, mu_meta, k0 + h, first[h], count[h], pos, spos);
            pos += np[h];
            spos += ns[h];
        }
        qn += (int)(tot & 0xffffu);
        nseg += (int)(tot >> 16);
        __syncwarp();
        return qn | (nseg << 12) | (redo << 24);
    }
    // a chunk with more pairs than the queue: occurrence group by group
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        bool todo = np[h] > 0;
        while (__any_sync(0xffffffffu, todo)) {
            const uint32_t m2 = todo ? (np[h] | (ns[h] << 16)) : 0u;
            uint32_t inc2 = m2;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, inc2, o);
                if (lane >= o) inc2 += y;
            }
            const bool fits = todo && (inc2 & 0xffffu) <= (uint32_t)(kQCap - qn);
            if (fits) {
                const uint32_t ex = inc2 - m2;
                write_occ<DBG>(G, M, B, slots, mu_meta, k0 + h, first[h], count[h], (uint32_t)qn + (ex & 0xffffu),
                               (uint32_t)nseg + (ex >> 16));
                todo = false;
            }
            const unsigned fitmask = __ballot_sync(0xffffffffu, fits);
            if (fitmask) {
                const uint32_t last = __shfl_sync(0xffffffffu, inc2, 31 - __clz(fitmask));
                qn += (int)(last & 0xffffu);
                nseg += (int)(last >> 16);
            }
            __syncwarp();
            if (__any_sync(0xffffffffu, todo)) {
                redo |= flush_queue<SU, EX>(G, M, trial_g, lane, qn, nseg);
                qn = 0;
                nseg = 0;
            }
        }
    }
    return qn | (nseg << 12) | (redo << 24);
}

template <bool SU, bool EX, bool DBG>
__global__ void __launch_bounds__(kWarps * 32, 1) scan_kernel(const __grid_constant__ ScanArgs A) {
    const uint32_t nl = A.pf.n_layers;
    const uint32_t per_warp = (uint32_t)((sizeof(WarpBuf) + nl * (sizeof(double) + sizeof(unsigned long long) +
                                                                   2 * sizeof(unsigned int)) + 15) & ~size_t(15));
    const uint32_t off_slots = 0;
    const uint32_t off_layers = off_slots + sizeof(SlotInfo) * ARA_MAX_SLOTS;
    const uint32_t off_bitmap = off_layers + sizeof(LayerInfo) * ARA_MAX_LAYERS;
    const uint32_t off_warps = off_bitmap + (A.pf.bitmap_words * 4u + 15u) / 16u * 16u;
    SlotInfo *slots = reinterpret_cast<SlotInfo *>(scan_smem + off_slots);
    LayerInfo *layers = reinterpret_cast<LayerInfo *>(scan_smem + off_layers);
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(scan_smem + off_bitmap);
    if (A.trial_list && A.n_list_dev && *A.n_list_dev == 0) return;   // a device-sized pass with nothing to do

    for (uint32_t t = threadIdx.x; t < A.pf.bitmap_words; t += blockDim.x) bitmap[t] = A.pf.bitmap[t];
    for (uint32_t t = threadIdx.x; t < A.pf.n_slots; t += blockDim.x) slots[t] = A.pf.slots[t];
    for (uint32_t t = threadIdx.x; t < nl; t += blockDim.x) layers[t] = A.pf.layers[t];
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpMem M;
    M.buf = off_warps + per_warp * warp;
    M.S = M.buf + sizeof(WarpBuf);
    M.hsh = M.S + nl * sizeof(double);
    M.cnt = M.hsh + nl * sizeof(unsigned long long);
    M.om = M.cnt + nl * sizeof(unsigned int);
    M.slots = off_slots;
    M.layers = off_layers;
    WarpBuf &B = wbuf(M);
    double *S = wS(M);
    unsigned long long *hsh = whsh(M);
    unsigned int *cntv = wcnt(M);
    unsigned int *omv = wom(M);
    const bool dbg = DBG;
    SampleArgs G{A.pf.recs, A.pf.tables, A.pf.rec_mu, A.pf.srecs, A.pf.rec_orig, A.status, A.seed,
                 (A.flags & ARA_EXACT) != 0,
                 (A.flags & ARA_RNG_SUPPLIED) ? 3u : (A.flags & ARA_RNG_RECORD) ? 1u : (A.flags & ARA_RNG_OCCURRENCE) ? 2u : 0u,
                 A.zp_sup, A.zp_stride, A.ze_sup, 0};
    const uint64_t n_trials = A.yet.n_trials;
    const uint64_t n_work = A.trial_list ? (A.n_list_dev ? (uint64_t)*A.n_list_dev : A.n_list) : n_trials;
    const uint32_t C = A.pf.catalog, shift = A.pf.bitmap_shift;
    const uint2 *cidx = A.pf.cidx;
    const uint2 *mu_meta = A.pf.mu_meta;
    const unsigned lanemask_lt = (1u << lane) - 1u;

    while (true) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&A.status->next_trial, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n_work) break;
        if (A.trial_list) t = A.trial_list[t];
        const uint64_t base = A.yet.fixed_len ? t * (uint64_t)A.yet.fixed_len : A.yet.offsets[t];
        const uint32_t len = A.yet.fixed_len ? A.yet.fixed_len : (uint32_t)(A.yet.offsets[t + 1] - base);
        const uint32_t trial_g = (uint32_t)(A.yet.first_trial + t);        // global trial index i
        G.occ_base = base;
        for (uint32_t l = lane; l < nl; l += 32) { S[l] = 0.0; cntv[l] = 0u; hsh[l] = 0ull; omv[l] = 0u; }
        __syncwarp();
        int q = 0;                         // packed queue state (qn, nseg, redo)
        const uint32_t *ev = A.yet.events + base;
        const bool vec = (base & 3u) == 0;
        uint4 nxt = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
        {   // events c+4*lane .. +3 of chunk 0
            const uint32_t k = 4u * lane;
            if (vec && k + 3 < len) nxt = __ldcs(reinterpret_cast<const uint4 *>(ev + k));
            else {
                if (k < len) nxt.x = __ldcs(ev + k);
                if (k + 1 < len) nxt.y = __ldcs(ev + k + 1);
                if (k + 2 < len) nxt.z = __ldcs(ev + k + 2);
                if (k + 3 < len) nxt.w = __ldcs(ev + k + 3);
            }
        }
        // software pipeline over 128-event chunks: events of chunk c+2 in flight
        // (HBM), index entries of chunk c+1 in flight (L2), pairs of chunk c enqueued
        uint32_t hit_c = 0, k0_c = 0;
        uint4 first_c = make_uint4(0, 0, 0, 0), count_c = make_uint4(0, 0, 0, 0);
        for (uint32_t c = 0; c < len + 128; c += 128) {             // Alg.1 line 4
            uint32_t hit_n = 0, k0_n = c + 4u * lane;
            uint4 first_n = make_uint4(0, 0, 0, 0), count_n = make_uint4(0, 0, 0, 0);
            if (c < len) {
                const uint4 cur = nxt;
                {   // prefetch the next chunk's events
                    const uint32_t k = c + 128 + 4u * lane;
                    nxt = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
                    if (vec && k + 3 < len) nxt = __ldcs(reinterpret_cast<const uint4 *>(ev + k));
                    else if (k < len) {
                        nxt.x = __ldcs(ev + k);
                        if (k + 1 < len) nxt.y = __ldcs(ev + k + 1);
                        if (k + 2 < len) nxt.z = __ldcs(ev + k + 2);
                        if (k + 3 < len) nxt.w = __ldcs(ev + k + 3);
                    }
                }
                // presence bitmap (shared memory) for this lane's 4 occurrences
                const uint32_t ee[4] = {cur.x, cur.y, cur.z, cur.w};
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                    const uint32_t e = ee[qd];
                    if (k0_n + qd < len) {
                        if (e >= C) {
                            atomicAdd(&A.status->bad_event, 1u);
                        } else {
                            const uint32_t bit = e >> shift;
                            hit_n |= ((bitmap[bit >> 5] >> (bit & 31)) & 1u) << qd;
                        }
                    }
                }
                // index entries of this lane's hits: issued now, consumed next iteration
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                    uint2 ci = make_uint2(0u, 0u);
                    if ((hit_n >> qd) & 1u) ci = __ldg(cidx + ee[qd]);       // (first record, count)
                    if (qd == 0) { first_n.x = ci.x; count_n.x = ci.y; }
                    else if (qd == 1) { first_n.y = ci.x; count_n.y = ci.y; }
                    else if (qd == 2) { first_n.z = ci.x; count_n.z = ci.y; }
                    else { first_n.w = ci.x; count_n.w = ci.y; }
                }
            }
            if (__any_sync(0xffffffffu, hit_c != 0))
                q = enqueue_chunk<SU, EX, DBG>(G, M, trial_g, lane, q, k0_c, hit_c, first_c, count_c, mu_meta);
            hit_c = hit_n; k0_c = k0_n; first_c = first_n; count_c = count_n;
        }
        __syncwarp();
        int redo = q >> 24;
        if (q & 0xfff) redo |= flush_queue<SU, EX>(G, M, trial_g, lane, q & 0xfff, (q >> 12) & 0xfff);
        if (!EX && redo) {
            if (lane == 0) A.redo[atomicAdd(&A.status->n_redo, 1u)] = (uint32_t)t;
        }
        // aggregate terms on the trial sum (line 12, G6) -> YLT (line 17)
        for (uint32_t l = lane; l < nl; l += 32) {
            const LayerInfo &L = layers[l];
            A.ylt[(uint64_t)l * n_trials + t] = (float)fmin(fmax(S[l] - L.agg_r, 0.0), L.agg_l);
            if (A.occ_max) A.occ_max[(uint64_t)l * n_trials + t] = __uint_as_float(omv[l]);
            if (dbg) {
                if (A.dbg_count) A.dbg_count[(uint64_t)l * n_trials + t] = cntv[l];
                if (A.dbg_hash) A.dbg_hash[(uint64_t)l * n_trials + t] = hsh[l];
            }
        }
        __syncwarp();
    }
    (void)lanemask_lt;
}

static size_t scan_smem_bytes(const PortfolioDev &pf) {
    const size_t per_warp = (sizeof(WarpBuf) + pf.n_layers * (sizeof(double) + sizeof(unsigned long long) +
                                                              2 * sizeof(unsigned int)) + 15) & ~size_t(15);
    return sizeof(SlotInfo) * ARA_MAX_SLOTS + sizeof(LayerInfo) * ARA_MAX_LAYERS +
           ((size_t)pf.bitmap_words * 4 + 15) / 16 * 16 + kWarps * per_warp;
}

template <bool SU, bool EX>
static cudaError_t launch_scan_t(const ScanArgs &A, cudaStream_t s, int num_sms) {
    const size_t smem = scan_smem_bytes(A.pf);
    auto kern = (A.flags & ARA_DEBUG_LOOKUP) ? scan_kernel<SU, EX, true> : scan_kernel<SU, EX, false>;
    int per_sm = 0;
    cudaError_t err = prepare_launch((const void *)kern, smem, kWarps * 32, per_sm);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    kern<<<num_sms * per_sm, kWarps * 32, smem, s>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_scan(const PortfolioDev &pf, const YetDev &yet, uint64_t seed, uint32_t flags,
                        float *ylt, uint32_t *dbg_count, uint64_t *dbg_hash, RunStatus *status,
                        const uint32_t *trial_list, uint64_t n_list, uint32_t *redo, bool exact_kernel,
                        cudaStream_t s, int num_sms, float *occ_max, const float *zp_sup, uint64_t zp_stride,
                        const float *ze_sup, const unsigned int *n_list_dev) {
    ScanArgs A{pf, yet, seed, flags, ylt, dbg_count, dbg_hash, status, trial_list, n_list, n_list_dev, redo, occ_max,
               zp_sup, zp_stride, ze_sup};
    if (trial_list && n_list == 0 && !n_list_dev) return cudaSuccess;
    if (!(flags & ARA_SU)) return launch_scan_t<false, false>(A, s, num_sms);
    // the fp64 per-sample solve lives in a separate instantiation (its register
    // demand would otherwise throttle the table path)
    if (exact_kernel) return launch_scan_t<true, true>(A, s, num_sms);
    return launch_scan_t<true, false>(A, s, num_sms);
}

// ---------------------------------------------------------------------------
// Component kernels (row-level parity tests)
// ---------------------------------------------------------------------------
__global__ void sample_losses_kernel(const BetaRec *recs, TablePtr tables,
                                     const float *zp,
                                     const float *ze, uint64_t n, bool exact, float *out,
                                     RunStatus *status) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const BetaRec r = recs[t];
        const float v = combine_v(r, norm_quantile_f(zp[t]), norm_quantile_f(ze[t]));
        bool ok;
        out[t] = sample_loss_from_v<true>(r, tables, t, v, exact, ok);
        if (!ok) atomicAdd(&status->nonconverged, 1u);
    }
}

cudaError_t launch_sample_losses(const BetaRec *recs, TablePtr tables,
                                 const float *zp,
                                 const float *ze, uint64_t n, bool exact, float *out,
                                 RunStatus *status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + 255) / 256;
    sample_losses_kernel<<<(unsigned)(blocks < 1u << 20 ? blocks : 1u << 20), 256, 0, s>>>(
        recs, tables, zp, ze, n, exact, out, status);
    return cudaGetLastError();
}

// Row a6's fp64 solver alone (ara_beta_quantiles): x = I^-1(Phi(v); a, b)
// and y = 1 - x, both from lambda = logit x (full relative precision each)
__global__ void beta_quantiles_kernel(const double *a_, const double *b_, const double *v_, uint64_t n,
                                      double *x_out, double *y_out, RunStatus *status) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const double a = a_[t], b = b_[t], v = v_[t];
        const double lnB = lgamma(a) + lgamma(b) - lgamma(a + b);
        const double lam0 = (digamma_d(a) - digamma_d(b)) + v * sqrt(trigamma_d(a) + trigamma_d(b));
        bool ok;
        const double lam = lambda_exact64(v, a, b, lnB, lam0, ok);
        x_out[t] = 1.0 / (1.0 + exp(-lam));
        y_out[t] = 1.0 / (1.0 + exp(lam));
        if (!ok) atomicAdd(&status->nonconverged, 1u);
    }
}

cudaError_t launch_beta_quantiles(const double *a, const double *b, const double *v, uint64_t n, double *x_out,
                                  double *y_out, RunStatus *status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + 127) / 128;
    beta_quantiles_kernel<<<(unsigned)(blocks < 1u << 20 ? blocks : 1u << 20), 128, 0, s>>>(a, b, v, n, x_out,
                                                                                            y_out, status);
    return cudaGetLastError();
}

__global__ void draw_uniforms_kernel(uint64_t seed, const uint4 *ctr, uint64_t n, float *out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 c = ctr[t];
        out[t] = u01_from_bits(philox_lane0(c.x, c.y, c.z, c.w, seed));
    }
}

cudaError_t launch_draw_uniforms(uint64_t seed, const uint4 *ctr, uint64_t n, float *out,
                                 cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + 255) / 256;
    draw_uniforms_kernel<<<(unsigned)(blocks < 1u << 20 ? blocks : 1u << 20), 256, 0, s>>>(seed, ctr, n, out);
    return cudaGetLastError();
}

__global__ void normal_quantiles_kernel(const uint32_t *bits, uint64_t n, float *out) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x)
        out[t] = norm_quantile_from_bits(bits[t]);
}

cudaError_t launch_normal_quantiles(const uint32_t *bits, uint64_t n, float *out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + 255) / 256;
    normal_quantiles_kernel<<<(unsigned)(blocks < 1u << 20 ? blocks : 1u << 20), 256, 0, s>>>(bits, n, out);
    return cudaGetLastError();
}

}  // namespace ara
