// ara_kernels.cu -- sm_100a kernels of the ARA hot path (arXiv 1310.2274):
// record preparation, the fused YET scan (Algorithm 1,
// P:134-170), and component kernels used by the row-level parity tests.
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"
#include "ara_sampler.cuh"

namespace ara {

// ---------------------------------------------------------------------------
// Record preparation (preprocessing stage): beta parameters with the
// sigma_beta cap (G9), degenerate records (G10), sampler constants.
// fp64 on the device, stored fp32.
// ---------------------------------------------------------------------------
__device__ double digamma_d(double x) {
    double r = 0.0;
    while (x < 6.0) { r -= 1.0 / x; x += 1.0; }
    const double f = 1.0 / (x * x);
    return r + log(x) - 0.5 / x -
           f * (1.0 / 12 - f * (1.0 / 120 - f * (1.0 / 252 - f * (1.0 / 240 - f / 132))));
}
__device__ double trigamma_d(double x) {
    double r = 0.0;
    while (x < 6.0) { r += 1.0 / (x * x); x += 1.0; }
    const double f = 1.0 / (x * x);
    return r + 1.0 / x + f / 2.0 +
           f / x * (1.0 / 6 - f * (1.0 / 30 - f * (1.0 / 42 - f * (1.0 / 30))));
}

__global__ void prep_records_kernel(const ara_record *__restrict__ raw,
                                    const uint32_t *__restrict__ src, uint64_t n,
                                    BetaRec *__restrict__ out, float *__restrict__ out_mu) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const ara_record q = raw[src ? src[t] : t];
        const double mu = q.mean_loss, si = q.sigma_i, sc = q.sigma_c, mx = q.max_loss;
        out_mu[t] = q.mean_loss;
        BetaRec r;
        const double sigma = si + sc;                          // step 1
        if (sigma == 0.0 || mu == 0.0 || mu == mx) {           // G10
            r.a = -1.0f; r.b = 0.0f; r.c0 = 0.0f; r.wi = 0.0f; r.wc = 0.0f;
            r.scale = (sigma == 0.0) ? q.mean_loss : (mu == 0.0 ? 0.0f : q.max_loss);
            r.mu_l = 0.0f; r.sd_l = 0.0f;
            out[t] = r;
            continue;
        }
        const double mub = mu / mx, sb0 = sigma / mx;
        const double smax = sqrt(mub * (1.0 - mub));
        const double sb = (sb0 >= smax) ? smax * (1.0 - 1e-6) : sb0;
        const double kappa = (smax / sb) * (smax / sb) - 1.0;
        const float af = (float)(mub * kappa), bf = (float)((1.0 - mub) * kappa);
        const double a = af, b = bf;
        const float mf = __fdiv_rn(af, __fadd_rn(af, bf));     // same op as the sampler
        const double m = mf;
        const double lnB = lgamma(a) + lgamma(b) - lgamma(a + b);
        const double wi = si / sigma, wc = sc / sigma;
        const double nr = sqrt(wi * wi + wc * wc);
        r.a = af; r.b = bf;
        r.c0 = (float)(a * log(m) + b * log1p(-m) - lnB);
        r.wi = (float)(wi / nr); r.wc = (float)(wc / nr);
        r.scale = q.max_loss;
        r.mu_l = (float)(digamma_d(a) - digamma_d(b));
        r.sd_l = (float)sqrt(trigamma_d(a) + trigamma_d(b));
        out[t] = r;
    }
}

void launch_prep_records(const ara_record *raw, const uint32_t *src, uint64_t n, BetaRec *out,
                         float *out_mu, cudaStream_t s) {
    if (n == 0) return;
    const int threads = 256;
    const uint64_t blocks = (n + threads - 1) / threads;
    prep_records_kernel<<<(unsigned)(blocks < 65535 * 16 ? blocks : 65535 * 16), threads, 0, s>>>(
        raw, src, n, out, out_mu);
}

// ---------------------------------------------------------------------------
// The fused YET scan.  One warp owns one trial at a time (dynamic trial
// scheduler); per 32-occurrence chunk it streams the event ids (coalesced,
// evict-first), tests the shared-memory presence bitmap, fetches the
// event-major index entry from L2 for hits, and enqueues every present
// (occurrence, slot) pair into a warp-private shared-memory queue.  A flush
// samples all queued pairs with all 32 lanes busy, then reduces per
// (occurrence, layer) segment, applies the occurrence terms, and adds to
// the trial's per-layer fp64 sum.  At the end of the trial the aggregate
// terms give the YLT entry.  All reductions are fixed trees: the YLT is a
// pure function of the inputs.
// ---------------------------------------------------------------------------
constexpr int kWarps = 16;          // warps per CTA
constexpr int kQCap = 256;          // queue capacity (pairs) per warp (>= ARA_MAX_SLOTS)
static_assert(kQCap >= ARA_MAX_SLOTS, "queue must hold one occurrence's pairs");

struct WarpSmem {
    uint2 q[kQCap];                 // {device record, (k << 8) | slot}
    float xs[kQCap];                // sampled loss per queued pair
    double S[ARA_MAX_LAYERS];       // per-layer trial sums
    unsigned int cnt[ARA_MAX_LAYERS];
    unsigned long long hsh[ARA_MAX_LAYERS];
};

struct ScanArgs {
    PortfolioDev pf;
    YetDev yet;
    uint64_t seed;
    uint32_t flags;
    float *ylt;
    uint32_t *dbg_count;
    uint64_t *dbg_hash;
    RunStatus *status;
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

template <bool SU>
__device__ __forceinline__ void flush_queue(const ScanArgs &A, WarpSmem &W, const SlotInfo *slots,
                                            const LayerInfo *layers, int qn, uint32_t trial_g,
                                            int lane) {
    // phase 1: one loss per queued pair, all lanes busy
    for (int p = lane; p < qn; p += 32) {
        const uint2 e = W.q[p];
        const uint32_t slot = e.y & 0xffu, k = e.y >> 8;
        const SlotInfo &si = slots[slot];
        float x;
        if (SU) {
            const BetaRec r = A.pf.recs[e.x];
            if (r.a <= 0.0f) {
                x = r.scale;
            } else {
                const uint32_t bp = philox_lane0(trial_g, k, si.prog, 1u, A.seed);   // z_(Prog,E)
                const uint32_t be = philox_lane0(trial_g, k, si.elt, 2u, A.seed);    // z_(E)
                const float v = combine_v(r, norm_quantile_from_bits(bp), norm_quantile_from_bits(be));
                bool ok;
                int steps = 0, iters = 0;
                x = sample_loss_from_v(r, v, ok, steps, iters);
                if (!ok) atomicAdd(&A.status->nonconverged, 1u);
            }
        } else {
            x = __ldg(A.pf.rec_mu + e.x);
        }
        if (si.has_terms) x = si.share * fminf(fmaxf(x - si.ret, 0.0f), si.lim);     // line 8
        W.xs[p] = x;
    }
    __syncwarp();
    // phase 2: segments = runs of equal (occurrence, layer); sum (line 9),
    // occurrence terms (line 11), add to the layer's trial sum
    for (int base = 0; base < qn; base += 32) {
        const int p = base + lane;
        bool head = false;
        uint32_t layer = 0;
        double g = 0.0;
        if (p < qn) {
            const uint2 e = W.q[p];
            layer = slots[e.y & 0xffu].layer;
            const uint32_t key = ((e.y >> 8) << 8) | layer;
            if (p == 0) {
                head = true;
            } else {
                const uint2 ep = W.q[p - 1];
                head = (((ep.y >> 8) << 8) | slots[ep.y & 0xffu].layer) != key;
            }
            if (head) {
                double l = 0.0;
                for (int r = p; r < qn; ++r) {
                    const uint2 er = W.q[r];
                    if ((((er.y >> 8) << 8) | slots[er.y & 0xffu].layer) != key) break;
                    l += (double)W.xs[r];
                }
                const LayerInfo &L = layers[layer];
                g = fmin(fmax(l - L.occ_r, 0.0), L.occ_l);
            }
        }
        // deterministic per-layer reduction: one fixed-tree warp sum per
        // distinct layer present among this round's segment heads
        unsigned pending = __ballot_sync(0xffffffffu, head);
        while (pending) {
            const int leader = __ffs(pending) - 1;
            const uint32_t lay = __shfl_sync(0xffffffffu, layer, leader);
            const bool mine = head && layer == lay;
            const double s = warp_sum_f64(mine ? g : 0.0);
            if (lane == 0) W.S[lay] += s;
            pending &= ~__ballot_sync(0xffffffffu, mine);
        }
    }
    __syncwarp();
}

template <bool SU, int MW>
__global__ void __launch_bounds__(kWarps * 32, 1) scan_kernel(const __grid_constant__ ScanArgs A) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpSmem *wsm = reinterpret_cast<WarpSmem *>(smem_raw);
    SlotInfo *slots = reinterpret_cast<SlotInfo *>(wsm + kWarps);
    LayerInfo *layers = reinterpret_cast<LayerInfo *>(slots + ARA_MAX_SLOTS);
    uint32_t *bitmap = reinterpret_cast<uint32_t *>(layers + ARA_MAX_LAYERS);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t t = threadIdx.x; t < A.pf.bitmap_words; t += blockDim.x) bitmap[t] = A.pf.bitmap[t];
    for (uint32_t t = threadIdx.x; t < A.pf.n_slots; t += blockDim.x) slots[t] = A.pf.slots[t];
    for (uint32_t t = threadIdx.x; t < A.pf.n_layers; t += blockDim.x) layers[t] = A.pf.layers[t];
    __syncthreads();

    WarpSmem &W = wsm[warp];
    const bool dbg = (A.flags & ARA_DEBUG_LOOKUP) != 0;
    const uint32_t nl = A.pf.n_layers;
    const uint64_t n_trials = A.yet.n_trials;

    while (true) {
        unsigned long long t = 0;
        if (lane == 0) t = atomicAdd(&A.status->next_trial, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
        if (t >= n_trials) break;
        const uint64_t base = A.yet.fixed_len ? t * (uint64_t)A.yet.fixed_len : A.yet.offsets[t];
        const uint32_t len = A.yet.fixed_len ? A.yet.fixed_len
                                             : (uint32_t)(A.yet.offsets[t + 1] - base);
        const uint32_t trial_g = (uint32_t)(A.yet.first_trial + t);   // global index i
        for (uint32_t l = lane; l < nl; l += 32) { W.S[l] = 0.0; W.cnt[l] = 0u; W.hsh[l] = 0ull; }
        __syncwarp();
        int qn = 0;
        for (uint32_t c = 0; c < len; c += 32) {
            const uint32_t k = c + lane;
            uint32_t mask[MW];
#pragma unroll
            for (int w = 0; w < MW; ++w) mask[w] = 0u;
            uint32_t first = 0, cnt = 0;
            if (k < len) {
                const uint32_t e = __ldcs(A.yet.events + base + k);                  // line 4
                if (e >= A.pf.catalog) {
                    atomicAdd(&A.status->bad_event, 1u);
                } else {
                    const uint32_t bit = e >> A.pf.bitmap_shift;
                    if ((bitmap[bit >> 5] >> (bit & 31)) & 1u) {                      // line 6
                        const uint32_t *ix = A.pf.index + (uint64_t)e * A.pf.idx_stride;
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
#pragma unroll
                        for (int w = 0; w < MW; ++w) cnt += __popc(mask[w]);
                    }
                }
            }
            // enqueue whole occurrences, flushing when the queue would overflow
            bool todo = cnt > 0;
            while (__any_sync(0xffffffffu, todo)) {
                uint32_t incl = todo ? cnt : 0u;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                const uint32_t room = (uint32_t)(kQCap - qn);
                const bool fits = todo && incl <= room;
                if (fits) {
                    uint32_t pos = (uint32_t)qn + incl - cnt;
                    uint32_t rec = first;
#pragma unroll
                    for (int w = 0; w < MW; ++w) {
                        uint32_t mw = mask[w];
                        while (mw) {
                            const int bpos = __ffs(mw) - 1;
                            mw &= mw - 1;
                            const uint32_t slot = (uint32_t)(w * 32 + bpos);
                            W.q[pos++] = make_uint2(rec++, (k << 8) | slot);
                            if (dbg) {
                                const uint32_t lay = slots[slot].layer;
                                atomicAdd(&W.cnt[lay], 1u);
                                const uint64_t h = splitmix64(
                                    splitmix64(splitmix64((uint64_t)k) ^ slots[slot].elt) ^
                                    A.pf.rec_orig[rec - 1]);
                                atomicAdd(&W.hsh[lay], (unsigned long long)h);
                            }
                        }
                    }
                    todo = false;
                }
                const uint32_t added = __shfl_sync(0xffffffffu, fits ? incl : 0u, 31 - __clz(__ballot_sync(0xffffffffu, fits) | 1u));
                const unsigned fitmask = __ballot_sync(0xffffffffu, fits);
                qn += fitmask ? (int)added : 0;
                __syncwarp();
                if (__any_sync(0xffffffffu, todo)) {
                    flush_queue<SU>(A, W, slots, layers, qn, trial_g, lane);
                    qn = 0;
                }
            }
        }
        if (qn > 0) flush_queue<SU>(A, W, slots, layers, qn, trial_g, lane);
        // aggregate terms on the trial sum (line 12, G6) -> YLT (line 17)
        for (uint32_t l = lane; l < nl; l += 32) {
            const LayerInfo &L = layers[l];
            const double S = W.S[l];
            A.ylt[(uint64_t)l * n_trials + t] = (float)fmin(fmax(S - L.agg_r, 0.0), L.agg_l);
            if (dbg) {
                if (A.dbg_count) A.dbg_count[(uint64_t)l * n_trials + t] = W.cnt[l];
                if (A.dbg_hash) A.dbg_hash[(uint64_t)l * n_trials + t] = W.hsh[l];
            }
        }
        __syncwarp();
    }
}

static size_t scan_smem_bytes(const PortfolioDev &pf) {
    return sizeof(WarpSmem) * kWarps + sizeof(SlotInfo) * ARA_MAX_SLOTS +
           sizeof(LayerInfo) * ARA_MAX_LAYERS + sizeof(uint32_t) * (size_t)pf.bitmap_words;
}

template <bool SU, int MW>
static cudaError_t launch_scan_t(const ScanArgs &A, cudaStream_t s, int num_sms) {
    const size_t smem = scan_smem_bytes(A.pf);
    cudaError_t err = cudaFuncSetAttribute(scan_kernel<SU, MW>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_kernel<SU, MW>, kWarps * 32, smem);
    if (err != cudaSuccess) return err;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    scan_kernel<SU, MW><<<num_sms * per_sm, kWarps * 32, smem, s>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_scan(const PortfolioDev &pf, const YetDev &yet, uint64_t seed, uint32_t flags,
                        float *ylt, uint32_t *dbg_count, uint64_t *dbg_hash, RunStatus *status,
                        cudaStream_t s, int num_sms) {
    ScanArgs A{pf, yet, seed, flags, ylt, dbg_count, dbg_hash, status};
    const bool su = (flags & ARA_SU) != 0;
    if (pf.mask_words == 1) return su ? launch_scan_t<true, 1>(A, s, num_sms) : launch_scan_t<false, 1>(A, s, num_sms);
    if (pf.mask_words <= 3) return su ? launch_scan_t<true, 3>(A, s, num_sms) : launch_scan_t<false, 3>(A, s, num_sms);
    return su ? launch_scan_t<true, 7>(A, s, num_sms) : launch_scan_t<false, 7>(A, s, num_sms);
}

// ---------------------------------------------------------------------------
// Component kernels (row-level parity tests)
// ---------------------------------------------------------------------------
__global__ void sample_losses_kernel(const BetaRec *recs, const float *zp, const float *ze,
                                     uint64_t n, float *out, RunStatus *status) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const BetaRec r = recs[t];
        if (r.a <= 0.0f) { out[t] = r.scale; continue; }
        // z given as fp32 in (0,1): Phi^-1 on the smaller tail
        const float a = zp[t], b = ze[t];
        const float vp = (a < 0.5f) ? -1.41421356237f * erfcinvf(2.0f * a)
                                    : 1.41421356237f * erfcinvf(2.0f * (1.0f - a));
        const float ve = (b < 0.5f) ? -1.41421356237f * erfcinvf(2.0f * b)
                                    : 1.41421356237f * erfcinvf(2.0f * (1.0f - b));
        bool ok;
        int steps = 0, iters = 0;
        out[t] = sample_loss_from_v(r, combine_v(r, vp, ve), ok, steps, iters);
        if (!ok) atomicAdd(&status->nonconverged, 1u);
    }
}

cudaError_t launch_sample_losses(const BetaRec *recs, const float *zp, const float *ze, uint64_t n,
                                 float *out, RunStatus *status, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const uint64_t blocks = (n + 255) / 256;
    sample_losses_kernel<<<(unsigned)(blocks < 1u << 20 ? blocks : 1u << 20), 256, 0, s>>>(
        recs, zp, ze, n, out, status);
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

__global__ void max_event_kernel(const uint32_t *ev, uint64_t n, uint32_t *out) {
    uint32_t m = 0;
    const uint64_t n4 = n / 4;
    const uint4 *ev4 = reinterpret_cast<const uint4 *>(ev);
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n4;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(ev4 + t);
        m = max(m, max(max(v.x, v.y), max(v.z, v.w)));
    }
    for (uint64_t t = n4 * 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n;
         t += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, ev[t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

cudaError_t launch_max_event(const uint32_t *ev, uint64_t n, uint32_t *out, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess || n == 0) return e;
    max_event_kernel<<<148 * 4, 256, 0, s>>>(ev, n, out);
    return cudaGetLastError();
}

}  // namespace ara
