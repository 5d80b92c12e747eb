// ara_sampler.cuh -- device functions of the secondary-uncertainty sampler
// (section 3 of arXiv 1310.2274), fp32 on sm_100a.
//
//   draws    : Philox4x32-10 keyed by the run seed; z_(Prog,E) from counter
//              (i, k, program, 1), z_(E) from (i, k, XELT, 2) (readings G2,
//              G4); U(x) = (2(x>>9)+1) 2^-24, exact in fp32.
//   steps 2-4: v = wi * Phi^-1(z_P) + wc * Phi^-1(z_E) (G1)
//   step 5   : the smaller tail t = Phi(-|v|) and its side (G13)
//   quantile : x with I_x(a,b) = t (v <= 0) or 1 - I_x(a,b) = t (v > 0)
//              (G11), solved by Halley iteration on
//              ln(tail) as a function of lambda = logit(x), so that both x
//              and 1-x keep full relative precision and both tails are
//              near-linear.  The tail is evaluated from the continued
//              fraction of DLMF 8.17.22 with the division-free forward
//              (Wallis) recurrence and exact power-of-two rescaling.
//   loss     : max_l * x
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"

namespace ara {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// lane 0 of Philox for one counter
__device__ __forceinline__ uint32_t philox_lane0(uint32_t i, uint32_t k, uint32_t id, uint32_t tag,
                                                 uint64_t seed) {
    return philox4x32_10(make_uint4(i, k, id, tag), (uint32_t)seed, (uint32_t)(seed >> 32)).x;
}

__device__ __forceinline__ float u01_from_bits(uint32_t x) {
    return (float)(2u * (x >> 9) + 1u) * 5.9604644775390625e-08f;
}

// Phi^-1(U(x)) computed on the smaller tail, which is exact for U's grid:
// z = (2m+1) 2^-24; min(z, 1-z) = (2m+1) or (2^24-2m-1) times 2^-24.
__device__ __forceinline__ float norm_quantile_from_bits(uint32_t x) {
    const uint32_t m = x >> 9;
    const bool low = m < (1u << 22);
    const uint32_t num = low ? 2u * m + 1u : (1u << 24) - 2u * m - 1u;
    const float p2 = (float)num * 1.1920928955078125e-07f;   // 2 * tail, exact
    const float r = 1.41421356237f * erfcinvf(p2);            // -Phi^-1(tail) >= 0
    return low ? -r : r;
}

__device__ __forceinline__ float softplusf(float z) {
    // log(1 + e^z); absolute accuracy suffices where it is used
    return fmaxf(z, 0.0f) + __logf(1.0f + __expf(-fabsf(z)));
}

// 1 / (1 + d1/(1 + d2/(1 + ...))) of DLMF 8.17.22 for I_x(a,b), forward
// recurrence on the equivalent fraction b_n = q_n, a_n = q_{n-1} p_n where
// d_n = p_n / q_n; converged when consecutive convergents agree to 2e-7.
__device__ __forceinline__ float betacf_recip(float x, float a, float b, int &steps) {
    float Am = 1.0f, Bm = 0.0f;   // A_{n-2}, B_{n-2}
    float A = 1.0f, B = 1.0f;     // A_{n-1}, B_{n-1}
    float qprev = 1.0f;
    const float apb = a + b;
    int n = 1;
    for (; n < 600; n += 2) {
        const float m = (float)(n >> 1);
        // odd step n = 2m+1
        float u = fmaf(2.0f, m, a);
        float q = u * (u + 1.0f);
        float p = -(a + m) * (apb + m) * x;
        float c = qprev * p;
        float An = fmaf(q, A, c * Am), Bn = fmaf(q, B, c * Bm);
        Am = A; Bm = B; A = An; B = Bn; qprev = q;
        // even step n+1 = 2(m+1)
        const float m1 = m + 1.0f;
        u = fmaf(2.0f, m1, a);
        q = (u - 1.0f) * u;
        p = m1 * (b - m1) * x;
        c = qprev * p;
        An = fmaf(q, A, c * Am); Bn = fmaf(q, B, c * Bm);
        Am = A; Bm = B; A = An; B = Bn; qprev = q;
        // exact power-of-two rescale by A's exponent
        const int e = min(max((__float_as_int(A) >> 23) & 0xff, 1), 253);
        const float s = __int_as_float((254 - e) << 23);
        A *= s; B *= s; Am *= s; Bm *= s;
        // |h_n - h_{n-1}| <= eps |h_n|  <=>  |A B_{n-1} - A_{n-1} B| <= eps |A B_{n-1}|
        const float t1 = A * Bm;
        const float diff = fmaf(Am, B, -t1);
        if (fabsf(diff) <= 2e-7f * fabsf(t1)) break;
    }
    steps += n + 1;
    return B / A;
}

struct TailEval {
    float lnT;    // log of the matched tail probability at lambda
    float hp;     // d lnT / d lambda
    float dphi;   // d phi / d lambda = a(1-x) - b x
};

// Evaluate ln(tail) at lambda = logit(x) (see file header).
__device__ __forceinline__ TailEval tail_at(float lam, bool lower, float a, float b, float m,
                                            float lnm, float ln1m, float c0, int &steps) {
    const float ex = __expf(-lam);
    const float x = __frcp_rn(1.0f + ex);                 // x = sigmoid(lam)
    const float y = __frcp_rn(1.0f + __frcp_rn(ex));      // 1 - x, full relative precision
    const float lnx = -softplusf(-lam), lny = -softplusf(lam);
    const float d = x - m;
    // ln(x/m) and ln((1-x)/(1-m)); log1p near the centre keeps the large
    // a ln x + b ln(1-x) - ln B cancellation out of fp32
    const float t1 = (fabsf(d) < 0.5f * m) ? log1pf(__fdividef(d, m)) : lnx - lnm;
    const float t2 = (fabsf(d) < 0.5f * (1.0f - m)) ? log1pf(__fdividef(-d, 1.0f - m)) : lny - ln1m;
    const float phi = fmaf(a, t1, fmaf(b, t2, c0));      // ln(x^a (1-x)^b / B(a,b))
    const bool direct = x < __fdividef(a + 1.0f, a + b + 2.0f);
    const float xa = direct ? x : y, aa = direct ? a : b, bb = direct ? b : a;
    const float cf = betacf_recip(xa, aa, bb, steps);
    const float lnG = phi + __logf(__fdividef(cf, aa));  // ln of the directly computed tail
    const float G = __expf(lnG);
    const float lnOther = log1pf(-fminf(G, 1.0f));
    const float lnP = direct ? lnG : lnOther;
    const float lnQ = direct ? lnOther : lnG;
    TailEval r;
    r.lnT = lower ? lnP : lnQ;
    const float h = __expf(phi - r.lnT);
    r.hp = lower ? h : -h;
    r.dphi = fmaf(a, y, -b * x);
    return r;
}

// Solve for x = I^-1 on the given tail; returns x, sets *ok.
__device__ __forceinline__ float beta_quantile_tail(float t, bool lower, float v, const BetaRec &r,
                                                    bool &ok, int &steps, int &iters) {
    const float a = r.a, b = r.b;
    const float m = __fdiv_rn(a, a + b);
    const float lnm = logf(m), ln1m = log1pf(-m);
    const float lnt = logf(t);
    // initial guess: logit(X) ~ N(psi(a)-psi(b), psi1(a)+psi1(b)), bounded
    // by the tail asymptotes x^a/(a B) = t (lower) / (1-x)^b/(b B) = t (upper)
    float lam = fmaf(v, r.sd_l, r.mu_l);
    const float lnB = fmaf(a, lnm, fmaf(b, ln1m, -r.c0));
    if (lower && b >= 1.0f) lam = fmaxf(lam, __fdividef(lnt + __logf(a) + lnB, a));
    if (!lower && a >= 1.0f) lam = fminf(lam, -__fdividef(lnt + __logf(b) + lnB, b));
    float lo = -INFINITY, hi = INFINITY;
    ok = false;
    int it = 0;
    for (; it < 64; ++it) {
        const TailEval e = tail_at(lam, lower, a, b, m, lnm, ln1m, r.c0, steps);
        const float g = e.lnT - lnt;
        const bool toolow = lower ? (g < 0.0f) : (g > 0.0f);
        if (toolow) lo = lam; else hi = lam;
        const float hpp = e.hp * (e.dphi - e.hp);
        const float step = __fdividef(2.0f * g * e.hp, fmaf(2.0f * e.hp, e.hp, -g * hpp));
        float nl = lam - step;
        const float scale = fmaxf(1.0f, fabsf(lam));
        const bool small = fabsf(step) <= 2e-6f * scale;
        if (!(nl > lo && nl < hi) && !small) {
            if (isfinite(lo) && isfinite(hi)) nl = 0.5f * (lo + hi);
            else if (isfinite(lo)) nl = lo + 2.0f;
            else nl = hi - 2.0f;
        }
        const bool conv = fabsf(nl - lam) <= 1e-3f * scale;
        lam = nl;
        if (conv) { ok = true; ++it; break; }
    }
    iters += it;
    return __frcp_rn(1.0f + __expf(-lam));
}

// One loss draw (Alg.1 line 7) for record r and the two uniforms' bits.
__device__ __forceinline__ float sample_loss_from_v(const BetaRec &r, float v, bool &ok,
                                                    int &steps, int &iters) {
    if (r.a <= 0.0f) { ok = true; return r.scale; }       // degenerate (G10)
    const float t = 0.5f * erfcf(fabsf(v) * 0.70710678118654752f);
    const bool lower = v <= 0.0f;
    const float x = beta_quantile_tail(t, lower, v, r, ok, steps, iters);
    return r.scale * x;
}

__device__ __forceinline__ float combine_v(const BetaRec &r, float vp, float ve) {
    return fmaf(r.wi, vp, r.wc * ve);                     // steps 3-4
}

}  // namespace ara
