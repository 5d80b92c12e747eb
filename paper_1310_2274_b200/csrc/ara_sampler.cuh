// ara_sampler.cuh -- device functions of the secondary-uncertainty sampler
// (section 3 of arXiv 1310.2274) on sm_100a.
//
//   draws    : Philox4x32-10 keyed by the run seed; z_(Prog,E) from counter
//              (i, k, program, 1), z_(E) from (i, k, XELT, 2) (readings G2,
//              G4); U(x) = (2(x>>9)+1) 2^-24, exact in fp32.
//   steps 2-4: v = wi * Phi^-1(z_P) + wc * Phi^-1(z_E) (G1);
//              fp32, Phi^-1 taken on the smaller tail (exact for U's grid)
//   steps 5+ : x = I^-1(Phi(v); a, b) (G11).  The map
//              v -> lambda(v) = logit x(v) is smooth, so each record carries
//              a table of (lambda, dlambda/dv) at v = -7.75, -7.25, ..., 7.75, built
//              ONCE at ara_create_portfolio by an fp64 solve (below) and
//              evaluated per sample by quintic Hermite interpolation, the
//              second derivative coming from the ODE
//                  dlambda/dv = phi(v) B(a,b) / (x^a (1-x)^b),
//                  d2lambda/dv2 = lambda' (-v - (a(1-x) - b x) lambda').
//              Records whose table misses a midpoint check fall back to the
//              fp64 per-sample solve (mode kModeExact), as does ARA_EXACT.
//   loss     : max_l * x
//
// The fp64 solver: Halley iteration on ln(tail) as a function of lambda, so
// x and 1-x keep full relative precision and both tails are near-linear;
// the tail from the positive-term Gauss hypergeometric series of DLMF 8.17.8,
// on whichever of I_x(a,b) / I_{1-x}(b,a) sits below its switch point; the
// smaller tail t = Phi(-|v|) is matched directly (reading G13).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ara_internal.cuh"

namespace ara {

// ------------------------------------------------- fast fp32 intrinsics ---
// MUFU approximations with flush-to-zero: the sampler feeds them normal
// arguments (the erfinv log's argument is >= 2^-23, reciprocals are of
// 1 + e >= 1), where the .ftz forms return exactly what __expf / __logf /
// __fdividef return -- without the subnormal fix-ups those emit (3
// instructions each); a sigmoid's power that overflows to +inf or flushes to
// 0 gives x = 0 or 1, its limits
__device__ __forceinline__ float ex2_ftz(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float lg2_ftz(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_ftz(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ---------------------------------------------------------------- draws ---
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

__device__ __forceinline__ uint32_t philox_lane0(uint32_t i, uint32_t k, uint32_t id, uint32_t tag,
                                                 uint64_t seed) {
    return philox4x32_10(make_uint4(i, k, id, tag), (uint32_t)seed, (uint32_t)(seed >> 32)).x;
}

__device__ __forceinline__ float u01_from_bits(uint32_t x) {
    return (float)(2u * (x >> 9) + 1u) * 5.9604644775390625e-08f;
}

// Phi^-1(U(x)) = sqrt(2) erfinv(y), y = 2 U(x) - 1 = (2m + 1 - 2^23) 2^-23
// with m = x >> 9: exact in fp32, sign included, and 1 - y, 1 + y exact too.
// erfinv by Giles' single-precision approximation ("Approximating the
// erfinv function", GPU Computing Gems, 2011): w = -ln((1-y)(1+y)), a
// degree-8 polynomial in w - 2.5 (w < 5) or in sqrt(w) - 3, times y; sqrt(2)
// is folded into the coefficients.  Over the 2^23 values of U the relative
// error is <= 4e-7 (tests/test_gpu_parity.py), like erfcinvf's 4 ulp, at about
// half the instructions; the tail branch (|v| > 2.93) is taken by 0.34 % of draws.
__device__ __forceinline__ float norm_quantile_from_bits(uint32_t x) {
    const int yi = (int)((x >> 9) << 1) + 1 - (1 << 23);
    const float y = (float)yi * 1.1920928955078125e-07f;      // exact
    // 1 - y^2 by one fma: the exact product rounded once, the same value as
    // (1 - y)(1 + y) (both factors exact on U's grid); w - 2.5 = -ln(1 - y^2) - 2.5 in one fma
    const float l = lg2_ftz(fmaf(-y, y, 1.0f));
    float w = fmaf(l, -0.69314718055994530942f, -2.5f);     // w - 2.5
    float p;                                                  // sqrt(2) x Giles' coefficients
    if (w < 2.5f) {
        p = 3.974260232e-08f;
        p = fmaf(p, w, 4.854626601e-07f);
        p = fmaf(p, w, -4.982822671e-06f);
        p = fmaf(p, w, -6.210528108e-06f);
        p = fmaf(p, w, 3.091200308e-04f);
        p = fmaf(p, w, -1.773034941e-03f);
        p = fmaf(p, w, -5.908134035e-03f);
        p = fmaf(p, w, 3.488026612e-01f);
        p = fmaf(p, w, 2.123313550e+00f);
    } else {
        w = sqrtf(w + 2.5f) - 3.0f;
        p = -2.831457176e-04f;
        p = fmaf(p, w, 1.427656483e-04f);
        p = fmaf(p, w, 1.908259482e-03f);
        p = fmaf(p, w, -5.195012320e-03f);
        p = fmaf(p, w, 8.116889673e-03f);
        p = fmaf(p, w, -1.077978815e-02f);
        p = fmaf(p, w, 1.334857863e-02f);
        p = fmaf(p, w, 1.416581041e+00f);
        p = fmaf(p, w, 4.006434241e+00f);
    }
    return p * y;
}

// Phi^-1 of an arbitrary fp32 probability in (0,1) (component entry point)
__device__ __forceinline__ float norm_quantile_f(float z) {
    return (z < 0.5f) ? -1.41421356237f * erfcinvf(2.0f * z) : 1.41421356237f * erfcinvf(2.0f * (1.0f - z));
}

__device__ __forceinline__ float combine_v(const BetaRec &r, float vp, float ve) {
    return fmaf(r.wi, vp, r.wc * ve);                     // steps 3-4
}

// -------------------------------------------------------- fp64 solver ----
// ln F(a+b, 1; a+1; x) = ln sum_{n>=0} (a+b)_n / (a+1)_n x^n, the Gauss
// hypergeometric factor of I_x(a,b) = x^a (1-x)^b / (a B(a,b)) F(a+b,1;a+1;x)
// (DLMF 8.17.8).  Every term is positive (no cancellation) and, for
// x < (a+1)/(a+b+2), the term ratio (a+b+n) x / (a+1+n) stays below
// rmax = max((a+b) x / (a+1), x) < 1, so the series is summed until the next
// term cannot move the sum: t rmax / (1 - rmax) <= 2^-54 s.  ok = false if
// that takes more than 400000 terms (ratio within ~1e-4 of 1).
__device__ __forceinline__ double hyp2f1_ln64(double x, double a, double b, bool &ok) {
    const double r0 = (a + b) * x / (a + 1.0);
    const double rmax = fmax(r0, x);
    const double stop = 5.551115123125783e-17 * (1.0 - rmax) / rmax;
    double t = 1.0, s = 1.0, num = a + b, den = a + 1.0;
    ok = false;
    for (int n = 0; n < 400000; ++n) {
        t *= num * x / den;
        s += t;
        num += 1.0;
        den += 1.0;
        if (t <= stop * s) { ok = true; break; }
    }
    return log(s);
}

struct Tail64 {
    double lnT, hp, dphi, x, y, lnx, lny;
};

// ln of the matched tail (P = I_x(a,b) if lower, else Q = 1 - P) at lambda = logit x
__device__ __forceinline__ Tail64 tail64(double lam, bool lower, double a, double b, double lnB, bool &ok) {
    Tail64 r;
    const double e = exp(-fabs(lam));
    const double sp = log1p(e);                            // softplus(-|lam|)
    const double lnx = lam >= 0.0 ? -sp : lam - sp;
    const double lny = lam >= 0.0 ? -lam - sp : -sp;
    const double x = exp(lnx), y = exp(lny);
    const double phi = a * lnx + b * lny - lnB;            // ln(x^a y^b / B)
    // the series for I_x(a,b) below (a+1)/(a+b+2), else the one for
    // I_y(b,a) = 1 - I_x(a,b).  The other tail, 1 - G, is only the matched one
    // near that switch point (the bulk of the distribution), where it is not
    // small, so log1p(-G) loses no relative precision
    const bool direct = x < (a + 1.0) / (a + b + 2.0);
    const double lnF = direct ? hyp2f1_ln64(x, a, b, ok) : hyp2f1_ln64(y, b, a, ok);
    const double lnG = phi + lnF - log(direct ? a : b);
    const double G = exp(lnG);
    const double lnOther = log1p(-fmin(G, 1.0));
    r.lnT = lower ? (direct ? lnG : lnOther) : (direct ? lnOther : lnG);
    const double h = exp(phi - r.lnT);
    r.hp = lower ? h : -h;
    r.dphi = a * y - b * x;
    r.x = x; r.y = y; r.lnx = lnx; r.lny = lny;
    return r;
}

// lambda = logit(x) with tail(x) = exp(lnt) (lower: I_x(a,b); upper: 1 - I_x(a,b)).
__device__ __forceinline__ double solve_logit64(double lnt, bool lower, double a, double b,
                                                double lnB, double lam, bool &ok) {
    double lo = -INFINITY, hi = INFINITY;
    ok = false;
    bool series_ok = true;
    for (int it = 0; it < 300; ++it) {
        bool sok;
        const Tail64 e = tail64(lam, lower, a, b, lnB, sok);
        series_ok = series_ok && sok;
        const double g = e.lnT - lnt;
        if (g == 0.0) { ok = true; break; }
        const bool toolow = lower ? (g < 0.0) : (g > 0.0);
        if (toolow) lo = lam; else hi = lam;
        const double hpp = e.hp * (e.dphi - e.hp);
        double nl = lam - 2.0 * g * e.hp / (2.0 * e.hp * e.hp - g * hpp);
        const double scale = fmax(1.0, fabs(lam));
        if (!(nl > lo && nl < hi)) {
            if (isfinite(lo) && isfinite(hi)) nl = 0.5 * (lo + hi);
            else if (isfinite(lo)) nl = lo + fmax(2.0, fabs(lo));      // expand geometrically
            else nl = hi - fmax(2.0, fabs(hi));
        }
        const bool conv = fabs(nl - lam) <= 1e-13 * scale || (hi - lo) <= 1e-13 * scale;
        lam = nl;
        if (conv) { ok = true; break; }
    }
    ok = ok && series_ok;
    return lam;
}

__device__ __forceinline__ double digamma_d(double x) {
    double r = 0.0;
    while (x < 6.0) { r -= 1.0 / x; x += 1.0; }
    const double f = 1.0 / (x * x);
    return r + log(x) - 0.5 / x -
           f * (1.0 / 12 - f * (1.0 / 120 - f * (1.0 / 252 - f * (1.0 / 240 - f / 132))));
}
__device__ __forceinline__ double trigamma_d(double x) {
    double r = 0.0;
    while (x < 6.0) { r += 1.0 / (x * x); x += 1.0; }
    const double f = 1.0 / (x * x);
    return r + 1.0 / x + f / 2.0 + f / x * (1.0 / 6 - f * (1.0 / 30 - f * (1.0 / 42 - f * (1.0 / 30))));
}

// x = I^-1(Phi(v); a, b) by the fp64 solve (initial guess: logit(X) normal,
// moments psi(a)-psi(b), psi1(a)+psi1(b)); returns lambda
__device__ __forceinline__ double lambda_exact64(double v, double a, double b, double lnB, double lam0,
                                                 bool &ok) {
    const bool lower = v <= 0.0;
    const double t = 0.5 * erfc(fabs(v) * 0.70710678118654752440);
    return solve_logit64(log(t), lower, a, b, lnB, lam0, ok);
}

// ------------------------------------------------------------ table eval --

// x = 1/(1 + e^-lambda) at a table node: e^-lambda overflows to +inf for
// lambda < -88.7 (rcp(inf) = +0: x = 0) and flushes to 0 above 87.3 (x = 1)
__device__ __forceinline__ float sigmoid_node(float lam) {
    return rcp_ftz(1.0f + ex2_ftz(-1.44269504088896340736f * lam));
}

// quintic Hermite on [v_i, v_i + h] from the two nodes' (lambda, lambda'),
// lambda'' from the ODE at each node, evaluated in Horner form in t in [0,1]:
// p(t) = l0 + B t + C/2 t^2 + t^3 (c3 + c4 t + c5 t^2) with B = h l0', C = h^2 l0'',
// E = h l1', F = h^2 l1'', D = l1 - l0.  p, p', p'' at t = 1 leave the residuals
// R0 = D - B - C/2, R1 = E - B - C, R2 = F - C, and c3 = 10 R0 - 4 R1 + R2/2,
// c4 = -15 R0 + 7 R1 - R2, c5 = 6 R0 - 3 R1 + R2/2 (the same polynomial as the
// expanded c3 = 10D - 6B - 3C/2 - 4E + F/2, ... in 5 fewer operations).  Every
// operation an explicit fmaf / fmul / fadd, so the rounding is the same in every
// kernel instantiation (no contraction choice).
__device__ __forceinline__ float quintic_from_nodes(float2 n0, float2 n1, int i, float t, float a, float b) {
    constexpr float kH2 = kTabH * kTabH;
    const float v0 = fmaf((float)i, kTabH, kTabV0), v1 = __fadd_rn(v0, kTabH);
    const float apb = __fadd_rn(a, b);
    const float x0 = sigmoid_node(n0.x), x1 = sigmoid_node(n1.x);
    const float g0 = fmaf(-apb, x0, a), g1 = fmaf(-apb, x1, a);          // a(1-x) - b x
    const float s0 = __fmul_rn(n0.y, fmaf(-g0, n0.y, -v0));               // lambda'' = l' (-v - g l')
    const float s1 = __fmul_rn(n1.y, fmaf(-g1, n1.y, -v1));
    const float B = __fmul_rn(kTabH, n0.y);                               // h l0'
    const float Ch = __fmul_rn(0.5f * kH2, s0);                           // C / 2
    const float D = __fsub_rn(n1.x, n0.x);
    const float R0 = __fsub_rn(__fsub_rn(D, B), Ch);                      // D - B - C/2
    const float R1 = fmaf(-2.0f, Ch, fmaf(kTabH, n1.y, -B));              // E - B - C
    const float T = __fmul_rn(0.5f * kH2, __fsub_rn(s1, s0));             // R2 / 2
    const float c3 = fmaf(10.0f, R0, fmaf(-4.0f, R1, T));
    const float c4 = fmaf(-15.0f, R0, fmaf(7.0f, R1, __fmul_rn(-2.0f, T)));
    const float c5 = fmaf(6.0f, R0, fmaf(-3.0f, R1, T));
    float p = fmaf(c5, t, c4);
    p = fmaf(p, t, c3);
    p = fmaf(p, t, Ch);
    p = fmaf(p, t, B);
    return fmaf(p, t, n0.x);
}

// quintic Hermite in v on record `rec`'s table
__device__ __forceinline__ float lambda_table(const TablePtr &tables, uint64_t rec, float a, float b, float v) {
    const float u = (fminf(fmaxf(v, kTabV0), -kTabV0) - kTabV0) * (1.0f / kTabH);
    const int i = min((int)u, kTabNodes - 2);
    const float t = u - (float)i;
    const float2 *row = table_row(tables, rec, i);
    return quintic_from_nodes(__ldg(row), __ldg(row + 1), i, t, a, b);
}

__device__ __forceinline__ float sigmoidf_(float lam) {
    // 1/(1+e^-lam); e^-lam = inf for lam < -88.7 gives rcp(inf) = +0 (the loss
    // underflows to 0); e^-lam below 2^-126 flushes to 0, where 1/(1+e) is 1 either way
    return rcp_ftz(1.0f + ex2_ftz(-1.44269504088896340736f * lam));
}

// Per-sample fp64 solve (table-less records, ARA_EXACT); kept out of line so
// its register demand does not constrain the hot path.
static __device__ __noinline__ float sample_exact64(float af, float bf, float mu_l, float sd_l, float scale,
                                             float v, bool &ok) {
    const double a = af, b = bf;
    const double lnB = lgamma(a) + lgamma(b) - lgamma(a + b);
    const double lam = lambda_exact64((double)v, a, b, lnB, (double)mu_l + (double)v * sd_l, ok);
    const double x = 1.0 / (1.0 + exp(-lam));
    return (float)((double)scale * x);
}

// One loss draw (Alg.1 line 7) given v.  EX instantiates the fp64 fallback;
// kernels without it are only launched when every record has a table.
template <bool EX>
__device__ __forceinline__ float sample_loss_from_v(const BetaRec &r, const TablePtr &tables,
                                                    uint64_t rec, float v, bool exact, bool &ok) {
    ok = true;
    if (r.mode == kModeDegenerate) return r.scale;               // G10
    if (!EX || (r.mode == kModeTable && !exact)) {
        const float lam = lambda_table(tables, rec, r.a, r.b, v);
        return r.scale * sigmoidf_(lam);
    }
    return sample_exact64(r.a, r.b, r.mu_l, r.sd_l, r.scale, v, ok);
}

}  // namespace ara
