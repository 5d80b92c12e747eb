/*
 * ara_oracle.c -- the fp64 CPU ORACLE for Aggregate Risk Analysis with
 * secondary uncertainty (Varghese & Rau-Chaplin, arXiv 1310.2274).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT THE PRODUCT.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It shares no code, header, table or constant with the
 * CUDA path (paper_1310_2274_b200/csrc); neither includes the other.
 *
 * It is deliberately plain and slow: straight loops in the paper's order and
 * notation, IEEE fp64, no blocking, fusion or reordering.  Every function
 * cites the PAPER.md line (P:n) it follows, or the DESIGN.md reading (Gn,
 * numbered as in SURVEY.md section 8(c)) where the paper is silent/garbled.
 *
 * Pins (what checks this file against something other than itself) are in
 * tests/test_oracle_*.py: Random123 known-answer vectors, scipy/mpmath
 * special functions, closed-form beta quantiles, SPEC.md worked examples,
 * the closed-form mean/variance of the loss draw, and a brute-force
 * straight-line Python engine on tiny portfolios.
 *
 * What no paper number can confirm: the RNG keying is a reading (G2/G4), not
 * a value the paper prints.  Its implementation here is pinned (Random123
 * known-answer vectors; an independent brute-force engine with its own
 * Philox and keying; the distribution of the draws), but the paper prints no
 * config-level YLT/PML/TVaR to check the reading itself against.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Counter-based RNG: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).     */
/* Reading G4: z draws are not specified by the paper beyond "in U(0,1)"     */
/* (P:193); we use Philox4x32-10 keyed by the 64-bit seed.                   */
/* ------------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                       uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {               /* key schedule: bump between rounds */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Reading G4: U(x) = (2*(x>>9)+1) * 2^-24, exact in fp32 and fp64, never 0 or 1. */
double orc_u01(uint32_t x) {
    return (double)(2u * (x >> 9) + 1u) * 5.9604644775390625e-08; /* 2^-24 */
}

/* z_(Prog,E) for program p, global trial i, occurrence k (G2). */
double orc_z_prog(uint64_t seed, uint32_t p, uint64_t i, uint32_t k) {
    uint32_t ctr[4] = {(uint32_t)i, k, p, 1u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return orc_u01(o[0]);
}

/* z_(E) for global trial i, occurrence k, XELT j (G2). */
double orc_z_event(uint64_t seed, uint64_t i, uint32_t k, uint32_t j) {
    uint32_t ctr[4] = {(uint32_t)i, k, j, 2u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return orc_u01(o[0]);
}

/* Paper-literal alternatives to reading G2:
 * (A) z_(E) stored with each XELT record, so constant
 *     across trials and occurrences: counter (r, j, 0, 6), r = the record's
 *     index within XELT j;
 * (B) z_(E) per event occurrence, shared by every XELT ("Event-
 *     Occurrence-Specific"): counter (i, k, 0, 7). */
double orc_z_event_record(uint64_t seed, uint32_t j, uint32_t r) {
    uint32_t ctr[4] = {r, j, 0u, 6u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return orc_u01(o[0]);
}

double orc_z_event_occ(uint64_t seed, uint64_t i, uint32_t k) {
    uint32_t ctr[4] = {(uint32_t)i, k, 0u, 7u};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    orc_philox4x32_10(ctr, key, o);
    return orc_u01(o[0]);
}

/* ------------------------------------------------------------------------ */
/* Statistical functions (section 4.2).                            */
/* ------------------------------------------------------------------------ */

/* Phi(v), the standard normal CDF, via libm erfc. */
double orc_norm_cdf(double v) { return 0.5 * erfc(-v / sqrt(2.0)); }

/* Standard normal density. */
static double orc_norm_pdf(double v) {
    return exp(-0.5 * v * v) / sqrt(2.0 * M_PI);
}

/* Phi^-1(p): Wichura's AS241 (PPND16) rational approximations followed by
 * one Newton step on Phi.  Reading G1: step 2 of section 3.2
 * prints the CDF integral but maps U(0,1)->N(0,1), which needs the inverse. */
double orc_norm_quantile(double p) {
    if (!(p > 0.0 && p < 1.0)) return NAN;
    double q = p - 0.5, r, x;
    if (fabs(q) <= 0.425) {
        r = 0.180625 - q * q;
        x = q * (((((((2.5090809287301226727e+3 * r + 3.3430575583588128105e+4) * r +
                      6.7265770927008700853e+4) * r + 4.5921953931549871457e+4) * r +
                    1.3731693765509461125e+4) * r + 1.9715909503065514427e+3) * r +
                  1.3314166789178437745e+2) * r + 3.3871328727963666080e0) /
            (((((((5.2264952788528545610e+3 * r + 2.8729085735721942674e+4) * r +
                  3.9307895800092710610e+4) * r + 2.1213794301586595867e+4) * r +
                5.3941960214247511077e+3) * r + 6.8718700749205790830e+2) * r +
              4.2313330701600911252e+1) * r + 1.0);
    } else {
        r = (q < 0.0) ? p : 1.0 - p;
        r = sqrt(-log(r));
        if (r <= 5.0) {
            r -= 1.6;
            x = (((((((7.74545014278341407640e-4 * r + 2.27238449892691845833e-2) * r +
                      2.41780725177450611770e-1) * r + 1.27045825245236838258e0) * r +
                    3.64784832476320460504e0) * r + 5.76949722146069140550e0) * r +
                  4.63033784615654529590e0) * r + 1.42343711074968357734e0) /
                (((((((1.05075007164441684324e-9 * r + 5.47593808499534494600e-4) * r +
                      1.51986665636164571966e-2) * r + 1.48103976427480074590e-1) * r +
                    6.89767334985100004550e-1) * r + 1.67638483018380384940e0) * r +
                  2.05319162663775882187e0) * r + 1.0);
        } else {
            r -= 5.0;
            x = (((((((2.01033439929228813265e-7 * r + 2.71155556874348757815e-5) * r +
                      1.24266094738807843860e-3) * r + 2.65321895265761230930e-2) * r +
                    2.96560571828504891230e-1) * r + 1.78482653991729133580e0) * r +
                  5.46378491116411436990e0) * r + 6.65790464350110377720e0) /
                (((((((2.04426310338993978564e-15 * r + 1.42151175831644588870e-7) * r +
                      1.84631831751005468180e-5) * r + 7.86869131145613259100e-4) * r +
                    1.48753612908506148525e-2) * r + 1.36929880922735805310e-1) * r +
                  5.99832206555887937690e-1) * r + 1.0);
        }
        if (q < 0.0) x = -x;
    }
    /* one Newton step on Phi(x) = p, with the residual taken on the smaller tail */
    double resid = (p < 0.5) ? (orc_norm_cdf(x) - p) : ((1.0 - p) - orc_norm_cdf(-x));
    double d = orc_norm_pdf(x);
    if (d > 0.0) x -= resid / d;
    return x;
}

/* ln B(a,b) = lnGamma(a) + lnGamma(b) - lnGamma(a+b) (P:246's B(alpha,beta)). */
double orc_lnbeta(double a, double b) {
    int s;
    return lgamma_r(a, &s) + lgamma_r(b, &s) - lgamma_r(a + b, &s);
}

/* Continued fraction for I_x(a,b) (DLMF 8.17.22):
 *   I_x(a,b) = x^a (1-x)^b / (a B(a,b)) * 1/(1+ d1/(1+ d2/(1+ ...))),
 *   d_{2m}   =  m (b-m) x / ((a+2m-1)(a+2m)),
 *   d_{2m+1} = -(a+m)(a+b+m) x / ((a+2m)(a+2m+1)),
 * evaluated by the modified Lentz method; fast for x < (a+1)/(a+b+2).
 * Returns 1/(1+ d1/(1+ ...)); *ok=0 on non-convergence. */
static double orc_betacf(double x, double a, double b, int *ok) {
    const double tiny = 1e-300, eps = 1e-16;
    double f = 1.0, C = 1.0, D = 0.0;      /* f_0 = b_0 = 1 */
    *ok = 0;
    for (int n = 1; n < 200000; n++) {
        int m = n / 2;
        double d;
        if (n % 2 == 0)
            d = (m * (b - m) * x) / ((a + 2.0 * m - 1.0) * (a + 2.0 * m));
        else
            d = -((a + m) * (a + b + m) * x) / ((a + 2.0 * m) * (a + 2.0 * m + 1.0));
        D = 1.0 + d * D;
        if (fabs(D) < tiny) D = tiny;
        C = 1.0 + d / C;
        if (fabs(C) < tiny) C = tiny;
        D = 1.0 / D;
        double delta = C * D;
        f *= delta;
        if (fabs(delta - 1.0) < eps) { *ok = 1; break; }
    }
    return 1.0 / f;
}

/* Regularised incomplete beta I_x(a,b) = B(x;a,b)/B(a,b),
 * with the symmetry I_x(a,b) = 1 - I_{1-x}(b,a) for x > (a+1)/(a+b+2). */
double orc_beta_cdf(double x, double a, double b) {
    if (x <= 0.0) return 0.0;
    if (x >= 1.0) return 1.0;
    int ok;
    double lnB = orc_lnbeta(a, b);
    double front = exp(a * log(x) + b * log1p(-x) - lnB);
    if (x < (a + 1.0) / (a + b + 2.0)) {
        return front * orc_betacf(x, a, b, &ok) / a;
    }
    return 1.0 - front * orc_betacf(1.0 - x, b, a, &ok) / b;
}

/* Beta density x^(a-1)(1-x)^(b-1)/B(a,b). */
static double orc_beta_pdf(double x, double a, double b) {
    return exp((a - 1.0) * log(x) + (b - 1.0) * log1p(-x) - orc_lnbeta(a, b));
}

/* InvCDF_beta(p; a, b) (reading G11: the functional inverse of
 * I_x, not a reciprocal): the x in (0,1) with I_x(a,b) = p.  Safeguarded
 * Newton on a bracket [lo, hi] that every evaluation tightens; when a Newton
 * step leaves the bracket we bisect (geometrically when the bracket spans
 * decades, so that deep tails are reached).  Returns the iteration count, or
 * -1 when it does not converge (reading G12: the paper's "converges ...
 * within a certain error" is not quantified; we ask 1e-14 relative). */
int orc_beta_quantile(double p, double a, double b, double *out) {
    if (p <= 0.0) { *out = 0.0; return 0; }
    if (p >= 1.0) { *out = 1.0; return 0; }
    double lo = 0.0, hi = 1.0;
    double x = a / (a + b);                  /* start at the mean */
    for (int it = 1; it <= 2000; it++) {
        double F = orc_beta_cdf(x, a, b) - p;
        if (fabs(F) <= 1e-15 * p) { *out = x; return it; }   /* residual test */
        if (F < 0.0) lo = x; else hi = x;
        double dens = orc_beta_pdf(x, a, b);
        double xn = (dens > 0.0 && isfinite(dens)) ? x - F / dens : NAN;
        if (xn == x) { *out = x; return it; }                 /* step below 1 ulp */
        if (!(xn > lo && xn < hi)) {
            if (lo > 0.0 && hi / lo > 16.0 && hi <= 0.5) xn = sqrt(lo * hi);
            else if (lo == 0.0) xn = hi / 16.0;
            else if (hi == 1.0) xn = 1.0 - (1.0 - lo) / 16.0;
            else if (lo >= 0.5 && (1.0 - lo) / (1.0 - hi) > 16.0)
                xn = 1.0 - sqrt((1.0 - lo) * (1.0 - hi));
            else xn = 0.5 * (lo + hi);
        }
        if (fabs(xn - x) <= 1e-14 * x || (hi - lo) <= 1e-15 * lo) {
            *out = xn;
            return it;
        }
        x = xn;
    }
    *out = x;
    return -1;
}

/* ------------------------------------------------------------------------ */
/* Secondary uncertainty (section 3).                             */
/* ------------------------------------------------------------------------ */

/* Beta parameters with the sigma_beta cap (reading G9:
 * inclusive cap, "a value very close to" = sigma_max*(1-1e-6)). */
void orc_beta_params(double mu_l, double sigma, double max_l,
                     double *alpha, double *beta) {
    double sigma_b = sigma / max_l;
    double mu_b = mu_l / max_l;
    double sigma_b_max = sqrt(mu_b * (1.0 - mu_b));
    if (sigma_b >= sigma_b_max) sigma_b = sigma_b_max * (1.0 - 1e-6);
    double ratio = sigma_b_max / sigma_b;
    *alpha = mu_b * (ratio * ratio - 1.0);
    *beta = (1.0 - mu_b) * (ratio * ratio - 1.0);
}

/* Steps 1-5 of section 3.2.  Returns v; writes z = Phi(v) and
 * q = Phi(-v), both computed directly (reading G13). */
double orc_combine(double z_prog, double z_e, double sigma_i, double sigma_c,
                   double *z, double *q) {
    double sigma = sigma_i + sigma_c;                  /* step 1 */
    double v_prog = orc_norm_quantile(z_prog);         /* step 2, P:205 (G1) */
    double v_e = orc_norm_quantile(z_e);               /* step 2, P:206 (G1) */
    double wi = sigma_i / sigma, wc = sigma_c / sigma;
    double lc = v_prog * wi + v_e * wc;                /* step 3 */
    double v = lc / sqrt(wi * wi + wc * wc);           /* step 4 */
    *z = orc_norm_cdf(v);                              /* step 5 */
    *q = orc_norm_cdf(-v);
    return v;
}

/* Loss draw for one (record, z_prog, z_e): Loss = max_l * InvCDF_beta(z;
 * alpha, beta).  Degenerate records (reading G10): sigma = 0 gives
 * mu_l; mu_l = 0 gives 0; mu_l = max_l gives max_l.  Reading G13: match z
 * when z <= 1/2, else solve the complementary equation I_y(beta, alpha) = q
 * for y = 1 - x.  Returns 0, or -1 if the quantile did not converge. */
int orc_sample_loss(double mu_l, double sigma_i, double sigma_c, double max_l,
                    double z_prog, double z_e, double *loss) {
    double sigma = sigma_i + sigma_c;
    if (sigma == 0.0) { *loss = mu_l; return 0; }
    if (mu_l == 0.0) { *loss = 0.0; return 0; }
    if (mu_l == max_l) { *loss = max_l; return 0; }
    double alpha, beta, z, q, x;
    orc_beta_params(mu_l, sigma, max_l, &alpha, &beta);
    orc_combine(z_prog, z_e, sigma_i, sigma_c, &z, &q);
    int it;
    if (z <= 0.5) {
        it = orc_beta_quantile(z, alpha, beta, &x);
    } else {
        double y;
        it = orc_beta_quantile(q, beta, alpha, &y);
        x = 1.0 - y;
    }
    *loss = max_l * x;
    return it < 0 ? -1 : 0;
}

/* ------------------------------------------------------------------------ */
/* Financial terms (section 2.3; reading G5: max(., 0)).          */
/* ------------------------------------------------------------------------ */
double orc_occ_terms(double l, double occ_r, double occ_l) {
    return fmin(fmax(l - occ_r, 0.0), occ_l);
}
double orc_agg_terms(double s, double agg_r, double agg_l) {
    return fmin(fmax(s - agg_r, 0.0), agg_l);
}
/* XELT terms I (reading G7): share*min(max(x-R,0),L). */
double orc_xelt_terms(double x, double ret, double lim, double share) {
    return share * fmin(fmax(x - ret, 0.0), lim);
}

/* Order-independent lookup fingerprint of one present (occurrence k, XELT j,
 * record r) triple: nested splitmix64.  Used only to check the lookup step
 * (Alg.1 line 6) bit-exactly. */
static uint64_t orc_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
uint64_t orc_lookup_hash(uint32_t k, uint32_t j, uint32_t r) {
    return orc_splitmix64(orc_splitmix64(orc_splitmix64(k) ^ j) ^ r);
}

/* ------------------------------------------------------------------------ */
/* Algorithm 1 over dense direct-access tables.          */
/* ------------------------------------------------------------------------ */
typedef struct {
    /* catalog and XELTs */
    uint32_t catalog_size;
    uint32_t n_elts;
    const uint64_t *elt_off;      /* [n_elts+1] record ranges per XELT */
    const uint32_t *rec_event;    /* [R] event id of each record */
    const double *rec_mean, *rec_si, *rec_sc, *rec_max;
    const double *elt_terms;      /* [n_elts*3] (retention, limit, share) or NULL */
    /* portfolio */
    uint32_t n_layers;
    const uint32_t *layer_prog;   /* [n_layers] */
    const uint64_t *layer_elt_off;/* [n_layers+1] */
    const uint32_t *layer_elts;   /* XELT ids per layer */
    const double *layer_terms;    /* [n_layers*4] OccR, OccL, AggR, AggL */
    /* YET */
    uint64_t n_trials;
    const uint64_t *trial_index;  /* [n_trials] global trial index i */
    const uint64_t *trial_off;    /* [n_trials+1] */
    const uint32_t *events;
    uint64_t seed;
    int su;
    int rng_mode;                 /* 0: reading G2; 1: (A) z_(E) per record; 2: (B) per occurrence;
                                     3: the paper's data model -- both draws supplied with the inputs */
    const double *zp_sup;         /* rng_mode 3: z_(Prog,E) of each YET occurrence, [program][occurrence] */
    const double *ze_sup;         /* rng_mode 3: z_(E) of each XELT record, [record] */
    uint64_t n_occ;               /* occurrences in the YET (stride of zp_sup) */
    /* dense direct-access table [n_elts][catalog_size] -> record id or -1 */
    int32_t *table;
    /* outputs [n_layers][n_trials] */
    double *ylt, *gross;
    double *occ_max;              /* or NULL: per (layer, trial) largest occurrence loss net of
                                     occurrence terms (the OEP basis; NEXT-3 reading G29) */
    uint32_t *count;
    uint64_t *hash;
    /* work split */
    uint64_t t_begin, t_end;
    int status;
} orc_job;

static void *orc_worker(void *arg) {
    orc_job *J = (orc_job *)arg;
    J->status = 0;
    for (uint32_t li = 0; li < J->n_layers; li++) {          /* line 2: each Layer */
        uint32_t prog = J->layer_prog[li];                    /* line 1: its Program */
        const double *T = J->layer_terms + 4 * (size_t)li;
        for (uint64_t t = J->t_begin; t < J->t_end; t++) {    /* line 3: each Trial */
            uint64_t i = J->trial_index[t];
            double S = 0.0, M = 0.0;
            uint32_t cnt = 0;
            uint64_t h = 0;
            for (uint64_t o = J->trial_off[t]; o < J->trial_off[t + 1]; o++) { /* line 4 */
                uint32_t k = (uint32_t)(o - J->trial_off[t]);
                uint32_t e = J->events[o];
                double l_e_sum = 0.0;
                for (uint64_t x = J->layer_elt_off[li]; x < J->layer_elt_off[li + 1]; x++) { /* line 5 */
                    uint32_t j = J->layer_elts[x];
                    int32_t r = J->table[(size_t)j * J->catalog_size + e];   /* line 6 lookup */
                    if (r < 0) continue;                                     /* absent: zero loss */
                    uint32_t rloc = (uint32_t)(r - (int64_t)J->elt_off[j]);
                    cnt++;
                    h += orc_lookup_hash(k, j, rloc);
                    double l_e;
                    if (J->su) {                                             /* line 7 */
                        double zp = J->rng_mode == 3 ? J->zp_sup[(size_t)prog * J->n_occ + o]
                                  : orc_z_prog(J->seed, prog, i, k);
                        double ze = J->rng_mode == 3 ? J->ze_sup[r]
                                  : J->rng_mode == 1 ? orc_z_event_record(J->seed, j, rloc)
                                  : J->rng_mode == 2 ? orc_z_event_occ(J->seed, i, k)
                                  : orc_z_event(J->seed, i, k, j);               /* G2 / (A) / (B) / supplied */
                        if (orc_sample_loss(J->rec_mean[r], J->rec_si[r], J->rec_sc[r],
                                            J->rec_max[r], zp, ze, &l_e) != 0)
                            J->status = -1;
                    } else {
                        l_e = J->rec_mean[r];                                /* primary only */
                    }
                    if (J->elt_terms) {                                      /* line 8 */
                        const double *I = J->elt_terms + 3 * (size_t)j;
                        l_e = orc_xelt_terms(l_e, I[0], I[1], I[2]);
                    }
                    l_e_sum += l_e;                                          /* line 9 */
                }
                double g = orc_occ_terms(l_e_sum, T[0], T[1]);               /* line 11 (G6) */
                S += g;
                if (g > M) M = g;                                            /* OEP basis (G29) */
            }
            size_t oi = (size_t)li * J->n_trials + t;
            J->gross[oi] = S;
            if (J->occ_max) J->occ_max[oi] = M;
            J->ylt[oi] = orc_agg_terms(S, T[2], T[3]);                      /* lines 12, 17 (G6) */
            J->count[oi] = cnt;
            J->hash[oi] = h;
        }
    }
    return NULL;
}

/* Run Algorithm 1 for every layer of the portfolio over the given trials.
 * Builds the paper's dense direct-access tables first (the preprocessing
 * stage).  Returns 0, -1 (a quantile did not converge),
 * -2 (bad input) or -3 (out of memory). */
int orc_run(uint32_t catalog_size, uint32_t n_elts, const uint64_t *elt_off,
            const uint32_t *rec_event, const double *rec_mean, const double *rec_si,
            const double *rec_sc, const double *rec_max, const double *elt_terms,
            uint32_t n_layers, const uint32_t *layer_prog, const uint64_t *layer_elt_off,
            const uint32_t *layer_elts, const double *layer_terms, uint64_t n_trials,
            const uint64_t *trial_index, const uint64_t *trial_off, const uint32_t *events,
            uint64_t seed, int su, int n_threads, double *ylt, double *gross,
            uint32_t *count, uint64_t *hash, double *occ_max, int rng_mode,
            const double *zp_sup, const double *ze_sup) {
    size_t slots = (size_t)n_elts * catalog_size;
    int32_t *table = (int32_t *)malloc((slots ? slots : 1) * sizeof(int32_t));
    if (!table) return -3;
    for (size_t s = 0; s < slots; s++) table[s] = -1;
    for (uint32_t j = 0; j < n_elts; j++) {
        for (uint64_t r = elt_off[j]; r < elt_off[j + 1]; r++) {
            uint32_t e = rec_event[r];
            if (e >= catalog_size) { free(table); return -2; }
            table[(size_t)j * catalog_size + e] = (int32_t)r;
        }
    }
    for (uint64_t o = 0; o < trial_off[n_trials]; o++)
        if (events[o] >= catalog_size) { free(table); return -2; }
    if (rng_mode == 3 && (!zp_sup || !ze_sup)) { free(table); return -2; }
    if (n_threads < 1) n_threads = 1;
    if ((uint64_t)n_threads > n_trials) n_threads = n_trials ? (int)n_trials : 1;
    orc_job *jobs = (orc_job *)calloc((size_t)n_threads, sizeof(orc_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    for (int w = 0; w < n_threads; w++) {
        orc_job *J = &jobs[w];
        J->catalog_size = catalog_size; J->n_elts = n_elts; J->elt_off = elt_off;
        J->rec_event = rec_event; J->rec_mean = rec_mean; J->rec_si = rec_si;
        J->rec_sc = rec_sc; J->rec_max = rec_max; J->elt_terms = elt_terms;
        J->n_layers = n_layers; J->layer_prog = layer_prog; J->layer_elt_off = layer_elt_off;
        J->layer_elts = layer_elts; J->layer_terms = layer_terms; J->n_trials = n_trials;
        J->trial_index = trial_index; J->trial_off = trial_off; J->events = events;
        J->seed = seed; J->su = su; J->table = table; J->rng_mode = rng_mode;
        J->zp_sup = zp_sup; J->ze_sup = ze_sup; J->n_occ = trial_off[n_trials];
        J->ylt = ylt; J->gross = gross; J->count = count; J->hash = hash; J->occ_max = occ_max;
        J->t_begin = n_trials * (uint64_t)w / (uint64_t)n_threads;
        J->t_end = n_trials * (uint64_t)(w + 1) / (uint64_t)n_threads;
        pthread_create(&th[w], NULL, orc_worker, J);
    }
    int status = 0;
    for (int w = 0; w < n_threads; w++) {
        pthread_join(th[w], NULL);
        if (jobs[w].status) status = jobs[w].status;
    }
    free(th); free(jobs); free(table);
    return status;
}

/* Convenience loop for the distribution pins: n independent loss draws. */
int orc_sample_batch(uint64_t n, const double *mu, const double *si, const double *sc,
                     const double *mx, const double *zp, const double *ze, double *out) {
    int st = 0;
    for (uint64_t t = 0; t < n; t++)
        if (orc_sample_loss(mu[t], si[t], sc[t], mx[t], zp[t], ze[t], &out[t]) != 0) st = -1;
    return st;
}
