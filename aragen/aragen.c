/*
 * aragen.c -- seeded synthetic INPUT generator (YET, XELT records) shared by
 * the tests, bench.py and smoke().  It holds none of the method's arithmetic:
 * no lookup, no sampler, no terms -- only the data the paper's Algorithm 1
 * takes as input, shaped like the paper's workloads (P:60, P:86,
 * P:261) with the value distributions stated in DESIGN.md ("input recipe").
 *
 * Randomness: its own copy of Philox4x32-10 (counter-based, so any trial or
 * record can be generated independently, in any order, on any rank).
 * Counter tags used here: 0 = YET event id, 3 = record values,
 * 4 = Fisher-Yates event choice, 5 = trial length.  (The method's own draws
 * use tags 1 and 2; those live in the oracle and in the CUDA path.)
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

static inline void gen_philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                              uint64_t seed, uint32_t out[4]) {
    uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
    for (int r = 0; r < 10; r++) {
        uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
        uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
        c1 = (uint32_t)p1;
        c3 = (uint32_t)p0;
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static inline double gen_u01(uint32_t x) {
    return (double)(2u * (x >> 9) + 1u) * 5.9604644775390625e-08;
}

/* uniform integer in [0, n) from a 32-bit word (multiply-shift) */
static inline uint32_t gen_below(uint32_t x, uint32_t n) {
    return (uint32_t)(((uint64_t)x * (uint64_t)n) >> 32);
}

/* --- YET event ids ------------------------------------------------------- */
typedef struct {
    uint64_t seed, first_trial, t0, t1;
    uint32_t catalog;
    const uint64_t *off;   /* CSR offsets, or NULL for fixed length */
    uint32_t fixed_len;
    uint32_t *out;
} yet_job;

static void *yet_worker(void *arg) {
    yet_job *J = (yet_job *)arg;
    uint32_t o[4];
    for (uint64_t t = J->t0; t < J->t1; t++) {
        uint64_t i = J->first_trial + t;
        uint64_t b = J->off ? J->off[t] : t * (uint64_t)J->fixed_len;
        uint64_t e = J->off ? J->off[t + 1] : b + J->fixed_len;
        for (uint64_t x = b; x < e; x++) {
            gen_philox((uint32_t)i, (uint32_t)(x - b), 0u, 0u, J->seed, o);
            J->out[x] = gen_below(o[0], J->catalog);
        }
    }
    return NULL;
}

/* Event ids of trials [first_trial, first_trial+n_trials): uniform over the
 * catalog, keyed by (global trial i, occurrence k).  Repeats allowed (G3). */
int aragen_yet(uint64_t seed, uint32_t catalog, uint64_t first_trial, uint64_t n_trials,
               const uint64_t *trial_off, uint32_t fixed_len, uint32_t *out, int n_threads) {
    if (catalog == 0) return -1;
    if (n_threads < 1) n_threads = 1;
    if ((uint64_t)n_threads > n_trials) n_threads = n_trials ? (int)n_trials : 1;
    yet_job *jobs = (yet_job *)calloc((size_t)n_threads, sizeof(yet_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    for (int w = 0; w < n_threads; w++) {
        yet_job *J = &jobs[w];
        J->seed = seed; J->first_trial = first_trial; J->catalog = catalog;
        J->off = trial_off; J->fixed_len = fixed_len; J->out = out;
        J->t0 = n_trials * (uint64_t)w / (uint64_t)n_threads;
        J->t1 = n_trials * (uint64_t)(w + 1) / (uint64_t)n_threads;
        pthread_create(&th[w], NULL, yet_worker, J);
    }
    for (int w = 0; w < n_threads; w++) pthread_join(th[w], NULL);
    free(th); free(jobs);
    return 0;
}

/* Trial lengths in [kmin, kmax] keyed by the global trial index ("800
 * to 1500" events per trial). */
void aragen_trial_lengths(uint64_t seed, uint64_t first_trial, uint64_t n_trials,
                          uint32_t kmin, uint32_t kmax, uint32_t *out) {
    uint32_t o[4];
    for (uint64_t t = 0; t < n_trials; t++) {
        gen_philox((uint32_t)(first_trial + t), 0xFFFFFFFFu, 0u, 5u, seed, o);
        out[t] = kmin + gen_below(o[0], kmax - kmin + 1u);
    }
}

/* --- XELT records -------------------------------------------------------- */
/* R distinct event ids for XELT j by a seeded partial Fisher-Yates over the
 * catalog, and per-record values (DESIGN.md input recipe):
 *   mu    = 10^(4+3u1)           log-uniform in [1e4, 1e7)
 *   max_l = (2+8u2) mu
 *   s_I   = (0.1+0.4u3) mu * sigma_scale
 *   s_C   = (0.05+0.25u4) mu * sigma_scale
 * rounded to fp32 (both sides then read identical values).  integer_mu != 0
 * rounds mu to an integer (for bit-exact primary-uncertainty checks). */
int aragen_elt(uint64_t seed, uint32_t j, uint32_t catalog, uint32_t n_rec,
               double sigma_scale, int integer_mu, uint32_t *ev, float *mu,
               float *s_i, float *s_c, float *mx) {
    if (n_rec > catalog) return -1;
    uint32_t *perm = (uint32_t *)malloc((size_t)catalog * sizeof(uint32_t));
    if (!perm) return -2;
    for (uint32_t e = 0; e < catalog; e++) perm[e] = e;
    uint32_t o[4];
    for (uint32_t r = 0; r < n_rec; r++) {
        gen_philox(j, r, 0u, 4u, seed, o);
        uint32_t s = r + gen_below(o[0], catalog - r);
        uint32_t tmp = perm[r]; perm[r] = perm[s]; perm[s] = tmp;
        ev[r] = perm[r];
        gen_philox(j, r, 0u, 3u, seed, o);
        double u1 = gen_u01(o[0]), u2 = gen_u01(o[1]), u3 = gen_u01(o[2]), u4 = gen_u01(o[3]);
        double m = pow(10.0, 4.0 + 3.0 * u1);
        if (integer_mu) m = floor(m + 0.5);
        float mf = (float)m;
        mu[r] = mf;
        mx[r] = (float)((2.0 + 8.0 * u2) * (double)mf);
        s_i[r] = (float)((0.1 + 0.4 * u3) * (double)mf * sigma_scale);
        s_c[r] = (float)((0.05 + 0.25 * u4) * (double)mf * sigma_scale);
    }
    free(perm);
    return 0;
}

/* Storage encoding of a YET (not part of the method): event ids bit-packed
 * LSB-first, id x in bits [x*bits, (x+1)*bits) of the little-endian uint32
 * word stream (ids must be < 2^bits).  out has ceil(n*bits/32) words, zeroed
 * here.  Threads split the ids at multiples of 32 ids (whole words). */
typedef struct { const uint32_t *ev; uint64_t x0, x1; uint32_t bits; uint32_t *out; } pack_job;

static void *pack_worker(void *arg) {
    pack_job *J = (pack_job *)arg;
    for (uint64_t x = J->x0; x < J->x1; x++) {
        uint64_t bit = x * J->bits, w = bit >> 5;
        uint32_t sh = (uint32_t)(bit & 31u), v = J->ev[x];
        J->out[w] |= v << sh;
        if (sh + J->bits > 32u) J->out[w + 1] |= v >> (32u - sh);
    }
    return NULL;
}

int aragen_pack_bits(const uint32_t *ev, uint64_t n, uint32_t bits, uint32_t *out, int n_threads) {
    if (bits < 1 || bits > 32) return -1;
    uint64_t words = (n * bits + 31) / 32;
    memset(out, 0, words * sizeof(uint32_t));
    if (bits < 32)
        for (uint64_t x = 0; x < n; x++)
            if (ev[x] >> bits) return -2;
    if (n_threads < 1) n_threads = 1;
    uint64_t blocks = (n + 31) / 32;          /* 32 ids end on a word boundary for any bits */
    if ((uint64_t)n_threads > blocks) n_threads = blocks ? (int)blocks : 1;
    pack_job *jobs = (pack_job *)calloc((size_t)n_threads, sizeof(pack_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    for (int w = 0; w < n_threads; w++) {
        pack_job *J = &jobs[w];
        J->ev = ev; J->bits = bits; J->out = out;
        J->x0 = blocks * (uint64_t)w / (uint64_t)n_threads * 32;
        J->x1 = blocks * (uint64_t)(w + 1) / (uint64_t)n_threads * 32;
        if (J->x1 > n) J->x1 = n;
        pthread_create(&th[w], NULL, pack_worker, J);
    }
    for (int w = 0; w < n_threads; w++) pthread_join(th[w], NULL);
    free(th); free(jobs);
    return 0;
}
