/*
 * ara.h -- C ABI of libara, the B200-native (sm_100a) hot path of Aggregate
 * Risk Analysis with secondary uncertainty (Varghese & Rau-Chaplin,
 * arXiv 1310.2274).  Citations: P:n = PAPER.md line n; Gn = a reading of the
 * paper listed in DESIGN.md (numbered as in SURVEY.md section 8(c)).
 *
 * Problem statement (Algorithm 1): Input YET, XELT, PF; Output
 * YLT; risk measures PML and TVaR from the YLT.
 *
 * Conventions for every entry point:
 *  - Return value: ARA_OK (0) or one of the ARA_E* codes below.  Nothing is
 *    thrown across the ABI.  ara_last_error() returns a thread-local message
 *    with context (layer / XELT / record index, or trial) for the last
 *    failure on the calling thread.
 *  - Pointers marked "host or device" are classified with
 *    cudaPointerGetAttributes; host memory may be pageable or pinned.
 *  - Inputs are copied: the caller may free its arrays after the call
 *    returns (device inputs are copied device-to-device on the context's
 *    stream, so they must stay valid until that stream reaches the copy).
 *  - Handles are owned by the library until the matching *_destroy call.
 *  - All device work is enqueued on the context's CUDA stream; calls that
 *    return host results synchronise that stream.
 *  - No CPU fallback exists: every step of the path runs in CUDA kernels.
 *    Creating a context fails with ARA_ECUDA when no device is usable.
 */
#ifndef ARA_H
#define ARA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define ARA_OK 0
#define ARA_EINVAL 1    /* invalid argument / failed validation            */
#define ARA_ERANGE 2    /* event id or index out of range                  */
#define ARA_EDUP 3      /* duplicate event in an XELT / XELT in a layer    */
#define ARA_ENOMEM 4    /* host or device allocation failed                */
#define ARA_ECUDA 5     /* CUDA runtime / launch error                     */
#define ARA_ECONVERGE 6 /* beta quantile failed to converge for >=1 sample;
                           outputs are still written, count in last_error  */
#define ARA_ENCCL 7     /* reserved (collectives live above the ABI)       */

/* ---- ara_run flags ----------------------------------------------------- */
#define ARA_SU 1u            /* apply secondary uncertainty (section 3)     */
#define ARA_DEBUG_LOOKUP 2u  /* also write per-(layer,trial) lookup count
                                and hash (bit-exact check of Alg.1 line 6) */
#define ARA_EXACT 4u         /* solve every beta quantile per sample in fp64
                                instead of the per-record quantile tables
                                (validation mode; slow)                    */
#define ARA_WIDE_PAIRS 16u   /* keep 8-byte {record, k} pair records even when
                                4-byte packed ones fit (same results; for tests
                                and comparison)                            */

#define ARA_RNG_RECORD 32u   /* paper-literal z_(E) (reading G2 alternative A,
                                P:71/P:76/P:90): one draw stored per XELT
                                record, constant across trials; Philox
                                counter (record index within its XELT, XELT
                                id, 0, 6)                                   */
#define ARA_RNG_OCCURRENCE 64u /* z_(E) per event occurrence shared by every
                                XELT (G2 alternative B); counter
                                (trial, occurrence, 0, 7).  Default (neither
                                flag): reading G2, counter (trial,
                                occurrence, XELT id, 2)                     */
#define ARA_ASYNC 256u       /* ara_run / ara_run_ep return as soon as the run is
                                enqueued: no host synchronisation; overflowing
                                trials and table-less records are handled by
                                device-sized passes (the overflow pool is
                                pre-sized by ara_prepare / the first run); range
                                errors, non-convergence and an exhausted pool
                                are latched and reported by the next
                                ara_ctx_synchronize.  ara_last_run_timings
                                waits for the run (for a portfolio of several
                                kernel groups: the last group's times; a
                                synchronous run sums them).  Every launch of
                                such a run can be captured into a CUDA graph. */
#define ARA_RNG_SUPPLIED 128u /* the paper's data model: z_(Prog,E)
                                of each YET occurrence and z_(E) of each XELT
                                record are inputs, supplied by ara_yet_set_z
                                and ara_portfolio_set_z; no draw is taken   */

/* ---- limits (validated) ------------------------------------------------ */
#define ARA_MAX_SLOTS 224    /* XELTs per layer; also the (layer, XELT) slots
                                of one kernel group: a larger portfolio (or
                                one of > 8 layers) is split into groups of
                                consecutive layers run one after the other
                                over the YET (same results)                 */
#define ARA_MAX_LAYERS 64    /* layers of one kernel group (internal)       */
#define ARA_MAX_PORTFOLIO_LAYERS 4096    /* layers per portfolio            */
#define ARA_MAX_PORTFOLIO_SLOTS 65536    /* sum over layers of XELTs per layer
                                            ("10,000 XELTs")          */
#define ARA_MAX_EVENTS_PER_TRIAL (1u << 24)
#define ARA_MAX_XELTS (1u << 24)          /* XELTs per portfolio (~10,000) */
#define ARA_MAX_PROGRAMS 256u             /* program ids 0..255 (up to 10) */

typedef struct ara_ctx ara_ctx;
typedef struct ara_portfolio ara_portfolio;
typedef struct ara_yet ara_yet;

/* One eXtended event loss XEL_i = {E_i, mu_l, sigma_I, sigma_C, max_l}
 * (P:76).  Constraints: 0 <= mean_loss <= max_loss,
 * sigma_i >= 0, sigma_c >= 0, max_loss > 0, all finite.  z_(E) is not
 * stored: it is drawn per (trial, occurrence, XELT) (reading G2). */
typedef struct {
    uint32_t event_id;
    float mean_loss;
    float sigma_i;
    float sigma_c;
    float max_loss;
} ara_record;

/* Layer terms T = (OccR, OccL, AggR, AggL).  Retentions
 * >= 0 and finite; limits > 0, +INFINITY allowed. */
typedef struct {
    double occ_retention;
    double occ_limit;
    double agg_retention;
    double agg_limit;
} ara_layer_terms;

/* Optional XELT financial terms I (Alg.1 line 8; reading G7):
 * x -> share * min(max(x - retention, 0), limit).  retention >= 0,
 * limit > 0 (+INF ok), 0 < share <= 1. */
typedef struct {
    double retention;
    double limit;
    double share;
} ara_elt_terms;

/* Thread-local description of the last failure ("" if none). */
const char *ara_last_error(void);

/* Library version as 10000*major + 100*minor + patch. */
int ara_version(void);

/* Create a context on CUDA device `device`, enqueuing all work on
 * `cuda_stream` (a cudaStream_t; NULL = the legacy default stream).
 * ARA_ECUDA if the device is unavailable. */
int ara_ctx_create(int device, void *cuda_stream, ara_ctx **out);
void ara_ctx_destroy(ara_ctx *ctx);
/* Block until all work enqueued by this context has finished; then report
 * (and clear) the errors latched by ARA_ASYNC runs since the last call:
 * ARA_ERANGE (event ids >= catalog_size), ARA_ECONVERGE, ARA_ENOMEM (trials
 * that overflowed their pair regions and did not fit the overflow pool:
 * their YLT entries were not written -- rerun without ARA_ASYNC). */
int ara_ctx_synchronize(ara_ctx *ctx);

/* Host-only validation of a portfolio (no device needed); same arguments
 * and checks as ara_create_portfolio.  Host pointers only.
 *   catalog_size        number of events in the catalogue (event ids < it)
 *   n_elts              number of XELTs, <= ARA_MAX_XELTS
 *   elt_rec_offsets     [n_elts+1] record ranges; records of XELT j are
 *                       records[elt_rec_offsets[j] .. elt_rec_offsets[j+1])
 *   records             [elt_rec_offsets[n_elts]] XELT records
 *   elt_terms           [n_elts] or NULL (identity, G7)
 *   n_layers            layers in the portfolio, <= ARA_MAX_PORTFOLIO_LAYERS
 *   layer_program       [n_layers] program id of each layer (keys z_(Prog,E)),
 *                       < ARA_MAX_PROGRAMS
 *   layer_elt_offsets   [n_layers+1] ranges into layer_elts
 *   layer_elts          XELT ids covered by each layer, no duplicates within
 *                       a layer; <= ARA_MAX_SLOTS per layer, sum of layer
 *                       sizes <= ARA_MAX_PORTFOLIO_SLOTS
 *   layer_terms         [n_layers]
 * Errors: ARA_EINVAL (bad value / shape), ARA_ERANGE (event id >=
 * catalog_size, XELT id >= n_elts), ARA_EDUP (duplicate event in an XELT or
 * duplicate XELT in a layer). */
int ara_validate_portfolio(uint32_t catalog_size, uint32_t n_elts,
                           const uint64_t *elt_rec_offsets, const ara_record *records,
                           const ara_elt_terms *elt_terms, uint32_t n_layers,
                           const uint32_t *layer_program, const uint64_t *layer_elt_offsets,
                           const uint32_t *layer_elts, const ara_layer_terms *layer_terms);

/* Preprocessing stage (direct-access lookup P:157): validate,
 * build the event-major direct-access index and the presence bitmap on the
 * host, upload, and derive the per-record beta parameters in a
 * device kernel.  Arguments as ara_validate_portfolio (host pointers). */
int ara_create_portfolio(ara_ctx *ctx, uint32_t catalog_size, uint32_t n_elts,
                         const uint64_t *elt_rec_offsets, const ara_record *records,
                         const ara_elt_terms *elt_terms, uint32_t n_layers,
                         const uint32_t *layer_program, const uint64_t *layer_elt_offsets,
                         const uint32_t *layer_elts, const ara_layer_terms *layer_terms,
                         ara_portfolio **out);
void ara_portfolio_destroy(ara_portfolio *pf);
/* Layout facts of a built portfolio (any pointer may be NULL):
 *   n_device_records  (layer, record) pairs held on the device
 *   n_table_less      records whose quantile table failed its midpoint check
 *                     (sampled by the fp64 per-sample solve instead)
 *   device_bytes      HBM held by the portfolio */
int ara_portfolio_info(const ara_portfolio *pf, uint64_t *n_device_records,
                       uint64_t *n_table_less, uint64_t *device_bytes);

/* Load a YET: trial i of this table has global index
 * first_trial + i (the Philox counters use the global index, so a
 * trial-sharded run is bit-identical to a single run, reading G2/G4).
 *   n_trials        trials in this table (>= 0)
 *   first_trial     global index of trial 0; first_trial + n_trials <= 2^32
 *   trial_offsets   [n_trials+1] host CSR offsets, or NULL for fixed length
 *   fixed_len       events per trial when trial_offsets == NULL
 *   event_ids       [total events] uint32, host or device, trial-major,
 *                   occurrence order within a trial; NULL: every id starts
 *                   as 0 (fill with ara_yet_refill / ara_yet_refill_packed)
 *   timestamps      NULL, or [total events] host floats that must be sorted
 *                   ascending within each trial; validated, then not
 *                   used (reading G19: the year loss is order-invariant)
 * Event ids are range-checked against the portfolio in ara_run (ARA_ERANGE). */
int ara_load_yet(ara_ctx *ctx, uint64_t n_trials, uint64_t first_trial,
                 const uint64_t *trial_offsets, uint32_t fixed_len, const uint32_t *event_ids,
                 const float *timestamps, ara_yet **out);
/* Replace the event ids of an existing YET (same shape) from host or device
 * memory; asynchronous on the context stream (the host buffer must stay valid
 * until the stream passes the copy; pinned memory makes it a true DMA). */
int ara_yet_refill(ara_ctx *ctx, ara_yet *yet, const uint32_t *event_ids);
/* The same from a bit-packed copy of the event ids (a storage encoding of the
 * YET, not part of the method): id x occupies bits
 * [x*bits, (x+1)*bits) of the little-endian uint32 word stream `packed`
 * (ceil(total*bits/32) words, host or device), bits in [1, 32]; with
 * bits = ceil(log2 catalog) the host->device copy moves bits/32 of the bytes
 * of ara_yet_refill.  Host words are staged on the device, device words are
 * read where they are (they must stay valid until the context stream passes
 * the unpack: a caller may copy host words into its own device buffer on
 * another stream and overlap that copy with earlier work); a kernel unpacks
 * them; asynchronous like ara_yet_refill.  Ids >= catalog_size are
 * caught by ara_run (ARA_ERANGE).  ARA_EINVAL for bits out of range. */
int ara_yet_refill_packed(ara_ctx *ctx, ara_yet *yet, uint32_t bits, const uint32_t *packed);
/* The paper's YET tuples (E, t, z_(Prog,E)): attach the
 * z_(Prog,E) of every occurrence, for each program, to a loaded YET.
 *   n_programs  programs supplied (>= 1); a run's portfolio may use programs
 *               0 .. n_programs-1
 *   z_prog      host [n_programs][total events] floats in (0,1): the value
 *               of occurrence o (trial-major, occurrence order, as the event
 *               ids) for program p is z_prog[p * total + o]
 * Copied; used by ara_run with ARA_RNG_SUPPLIED.  ARA_EINVAL on a value
 * outside (0,1) (with its program and occurrence). */
int ara_yet_set_z(ara_ctx *ctx, ara_yet *yet, uint32_t n_programs, const float *z_prog);
/* The paper's XEL records {E, mu_l, z_(E), sigma_I, sigma_C, max_l}:
 * attach z_(E) to every record of a built portfolio.
 *   z_event  host [total records] floats in (0,1), in the order of the
 *            records passed to ara_create_portfolio
 * Copied; used by ara_run with ARA_RNG_SUPPLIED.  ARA_EINVAL on a value
 * outside (0,1). */
int ara_portfolio_set_z(ara_ctx *ctx, ara_portfolio *pf, const float *z_event);
uint64_t ara_yet_num_trials(const ara_yet *yet);
void ara_yet_destroy(ara_yet *yet);

/* Algorithm 1 for every layer over every trial of `yet`:
 * lookup (line 6), secondary uncertainty (line 7, section 3) if
 * flags & ARA_SU else the mean loss, XELT terms (line 8), per-occurrence
 * sum (line 9), occurrence terms (line 11), aggregate terms on the trial sum
 * (line 12, reading G6), YLT (line 17).
 *   seed      64-bit key of the z_(Prog,E) / z_(E) Philox streams
 *   ylt       DEVICE [n_layers][n_trials] fp32, caller-allocated
 *   dbg_count NULL or DEVICE [n_layers][n_trials] present-pair counts
 *   dbg_hash  NULL or DEVICE [n_layers][n_trials] sum of lookup fingerprints
 * (dbg_* require flags & ARA_DEBUG_LOOKUP.)  Asynchronous except for the
 * convergence / range flags, read back at the end (one small D2H).
 * Errors: ARA_ERANGE (an event id >= catalog_size), ARA_ECONVERGE. */
int ara_run(ara_ctx *ctx, const ara_portfolio *pf, const ara_yet *yet, uint64_t seed,
            uint32_t flags, float *ylt, uint32_t *dbg_count, uint64_t *dbg_hash);

/* ara_run plus the basis of the occurrence exceedance curve (OEP; SURVEY
 * NEXT-3, reading G29: the paper's line-11 values, are the
 * occurrence losses; the OEP takes their per-trial maximum):
 *   occ_max   DEVICE [n_layers][n_trials] fp32, caller-allocated: the largest
 *             occurrence loss net of occurrence terms of each (layer, trial),
 *             0 for a trial without a present pair.  ara_risk_measures on it
 *             (per layer, layer >= 0) gives OEP PML / TVaR; its roll-up over
 *             layers (layer = -1) is NOT a portfolio OEP.
 * Same arguments, outputs and errors as ara_run; ARA_EINVAL if occ_max is
 * NULL or host memory. */
int ara_run_ep(ara_ctx *ctx, const ara_portfolio *pf, const ara_yet *yet, uint64_t seed,
               uint32_t flags, float *ylt, float *occ_max, uint32_t *dbg_count, uint64_t *dbg_hash);

/* Optional: allocate every scratch buffer ara_run needs for this
 * (portfolio, YET) pair with these flags, so that ara_run itself allocates
 * nothing (the pair slot: batch x region pairs; the per-trial pair counts;
 * with ARA_ASYNC the pre-sized overflow pool).  Without it ara_run grows the same
 * buffers on first use.  A run whose trials overflow their regions still
 * grows the overflow pool (exactly sized) when that happens.
 * Errors: ARA_EINVAL, ARA_ECUDA / ARA_ENOMEM-like allocation failures as ARA_ECUDA. */
int ara_prepare(ara_ctx *ctx, const ara_portfolio *pf, const ara_yet *yet, uint32_t flags);

/* Device time of the kernels of the last ara_run on this context (CUDA
 * events on its stream): compact_ms = YET stream + lookup (compact_kernel),
 * sample_ms = draws + sampler + terms + YLT (sample_kernel; the fused
 * kernel under ARA_EXACT), redo_ms = trials re-run by the fused fp64-capable
 * kernel (0 when none).  Any pointer may be NULL. */
int ara_last_run_timings(const ara_ctx *ctx, double *compact_ms, double *sample_ms, double *redo_ms);

/* Kernels launched by the last ara_run / ara_run_ep on this context (all
 * libara kernels: compaction + sampler per trial batch, the overflow pass,
 * the fp64 redo; or the one streaming kernel of the primary path) and the
 * trial batches of its two-kernel path (0 on the primary / fused paths).
 * Any pointer may be NULL. */
int ara_last_run_launches(const ara_ctx *ctx, uint32_t *kernel_launches, uint32_t *batches);

/* PML and TVaR (reading G17) at each return period of one layer's
 * YLT, or of the portfolio roll-up sum over layers (layer = -1, G16), by a
 * device radix select over the fp32 bit patterns (up to 4 return periods: one
 * cooperative launch selecting every needed rank at once in three digit passes
 * of 12/10/10 bits, TVaR tail sums in exact int64 fixed point; more return
 * periods: a select plus a sort of the tail, or per-rank selects).
 *   ylt        DEVICE fp32, laid out [n_shards][n_layers][n_total/n_shards]
 *              (n_shards = 1 for a single run; > 1 for an all-gathered set
 *              of per-rank shards -- the measures are permutation-invariant)
 *   n_total    trials over all shards (divisible by n_shards), >= 1
 *   rps        [n_rp] return periods, each > 1 (host)
 *   pml_out, tvar_out  [n_rp] host
 * PML(RP): r = (N+1)/RP on the descending order statistics L(1)>=...>=L(N),
 * linear interpolation, clamped to [L(N), L(1)]; TVaR(RP): mean of all
 * entries >= VaR, VaR = the descending order statistic of rank ceil(N/RP)
 * (integer RP) -- the conventions of SPEC S:345-387.  Synchronous. */
int ara_risk_measures(ara_ctx *ctx, const float *ylt, uint32_t n_layers, uint64_t n_total,
                      uint32_t n_shards, int32_t layer, const double *rps, uint32_t n_rp,
                      double *pml_out, double *tvar_out);

/* ara_risk_measures plus VaR at each level q = 1 - 1/RP (SPEC S:373-381,
 * the `var` field of RiskMeasures; SURVEY NEXT-3 "VaR at arbitrary levels"):
 *   var_out    NULL or [n_rp] host: the VaR that TVaR averages above, i.e.
 *              the descending order statistic of rank ceil(N/RP) (integer RP;
 *              otherwise N - floor((1 - 1/RP) N) clamped to [1, N]).
 * Same arguments, errors and synchronisation as ara_risk_measures. */
int ara_risk_measures_var(ara_ctx *ctx, const float *ylt, uint32_t n_layers, uint64_t n_total,
                          uint32_t n_shards, int32_t layer, const double *rps, uint32_t n_rp,
                          double *pml_out, double *tvar_out, double *var_out);

/* ara_risk_measures_var for several tables of one YLT in one call: the
 * layers listed in layers[n_sel] (-1 = the roll-up), each by the joint
 * select, launched back to back with one read-back at the end (a multi-layer
 * portfolio's measures in one synchronisation instead of one per table).
 *   pml_out, tvar_out, var_out (NULL ok)  host [n_sel][n_rp]
 * n_rp in [1, 4]; other arguments and errors as ara_risk_measures. */
int ara_risk_measures_batch(ara_ctx *ctx, const float *ylt, uint32_t n_layers, uint64_t n_total,
                            uint32_t n_shards, const int32_t *layers, uint32_t n_sel, const double *rps,
                            uint32_t n_rp, double *pml_out, double *tvar_out, double *var_out);

/* ara_risk_measures_batch without the read-back: the same launches, enqueued
 * on the context stream, the results written to DEVICE memory and the call
 * returning at once (no host synchronisation) -- so consecutive analyses
 * (ARA_ASYNC runs + measures) queue back to back on the GPU.
 *   d_out   DEVICE fp64 [n_sel][n_rp][3], caller-allocated: (PML, TVaR, VaR)
 *           of table i, return period q at d_out[3 (n_rp i + q) + 0..2];
 *           valid once the stream reaches the launches (e.g. after
 *           ara_ctx_synchronize or an event / copy on that stream).
 * Arguments and argument errors as ara_risk_measures_batch; ARA_EINVAL also
 * for a host d_out. */
int ara_risk_measures_async(ara_ctx *ctx, const float *ylt, uint32_t n_layers, uint64_t n_total,
                            uint32_t n_shards, const int32_t *layers, uint32_t n_sel, const double *rps,
                            uint32_t n_rp, double *d_out);

/* The exceedance curve (SPEC ExceedanceCurve S:345-352) of one
 * layer's YLT, or of the roll-up over layers (layer = -1, G16): the losses
 * sorted descending, L(1) >= ... >= L(N); the empirical exceedance
 * probability of rank i is i/(N+1) (implicit).  A device radix sort.
 *   ylt         DEVICE fp32 [n_shards][n_layers][n_total/n_shards] (as ara_risk_measures)
 *   losses_out  DEVICE fp32 [n_total], caller-allocated
 * Asynchronous on the context stream.  ARA_EINVAL: empty YLT, n_total >= 2^32,
 * bad layer / shard layout, host pointers. */
int ara_exceedance_curve(ara_ctx *ctx, const float *ylt, uint32_t n_layers, uint64_t n_total,
                         uint32_t n_shards, int32_t layer, float *losses_out);

/* ---- component entry points (row-level parity tests) ------------------ */

/* Secondary-uncertainty loss draws for n independent
 * (record, z_(Prog,E), z_(E)) triples, on the device: record preparation
 * (incl. the quantile table) then one draw each.  All pointers
 * host; z values must lie in (0,1).  flags: 0, or ARA_EXACT to solve each
 * quantile in fp64 instead of using the table.  loss_out[n] host.
 * ARA_ECONVERGE as ara_run. */
int ara_sample_losses(ara_ctx *ctx, uint64_t n, const ara_record *records,
                      const float *z_prog, const float *z_event, uint32_t flags,
                      float *loss_out);

/* Row a6's fp64 beta quantile on its own (readings G11-G13):
 * for each i, x_i = I^-1(Phi(v_i); alpha_i, beta_i), the x in (0,1) with
 * I_x(alpha, beta) = Phi(v), by the device's per-sample fp64 solve (the one
 * that builds the quantile tables and serves ARA_EXACT: Halley iteration on
 * the log of the matched tail in lambda = logit x, tails from the Gauss
 * hypergeometric series of DLMF 8.17.8).  x_out[i] = x and y_out[i] = 1 - x,
 * each to full relative precision (so both tails can be checked).
 *   alpha, beta  host [n], finite and > 0 (the sigma_beta-capped regime,
 *                ~1e-6, included)
 *   v            host [n], finite (the normal score of step 5)
 *   x_out, y_out host [n]
 * ARA_EINVAL on bad values; ARA_ECONVERGE (outputs written) if a solve did
 * not converge. */
int ara_beta_quantiles(ara_ctx *ctx, uint64_t n, const double *alpha, const double *beta, const double *v,
                       double *x_out, double *y_out);

/* The uniforms the path draws (reading G2/G4): for each of n (trial i,
 * occurrence k, id, tag) counters, U(lane 0 of Philox4x32-10(seed, ctr)).
 * ctr: host [n][4] uint32 (i, k, program-or-XELT id, tag 1|2); out host [n]. */
int ara_draw_uniforms(ara_ctx *ctx, uint64_t seed, uint64_t n, const uint32_t *ctr,
                      float *u_out);

/* Step 2 of section 3.2 (reading G1): the standard normal
 * v = Phi^-1(U(x)) the sampler takes from a Philox output word x, with
 * U(x) = (2(x >> 9) + 1) 2^-24 (G4), evaluated on the smaller tail as the
 * kernels do.  bits: host [n] uint32 words; v_out: host [n] (fp32). */
int ara_normal_quantiles(ara_ctx *ctx, uint64_t n, const uint32_t *bits, float *v_out);

#ifdef __cplusplus
}
#endif
#endif /* ARA_H */
