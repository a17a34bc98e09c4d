/*
 * cider.h — C ABI of the B200-native CIDER refinement decoder.
 *
 * This is the drop-in boundary for the reference's decoder hot path
 * (/root/reference/proj).  Every entry point replaces one reference
 * interface; the reference symbol it stands in for is cited beside it.
 *
 *   cider_denoise  = ura::StructuredDenoiser::logits          (denoiser.hpp:109-114, denoiser.cpp:253-259)
 *                    + module_b(..., incoming_out)            (denoiser.hpp:101-102)
 *   cider_refine   = ura::run_refinement                      (refine.hpp:60-62,  refine.cpp:199-205)
 *                    ura::run_with_remasking                  (refine.hpp:104-107, refine.cpp:277-292)
 *                    (rank mode: §7.1(3) adapter over ura::remask_pass, refine.cpp:238-275)
 *   cider_weights_init = ura::DenoiserParams::random_init     (denoiser.cpp:41-69), extended to
 *                    stacked layers / MLP width / attention
 *
 * Conventions (mirroring the reference's value-type API):
 *   - every buffer is caller-owned; host pointers unless the name says _device;
 *   - grids are K x L int32 row-major per bin (ura::SymbolGrid, grid.hpp:14-31), -1 = MASK;
 *   - evidence is L x Q fp32 row-major per bin (ura::EvidenceMatrix, grid.hpp:40-54);
 *   - logits are K x L x Q fp32 per bin (ura::LogitGrid, denoiser.hpp:28-40);
 *   - status: 0 ok, CIDER_EINVAL (3, -> std::domain_error), CIDER_ERUNTIME (4, -> std::runtime_error),
 *     the same exit-code mapping as uradec.cpp:817-829; cider_last_error() holds the message
 *     (thread-local), with the reference's prefixes ("denoiser failed at step t: ...").
 *   - calls on one context are serialised internally (one mutex + one CUDA stream), so a shared
 *     context is safe under concurrent callers, as Denoiser::logits is (uradec.cpp:184, 294-297).
 * There is no CPU fallback: every compute entry point fails with CIDER_ERUNTIME when no B200
 * (sm_100) device is present.
 */
#ifndef CIDER_H
#define CIDER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CIDER_OK 0
#define CIDER_EINVAL 3
#define CIDER_ERUNTIME 4

#define CIDER_FP32 0 /* SIMT fp32 GEMMs, fp32 activations: the parity mode */
#define CIDER_BF16 1 /* tcgen05 bf16 GEMMs with fp32 accumulation in TMEM: the throughput mode */

#define CIDER_REMASK_NONE 0
#define CIDER_REMASK_THRESHOLD 1 /* reference rule: rows with conf < phi_s (refine.cpp:245-252) */
#define CIDER_REMASK_RANK 2      /* floor(frac*K) lowest-confidence rows, ties -> lower row */

#define CIDER_MAX_THRESHOLDS 8

typedef struct cider_ctx cider_ctx;

/* Model hyper-parameters. Reference mode ("ref-exact") is layers=1, hidden=dim, heads=0:
 * exactly ura::DenoiserParams (denoiser.hpp:54-75). */
typedef struct {
    int m;               /* GF(2^m), Q = 2^m (gf.hpp:14-37) */
    uint32_t prim_poly;  /* 0 -> GfContext::default_prim_poly(m) (gf.cpp:8-20) */
    int dim;             /* D */
    int hidden;          /* H, TwoLayerMap hidden width (denoiser.hpp:44-50) */
    int layers;          /* N stacked Module A + Module B blocks (shared E, W, V) */
    int heads;           /* 0 = sum-pool Psi (denoiser.cpp:196-203); >0 = extrinsic pooling attention */
    double tau_demix;    /* denoiser.hpp:58 */
    double evidence_scale; /* beta_S, denoiser.hpp:59 */
    int precision;       /* CIDER_FP32 | CIDER_BF16 */
} cider_model_desc;

/* Parity-check matrix as (check, slot, coeff) triples (ura::ParityCheckMatrix, ldpc.hpp:23-47).
 * Any order; the library sorts by (check, slot) and validates like ldpc.cpp:11-30. */
typedef struct {
    int checks;
    int slots;
    int n_edges;
    const int32_t* edges; /* n_edges x 3 */
} cider_code_desc;

/* ura::RevealSchedule (refine.hpp:13-18). */
typedef struct {
    int steps;
    double tau_max;
    double tau_min;
    int first_reveal;
} cider_schedule;

/* ura::RemaskConfig (refine.hpp:33-36) plus the rank-selection mode of BASELINE config 3. */
typedef struct {
    int mode;                              /* CIDER_REMASK_* */
    int n_thresholds;
    double thresholds[CIDER_MAX_THRESHOLDS]; /* strictly descending, each in (0,1) */
    double rank_fraction;                  /* CIDER_REMASK_RANK: k_low = floor(rank_fraction*K) */
} cider_remask;

/* Per-bin slice of ura::RefineTrace (refine.hpp:48-54); every pointer nullable.
 * remask_rows / remask_steps are B x CIDER_MAX_THRESHOLDS (0 where a stage did not run);
 * remask_mask is B x K (1 = row re-decoded by the last remask stage that ran).
 * The reference's per-pass records: pass_first_reveals (B x (1 + CIDER_MAX_THRESHOLDS), the t = 1
 * reveal count of every pass run, in order; n_passes[b] of them are valid) = pass_first_reveals;
 * reveal_counts (B x max_steps, per step of the most recent pass, zero past its n_reveal_counts[b]
 * steps) = reveal_counts; first_step_sites (B x K x L, 1 = revealed at t = 1 of the most recent
 * pass) = first_step_sites as a mask (the reference lists the same (row, slot) pairs in row-major order). */
typedef struct {
    int32_t* first_reveals; /* B: reveal count of the first pass's t=1 step */
    int32_t* remask_rows;
    int32_t* remask_steps;
    int32_t* remask_mask;
    int32_t* pass_first_reveals;
    int32_t* n_passes;
    int max_steps;
    int32_t* reveal_counts;
    int32_t* n_reveal_counts;
    uint8_t* first_step_sites;
} cider_trace;

/* ---- weights (A15) -------------------------------------------------------------------- */
/* Flat layout, in draw order:
 *   embed (Q+1)xD | out_proj QxD | sym_embed QxD |
 *   per layer: gate_a {w1 Hx2D, b1 H, w2 DxH, b2 D} check_agg {w1 HxD, b1 H, w2 DxH, b2 D}
 *              fuse_b {w1 Hx2D, b1 H, w2 DxH, b2 D} |
 *   per layer (heads>0 only): attn_query D | attn_key DxD                                   */
size_t cider_weights_count(const cider_model_desc* model);
int cider_weights_init_f64(const cider_model_desc* model, uint64_t seed, double* out);
int cider_weights_init(const cider_model_desc* model, uint64_t seed, float* out);

/* ---- context -------------------------------------------------------------------------- */
int cider_create(const cider_model_desc* model, const float* weights, const cider_code_desc* code,
                 int device, cider_ctx** out);
void cider_destroy(cider_ctx* ctx);
const char* cider_last_error(void);
/* max bins resident per internal chunk (default: sized from free HBM); 0 = automatic */
int cider_set_chunk(cider_ctx* ctx, int max_bins_per_chunk);

/* ---- the path --------------------------------------------------------------------------- */
/* One denoiser forward for B bins of K rows (= Denoiser::logits). X: B x K x L int32 (-1 = MASK),
 * S: B x L x Q, logits: B x K x L x Q (nullable), incoming: B x layers x K x L x D (nullable;
 * the per-slot aggregated check messages of each layer, = module_b incoming_out). */
int cider_denoise(cider_ctx* ctx, int B, int K, const int32_t* X, const float* S, float* logits,
                  float* incoming);

/* Full refinement (+ remasking) for B bins of K rows (= run_refinement / run_with_remasking).
 * S: B x L x Q, grid: B x K x L. final_logits (nullable): B x K x L x Q logits of the last
 * final (gamma = 0) pass, as run_refinement's final_pass_logits out-param. */
int cider_refine(cider_ctx* ctx, int B, int K, const float* S, const cider_schedule* sched,
                 const cider_remask* remask, int32_t* grid, float* final_logits, cider_trace* trace);

/* One remask pass with the caller's row confidences (= ura::remask_pass, refine.hpp:97-100,
 * refine.cpp:238-275 — any ConfidenceScorer's score_rows): for B bins, rows k with
 * confidences[b*K + k] < threshold are masked and re-decoded for remask_steps(T, n_low, K) steps from
 * grid_in (B x K x L, symbols in [0, Q)); the other rows of grid_out are grid_in's, bit for bit.
 * final_logits (nullable, B x K x L x Q): the pass's gamma = 0 logits, written only for bins that had
 * a low row (the reference leaves final_pass_logits untouched otherwise). trace (nullable): the pass's
 * RefineTrace records (remask_rows / remask_steps stage 0, remask_mask = the low rows). */
int cider_remask_pass(cider_ctx* ctx, int B, int K, const float* S, const cider_schedule* sched,
                      const int32_t* grid_in, const double* confidences, double threshold, int32_t* grid_out,
                      float* final_logits, cider_trace* trace);

/* Teacher-forcing probe (test / diagnostic entry point): cider_refine over B host bins
 * (remask NONE or RANK) as ONE device chunk, recording for the n_probe bins probe_bins[] every denoiser
 * forward's input grid and output logits and every pass's output grid, in execution order. Record r
 * (r < *n_records <= max_records): meta[r] = {pass, t, steps, kind}; kind 0 = the forward of step t,
 * 1 = the gamma = 0 forward, 2 = the pass output after the final argmax (no logits). probe_X:
 * n_probe x max_records x K x L; probe_logits (nullable): n_probe x max_records x K x L x Q. */
int cider_refine_probe(cider_ctx* ctx, int B, int K, const float* S, const cider_schedule* sched,
                       const cider_remask* remask, int32_t* grid, int n_probe, const int32_t* probe_bins,
                       int max_records, int32_t* meta, int32_t* probe_X, float* probe_logits, int* n_records);

/* Ragged loads (the protocol's bins carry K_chi in 1..k_max, protocol.cpp:41-88):
 * B bins with loads[b] users each, S: B x L x Q; bins are bucketed by load and each bucket runs as
 * one device batch with sched_by_load[K-1] / remask_by_load[K-1] (nullable: no remasking), the
 * per-load tables of run_protocol's DecoderBank. grids: the bins' K x L grids concatenated in input
 * order (sum(loads) x L). Results equal per-bin cider_refine calls. */
int cider_refine_ragged(cider_ctx* ctx, int B, const int32_t* loads, const float* S, int k_max,
                        const cider_schedule* sched_by_load, const cider_remask* remask_by_load, int32_t* grids);

/* Same, with S and grid in device memory (allocated by cider_device_alloc); async on the
 * context stream; trace ignored. */
int cider_refine_device(cider_ctx* ctx, int B, int K, const float* S_device,
                        const cider_schedule* sched, const cider_remask* remask,
                        int32_t* grid_device);

/* ---- GF(Q) check-node update in the WHT domain --------------------- */
/* = ura::update_check_wht (bp.cpp:222-269) for n_checks checks of degree d at once: v2c and c2v are
 * n_checks x d x Q (fp64), coeffs n_checks x d; c2v[i] is the extrinsic message to edge i
 * (check_update_wht(gf, others, their coeffs, coeff_i), bp.cpp:128-149). Host buffers. */
int cider_check_update_wht(int m, int n_checks, int d, const double* v2c, const int32_t* coeffs, double* c2v,
                           int device);

/* ---- batched GF(Q) FFT-BP decoder -------------------------------------- */
/* A code-only context: GF(2^m) tables and the Tanner graph on one device. */
typedef struct cider_bp_ctx cider_bp_ctx;
/* ura::BpConfig (bp.hpp:20-25) with the WHT backend (bp.cpp:222-269). */
typedef struct {
    int max_iters;        /* >= 1 */
    double message_floor; /* > 0 */
    int early_exit;       /* stop a bin at its first zero-syndrome iteration */
} cider_bp_config;
int cider_bp_create(int m, uint32_t prim_poly, const cider_code_desc* code, int device, cider_bp_ctx** out);
void cider_bp_destroy(cider_bp_ctx* ctx);
/* = ura::bp_decode (bp.cpp:271-347) for B independent belief sets: lambda B x L x Q (fp64), hard B x L,
 * marginals B x L x Q (nullable), converged / iters B (nullable). Host buffers. */
int cider_bp_decode(cider_bp_ctx* ctx, int B, const double* lambda, const cider_bp_config* cfg, int32_t* hard,
                    double* marginals, int32_t* converged, int32_t* iters);
/* = ura::sic_decode (bp.cpp:349-368): S B x L x Q (fp64 evidence), grid B x K x L (rows in decode order),
 * stage_converged / stage_iters B x K (nullable). cancel_value NaN -> log(K/Q) (bp.cpp:352-353). */
int cider_sic_decode(cider_bp_ctx* ctx, int B, int K, const double* S, const cider_bp_config* cfg, double cancel_value,
                     int32_t* grid, int32_t* stage_converged, int32_t* stage_iters);

/* ---- batched AMP slot detector (the evidence the path consumes) --------- */
/* A dataset context: the per-slot sensing dictionaries (fixed per dataset, sim.hpp:60-62) on one
 * device. dicts: L x q x n_s complex (re, im interleaved), each slot column-major as
 * ura::SensingMatrix::cols (sim.hpp:18-26). */
typedef struct cider_amp_ctx cider_amp_ctx;
/* ura::AmpConfig (amp.hpp:14-19) */
typedef struct {
    int iters;             /* >= 1 */
    double rho_bg;         /* in (0, 1) */
    double sigma_u2;       /* > 0 */
    double evidence_floor; /* natural log */
} cider_amp_config;
int cider_amp_create(int L, int q, int n_s, const double* dicts, int device, cider_amp_ctx** out);
void cider_amp_destroy(cider_amp_ctx* ctx);
/* = ura::detect_frame (amp.cpp:133-148) for B independent frames: y B x L x n_s complex (interleaved),
 * S B x L x q (fp64 evidence rows = evidence_row(amp_detect(...)), amp.cpp:63-131). Host buffers.
 * Errors as the reference: 3 for an invalid config (std::domain_error), 4 for a non-finite residual
 * ("amp_detect: non-finite residual at iteration i", std::runtime_error). */
int cider_amp_detect(cider_amp_ctx* ctx, int B, const double* y, const cider_amp_config* cfg, double* S);

/* ---- device plumbing used by the benchmark (no PyTorch on the path) --------------------- */
int cider_device_count(int* n);
int cider_device_alloc(cider_ctx* ctx, size_t bytes, void** ptr);
int cider_device_free(cider_ctx* ctx, void* ptr);
int cider_host_alloc(size_t bytes, void** ptr); /* pinned */
int cider_host_free(void* ptr);
int cider_memcpy_h2d(cider_ctx* ctx, void* dst, const void* src, size_t bytes); /* async, ctx stream */
int cider_memcpy_d2h(cider_ctx* ctx, void* dst, const void* src, size_t bytes); /* async, ctx stream */
int cider_synchronize(cider_ctx* ctx);
int cider_flush_l2(cider_ctx* ctx); /* writes a buffer larger than L2 on the ctx stream */
/* CUDA events on the ctx stream: slot in [0, 64) */
int cider_event_record(cider_ctx* ctx, int slot);
int cider_event_elapsed(cider_ctx* ctx, int slot_a, int slot_b, float* ms);

/* Instrumentation: kernel launches issued by this context so far, and (when profiling is on)
 * per-kernel-class CUDA-event times accumulated on the ctx stream. */
int cider_set_profiling(cider_ctx* ctx, int on);
int64_t cider_launch_count(cider_ctx* ctx);
int cider_kernel_stats(cider_ctx* ctx, int idx, char* name, int name_len, int64_t* launches,
                       double* total_ms, double* flops, double* bytes);
int cider_reset_stats(cider_ctx* ctx);

/* ---- multi-GPU result gather (NCCL, the only collective on the path) --------------------- */
/* Debug guard bands — an out-of-bounds write check for the device kernels (compute-sanitizer is not
 * available on the GPU pool): after cider_set_debug_guard(ctx, bytes > 0) every workspace buffer is
 * allocated with `bytes`-byte 0xA5 bands before and after it (existing workspace, graphs and tensor
 * maps are dropped); cider_debug_check counts band bytes that were overwritten (0 = clean; the damaged
 * buffers are named in cider_last_error). cider_debug_poke is the positive control for tests. */
int cider_set_debug_guard(cider_ctx* ctx, size_t bytes);
int cider_debug_check(cider_ctx* ctx, int64_t* damaged_bytes);
int cider_debug_poke(cider_ctx* ctx, const char* buffer, int64_t offset_past_end);
/* decoded grids (int32, device) -> one byte per symbol (Q <= 256), async on the ctx stream: the
 * payload of the final gather (134 MB for all 262,144 c5 bins) */
int cider_grid_pack_u8(cider_ctx* ctx, const int32_t* grid_device, uint8_t* out_device, size_t n);
int cider_nccl_unique_id(char out[128]);
int cider_nccl_init(cider_ctx* ctx, const char id[128], int rank, int world);
/* all ranks contribute n_bytes from send_device; recv_device (n_bytes*world) filled on every rank */
int cider_nccl_allgather(cider_ctx* ctx, const void* send_device, void* recv_device, size_t n_bytes);

/* ---- host-side workload (BASELINE configs) and metrics ---------------------------------- */
typedef struct {
    int m;              /* GF(2^m) */
    int slots;          /* L */
    int checks;         /* P */
    int col_weight;     /* 3 */
    int k;              /* users per bin */
    double snr_db;
    double p_erase;
    double p_false;
    uint64_t master_seed; /* 0: H from derive_seed(0,1), bin b from derive_seed(0,16+b) */
} cider_workload_desc;

/* H = build_random_ldpc(gf, L, P, col_weight, make_rng(derive_seed(seed,1))) (uradec.cpp:45-52).
 * edges: L*col_weight x 3, sorted by (check, slot). */
int cider_workload_code(const cider_workload_desc* w, int32_t* edges);
/* Bins [first, first+n): truth (n x K x L, = sample_codewords) and S (n x L x Q fp32). */
int cider_workload_bins(const cider_workload_desc* w, const int32_t* edges, int64_t first, int n,
                        int32_t* truth, float* S, int threads);
/* The same bins generated on the device, into device buffers (truth_device n x K x L,
 * S_device n x L x Q, e.g. from cider_device_alloc): one thread per bin replays the host generator's
 * mt19937_64 stream and libstdc++ distributions; S equal to cider_workload_bins' up to the last ulp
 * of a double exp/log (float results identical in practice). Synchronous. */
int cider_workload_bins_device(const cider_workload_desc* w, const int32_t* edges, int64_t first, int n,
                               int32_t* truth_device, float* S_device, int device);
/* Parity-check files (= ura::save_parity_file / load_parity_file, ldpc.cpp:197-226).
 * load: edges (max_edges x 3, sorted (check, slot)) + header fields; a malformed or invalid file is
 * CIDER_ERUNTIME with the reference's messages ("load_parity_file: malformed header in ..."). */
int cider_save_parity_file(const char* path, const cider_code_desc* code, int q, int col_weight, uint32_t prim_poly,
                           uint64_t seed);
int cider_load_parity_file(const char* path, int max_edges, int32_t* edges, int* n_edges, int* checks, int* slots, int* q,
                           int* col_weight, uint32_t* prim_poly, uint64_t* seed);
/* ---- the reference's dataset format (dataset.hpp:19-99, dataset.cpp) ---------- */
/* ura::RunConfig (dataset.hpp:19-41); rho_bg / sigma_u2 < 0 = derive the default */
typedef struct {
    char scale[32];
    int q, l, p, col_weight, k, n_s;
    double eb_db, noise_var;
    int amp_iters;
    double rho_bg, sigma_u2, evidence_floor;
    uint64_t seed;
    int frames;
} cider_run_config;
/* = config_to_json (canonical: keys sorted, nlohmann::json's number layout) / config_fingerprint
 * (FNV-1a 64 of it, 16 hex digits + NUL) / file_fingerprint / format_double (shortest round trip) */
int cider_config_to_json(const cider_run_config* cfg, char* out, int cap);
int cider_config_fingerprint(const cider_run_config* cfg, char out[17]);
int cider_file_fingerprint(const char* path, char out[17]);
int cider_format_double(double x, char* out, int cap);
/* = load_dataset (dataset.cpp:176-220) of a JSON Lines dataset: the header's config and fingerprints,
 * *n_frames, and the first min(frames_cap, n) frames: seeds, truth (n x k x l), evidence (n x l x q,
 * fp64) and snr_db (each nullable). Call with frames_cap = 0 to size the buffers. Malformed or
 * inconsistent files fail with CIDER_ERUNTIME and the reference's messages. */
int cider_dataset_load(const char* path, cider_run_config* cfg, char fingerprint[17], char h_fingerprint[17],
                       int* n_frames, int frames_cap, uint64_t* seeds, int32_t* truth, double* evidence, double* snr_db);

/* Permutation-invariant SER/CER (= ura::ser_cer, metrics.cpp:124-145) summed over n bins. */
int cider_ser_cer(int n, int K, int L, const int32_t* truth, const int32_t* pred, double* ser_sum,
                  double* cer_sum);

#ifdef __cplusplus
}
#endif

#endif /* CIDER_H */
