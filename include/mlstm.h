/*
 * mlstm.h -- C ABI of libmlstm.so: the data-parallel, mixed-precision training step of a
 * single-layer multiplicative-LSTM byte-level language model (Puri et al., arXiv 1808.01371).
 *
 * Citations: "P:L" = line L of the paper's PAPER.md (section in brackets); "S:L" = SPEC.md line L;
 * "Qn" = reading n in DESIGN.md (numbering follows SURVEY.md §8c).
 *
 * Conventions shared by every entry point
 *  - Plain C types only.  Pointers documented "device" must point to CUDA device memory of the
 *    device that was current when mlstm_init ran; "host" pointers to ordinary host memory.
 *  - One context per process per GPU (one process per GPU, torch.distributed for rendezvous).
 *  - Errors: every call returns an mlstm_status; on failure mlstm_last_error() returns a
 *    thread-local message.  Argument errors (MLSTM_EINVAL) have no side effects.  A CUDA or NCCL
 *    failure makes the context sticky-failed: every later call on it returns the same code.
 *    No C++ exception crosses this boundary.  There is no CPU fallback: without an sm_100a
 *    device mlstm_init fails with MLSTM_ECUDA.
 *  - Canonical parameter layout (flat, row-major, used by get/set_params, get_grads, opt state):
 *      E[256 x e] | W_mx[h x e] | W_mh[h x h] | W_x[4h x e] | W_h[4h x h] | b[4h] | W_dec[256 x h] | b_dec[256]
 *    with the 4h gate rows ordered i, f, o, u.  P = 5h^2 + 5he + 4h + 256e + 256h + 256.
 *    With weight_norm = 1 the four W slots hold the directions v and the gains follow b_dec:
 *      ... | b_dec[256] | g_mx[h] | g_mh[h] | g_x[4h] | g_h[4h]          (P grows by 10h, Q24)
 */
#ifndef MLSTM_H_
#define MLSTM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mlstm_ctx mlstm_ctx; /* opaque; owns host metadata, descriptors, NCCL comm */

typedef enum {
  MLSTM_OK = 0,
  MLSTM_EINVAL = 1,    /* bad argument or config; no side effects                      */
  MLSTM_ECUDA = 2,     /* CUDA failure or no sm_100a device; context becomes failed     */
  MLSTM_ENCCL = 3,     /* NCCL failure; context becomes failed                          */
  MLSTM_ENOMEM = 4,    /* workspace smaller than mlstm_workspace_bytes()                */
  MLSTM_ESTATE = 5,    /* call not valid in the context's current state                 */
  MLSTM_EDIVERGED = 6  /* diverge_patience consecutive steps with a non-finite loss or an
                          overflow at alpha = scale_min                          */
} mlstm_status;

enum { MLSTM_FP32 = 0, MLSTM_MIXED = 1 };                   /* precision   */
enum { MLSTM_LR_NONE = 0, MLSTM_LR_LINEAR = 1, MLSTM_LR_SQRT = 2 };
enum { MLSTM_ASYNC = 1u };                                  /* train_step flag: no host sync  */
enum { MLSTM_SLOT_TRAIN = 0, MLSTM_SLOT_EVAL = 1 };         /* persisted-state slots (Q5)     */

/* Model/optimiser configuration.  Defaults (mlstm_default_config) are the paper's 4096-d model
 * where the paper states a value and DESIGN.md's readings where it is silent. */
typedef struct {
  int32_t hidden;       /* h: mLSTM width; 4096. Must be a multiple of 64.       */
  int32_t embed;        /* e: byte-embedding width; paper silent, 64 (Q2). Multiple of 64.    */
  int32_t vocab;        /* must be 256: byte level                                */
  int32_t seq_len;      /* T: TBTT window, 256                                         */
  int32_t batch;        /* B: rows per rank ("local batch"); global batch = B * world   */
  int32_t micro_batch;  /* rows per micro-batch (0 = batch); must divide batch.  Each step runs the
                           forward/backward per micro-batch and accumulates gradients in fp32
                           (P:130), then one allreduce + one update (4096 rows/GPU)    */
  int32_t precision;    /* MLSTM_MIXED (fp16 storage/multiply, fp32 accumulate) or MLSTM_FP32   */
  int32_t weight_norm;  /* 0 or 1: weight normalisation of W_mx, W_mh, W_x, W_h (Q24):
                           w_r = g_r v_r / ||v_r|| per output row; v in the W slots of the
                           canonical layout, the 10h gains appended after b_dec; P grows by 10h  */
  uint64_t seed;        /* parameter init: counter-based SplitMix64, U(+-1/sqrt(cols)) (Q12)   */
  double lr0;           /* initial LR, 3e-3                                            */
  int64_t decay_iters;  /* linear decay to 0 over this many iterations, 100000         */
  double beta1, beta2, eps; /* Adam constants 0.9, 0.999, 1e-8 (Q11)                           */
  float scale_init, scale_min, scale_max; /* loss scale alpha: 2^16, 1, 2^24 (Q9)        */
  int32_t scale_growth_interval;          /* clean steps before alpha doubles, 2000 (Q9)        */
  int32_t diverge_patience;               /* MLSTM_EDIVERGED after this many, 50        */
  int32_t recurrence;  /* 0 = library default (one tcgen05 GEMM launch per timestep and GEMM, the
                          faster implementation as measured), 1 = the persistent
                          dataflow kernels (one launch for the T forward timesteps and one for BPTT;
                          mixed precision, 256 rows per micro-batch, h a multiple of 256 <= 4736,
                          otherwise the per-timestep path), 2 = per-timestep, 3 = persistent
                          forward with per-timestep BPTT.  MLSTM_RECUR=0/1 in the environment at
                          mlstm_init overrides (A/B measurements).                             */
} mlstm_config;

/* Result of one step; every field is the global value over all ranks. */
typedef struct {
  double loss_nats;   /* mean softmax cross-entropy over all B_g*T positions (Q7)      */
  double bpc;         /* loss_nats * log2(e)                                           */
  double lr;          /* learning rate the step used: lr0 * max(0, 1 - it/decay_iters) */
  float loss_scale;   /* alpha the step's backward used                                */
  int32_t skipped;    /* 1 if the update was skipped because the reduced gradients overflowed  */
  int64_t step;       /* iteration index `it` of this step (the LR clock, Q10)                 */
  int64_t applied;    /* Adam update count tau after this step (skipped steps excluded)        */
} mlstm_step_result;

/* Fills the defaults described above with hidden=4096, embed=64, seq_len=256, batch=256. */
void mlstm_default_config(mlstm_config* cfg);

/* Parameter count P for the config (canonical layout above). */
int64_t mlstm_param_count(const mlstm_config* cfg);

/* Device workspace the caller must allocate (e.g. torch.empty(uint8, device=cuda)) and keep
 * alive, untouched, until mlstm_destroy.  Returns 0 for an invalid config. */
size_t mlstm_workspace_bytes(const mlstm_config* cfg);

/* The gradient allreduce's bucket plan for `world` ranks (fp16 SUM of the weight gradients;
 * SURVEY 8(e)), host only: element ranges of the canonical gradient layout, in the order they are
 * reduced.  out: host int64 [cap][3] = (offset, count, after) per bucket, after = the work the bucket
 * waits for: 0 = dW_dec (computed before BPTT; the bucket is W_dec and b_dec and overlaps the backward),
 * 1 = the first row half of dW_h (units [0, h/2) of every gate; four contiguous ranges), 2 = dW_h,
 * 3 = dW_mh, 4 = every other gradient (end of the backward).  The buckets tile [0, P) exactly once.
 * world == 1, micro-batching or MLSTM_AR_OVERLAP=0: one bucket [0, P) after 4.  *n = number of
 * buckets; MLSTM_EINVAL if cap < *n (then *n is still set) or the config is invalid. */
mlstm_status mlstm_allreduce_plan(const mlstm_config* cfg, int32_t world, int64_t* out, int32_t cap, int32_t* n);

/* NCCL unique id for a multi-rank run (NCCL, no parameter server).  Rank 0 calls it
 * and broadcasts the 128 bytes to the other ranks (torch.distributed). */
mlstm_status mlstm_nccl_unique_id(uint8_t out[128]);

/* Creates a context on the current CUDA device.
 *  workspace: device, >= mlstm_workspace_bytes(cfg) bytes, 256-byte aligned, caller-owned.
 *  cuda_stream: cudaStream_t every kernel is enqueued on (NULL = legacy default stream).
 *  nccl_id: 128 bytes from mlstm_nccl_unique_id (same on all ranks); may be NULL iff world == 1.
 *  rank/world: this process's rank and the number of data-parallel ranks.  Rows of the global
 *  batch [rank*B, (rank+1)*B) belong to this rank ("distributed evenly").
 * Initialises fp32 master parameters (Q12), fp16 working copies, zero Adam moments and
 * zero persisted state (h, c) in both slots, and alpha = scale_init. */
mlstm_status mlstm_init(const mlstm_config* cfg, void* workspace, size_t workspace_bytes,
                        void* cuda_stream, const uint8_t* nccl_id, int rank, int world,
                        mlstm_ctx** out);

/* One training iteration:
 *   bytes: device, uint8 [B][T+1] row-major; inputs = bytes[:, 0:T], targets = bytes[:, 1:T+1]
 *          (Q6; consecutive windows of a row overlap by one byte).
 *   reset: device uint8 [B] or NULL; rows with reset[b] != 0 start from zero state.
 * Forward over T steps from the persisted train-slot state, softmax-CE, BPTT (truncated at the
 * window start), fp16 gradient SUM-allreduce over ranks, overflow check on the reduced buffer,
 * loss-scale update, unscale + Adam on fp32 masters, fp16 cast; the final (h, c) is persisted.
 * out: host; filled after the step completes (the call synchronises the stream) unless
 * MLSTM_ASYNC is set: then the call only enqueues the step and returns, and *out (which must stay
 * valid) is filled, in step order, by the next synchronising call (mlstm_sync, a train_step without
 * the flag, or a 9th outstanding async step, which delivers the oldest).  Up to 8 async results are
 * kept in a pinned ring; each delivered result runs the divergence detector, so an async run still
 * returns MLSTM_EDIVERGED (from the delivering call).
 * Input buffers must stay valid until the step has executed on the stream. */
mlstm_status mlstm_train_step(mlstm_ctx* ctx, const uint8_t* bytes, const uint8_t* reset,
                              uint32_t flags, mlstm_step_result* out);

/* Waits for every outstanding MLSTM_ASYNC step and fills their results (oldest first).  Returns the
 * first failure among them (e.g. MLSTM_EDIVERGED) after all were delivered; MLSTM_OK if none. */
mlstm_status mlstm_sync(mlstm_ctx* ctx);

/* Same step, end to end from HOST buffers: host bytes [B][T+1] (and optional host reset [B])
 * are copied to the device inside the call; the result struct is copied back and the stream is
 * synchronised before returning. */
mlstm_status mlstm_train_step_host(mlstm_ctx* ctx, const uint8_t* bytes_host,
                                   const uint8_t* reset_host, mlstm_step_result* out);

/* Forward-only evaluation of one window of Be <= micro-batch rows from the eval-slot state (state
 * persisted across evaluation minibatches; no update).  bytes: device uint8 [Be][T+1].  reset: device
 * uint8 [Be] or NULL: 0 = continue the row's state, 1 = start it from zero, 2 = idle row (state
 * reset, its positions not counted; the data loader's rows without a shard, mlstm_data.h).
 * Outputs (host, any may be NULL): nats_sum = global sum of per-position CE (all ranks), tokens =
 * counted positions (T per row with reset != 2, all ranks), bpc = nats_sum/tokens*log2(e) (0 if no
 * tokens). */
mlstm_status mlstm_eval(mlstm_ctx* ctx, const uint8_t* bytes, int32_t Be, const uint8_t* reset,
                        double* nats_sum, int64_t* tokens, double* bpc);

/* Pure functions (no context). */
double mlstm_lr_at(double lr0, int64_t it, int64_t decay_iters);
double mlstm_scale_lr(double base_lr, int rule, int64_t batch, int64_t ref_batch);
double mlstm_bpc_from_nats(double nats);

/* Host copies in the canonical layout (fp32, P elements).  Synchronous. */
mlstm_status mlstm_get_params(mlstm_ctx* ctx, float* host_out);
mlstm_status mlstm_set_params(mlstm_ctx* ctx, const float* host_in);  /* also recasts fp16  */
/* Gradient of the last train step: global mean over ranks, unscaled by that step's alpha,
 * canonical layout, fp32 (read back from the reduced fp16 (mixed) / fp32 buffer). */
mlstm_status mlstm_get_grads(mlstm_ctx* ctx, float* host_out);

/* Persisted state of a slot (MLSTM_SLOT_TRAIN / MLSTM_SLOT_EVAL): h and c, fp32 [batch][h] each. */
mlstm_status mlstm_get_state(mlstm_ctx* ctx, int slot, float* h_out, float* c_out);
mlstm_status mlstm_set_state(mlstm_ctx* ctx, int slot, const float* h_in, const float* c_in);

/* Optimiser + scaler state: Adam moments m, v (fp32 [P] each, canonical), tau (applied
 * updates), alpha, clean-step counter, and the LR clock `it`. */
mlstm_status mlstm_get_opt_state(mlstm_ctx* ctx, float* m_out, float* v_out, int64_t* tau,
                                 float* alpha, int32_t* clean_steps, int64_t* it);
mlstm_status mlstm_set_opt_state(mlstm_ctx* ctx, const float* m_in, const float* v_in,
                                 int64_t tau, float alpha, int32_t clean_steps, int64_t it);

/* Debug read of an internal buffer of the LAST train step (last micro-batch), converted to fp32 on
 * the host.  name: "m" / "a" (the recurrence's stashes m_t = (W_mx x_t) . a_t and a_t = W_mh h_{t-1},
 * [T][B][h], as the hot path wrote them), "logits" ([T][B][256]), "h" ([T][B][h]), "c" ([T][B][h]),
 * "loss_rows" (per-position CE [T][B]), "tab" ([256][5h] input-projection table), "onehot"
 * ([256][T][B]), "x" (E16[bytes] gathered by a debug-only kernel, [T][B][e]).
 * n: capacity of host_out in floats; MLSTM_EINVAL if too small or name unknown. */
mlstm_status mlstm_debug_dump(mlstm_ctx* ctx, const char* name, float* host_out, size_t n);

/* Overflow predicate of the optimiser kernel, exposed for bit-exact testing: returns in
 * *flag whether any of the n elements of the device buffer is non-finite.  dtype: 0 = fp16,
 * 1 = fp32. */
mlstm_status mlstm_check_overflow(mlstm_ctx* ctx, const void* device_buf, int64_t n, int dtype,
                                  int32_t* flag);

/* Per-phase device time (CUDA events on the step stream) accumulated over train steps since the
 * last reset, in ms, when profiling is enabled.  Phase order: see mlstm_phase_name().  Enabling
 * or disabling re-records the step graph.  Returns the number of phases in *n_phases. */
mlstm_status mlstm_profile_enable(mlstm_ctx* ctx, int enable);
mlstm_status mlstm_phase_times(mlstm_ctx* ctx, double* ms_out, int32_t* launches_out,
                               int32_t* n_phases);
const char* mlstm_phase_name(int phase);

/* Number of kernel launches one train step enqueues (excluding NCCL). */
int32_t mlstm_launches_per_step(mlstm_ctx* ctx);

/* Which implementation runs the recurrence ("sequential nature"; north_star kernels (b), (c-1)):
 * 1 = the persistent dataflow kernels (mlstm_config.recurrence = 1 and a covered shape), 3 = the
 * persistent forward with per-timestep BPTT (recurrence = 3), 0 = one tcgen05 / SIMT GEMM launch per
 * timestep and GEMM.  -1 for a null context. */
int32_t mlstm_recurrence_kind(mlstm_ctx* ctx);

/* Diagnostics: times `iters` launches of the tensor-core GEMM engine on random fp16 operands
 * D[M x N] = A[M x K] B[N x K]^T (fp32 out), engine 1 = one CTA per 128-row tile, 2 = CTA pair
 * (cta_group::2) per 256-row tile, 3 = the library's own plan for the shape (CTA pairs with the
 * K loop split over a cluster when needed); bn = tile N (64/128/256; 0 = library's choice).  Allocates
 * and frees its own device buffers.  *ms = average device time per launch (CUDA events). */
mlstm_status mlstm_gemm_bench(int engine, int M, int N, int K, int bn, int iters, double* ms);

/* Diagnostics: intra-kernel timeline of the tensor-core GEMM kernels.  mlstm_trace_enable(cap)
 * installs a device buffer of cap records (0 disables); every GEMM CTA then appends one record of
 * 12 uint64: {epilogue tag, cta index, t_start, t_first_tma, t_first_data, t_acc_ready, t_reduced,
 * t_end, t_partial_reduce_done, t_tile_begin, t_tile_end, 0} (%globaltimer ns; 0 where not
 * applicable).  Tags: 1 F1, 2 F2, 3 B1, 4 B2, 5 decoder,
 * 6 dH_dec, 7 input table, 8 weight gradient, 9 split partial.  mlstm_trace_read copies up to
 * `capacity` records (12*capacity uint64) and resets the count. */
mlstm_status mlstm_trace_enable(int capacity);
mlstm_status mlstm_trace_read(uint64_t* out, int capacity, int* n);

const char* mlstm_last_error(void);
void mlstm_destroy(mlstm_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* MLSTM_H_ */
