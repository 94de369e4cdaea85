/*
 * beast_b200.h -- C ABI of the B200-native IMPALA learner-step library
 * (libbeast_b200.so).  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *  - Every pointer argument is CALLER-OWNED DEVICE memory unless stated
 *    otherwise; tensors are contiguous and time-major ((T, B, ...), batch on
 *    axis 1, rollout.py:116-144).  The library allocates nothing.
 *  - `stream` is a cudaStream_t (void* here); every entry point only enqueues
 *    work on it (stream-ordered, re-entrant, no host synchronisation).
 *  - Return value: BP_OK, or a BP_ERR_* code for argument / launch errors
 *    (bp_last_error() gives a thread-local message).  Data-dependent
 *    violations that the reference raises as exceptions are reported by
 *    OR-ing BP_STATUS_* bits into the device word `status` (nullable); the
 *    Python layer checks it and raises SchemaError / NonFiniteError.
 *
 * Each entry point names the reference function it replaces
 * (paths relative to /root/reference/pkg/src/beastpipe/).
 */
#ifndef BEAST_B200_H_
#define BEAST_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BP_OK 0
#define BP_ERR_ARG 1         /* bad shape / config argument  (reference: SchemaError, ValueError) */
#define BP_ERR_UNSUPPORTED 2 /* shape outside what the kernels handle */
#define BP_ERR_LAUNCH 3      /* CUDA launch / driver error */

/* device status word bits */
#define BP_STATUS_ACTION_RANGE 1u   /* action outside [0, A)       -> SchemaError  (vtrace.py:64-65, rollout.py:184-188) */
#define BP_STATUS_NONFINITE_IN 2u   /* NaN/inf in an input         -> NonFiniteError (vtrace.py:83-91) */
#define BP_STATUS_NEG_DISCOUNT 4u   /* discount < 0                -> SchemaError  (vtrace.py:109-110) */
#define BP_STATUS_NONFINITE_LOSS 8u /* non-finite total loss       -> NonFiniteError (vtrace.py:202-205) */
#define BP_STATUS_NONFINITE_GRAD 16u/* non-finite gradient         -> NonFiniteError (model.py:251-252) */
#define BP_STATUS_BATCH_NONFINITE 32u /* learner loss only: NaN/inf in a batch field (reward,
                                         behaviour logits) -> SchemaError in the learner step
                                         (validate_batch, rollout.py:189-192), NonFiniteError in
                                         compute_losses (vtrace.py:83-91) */
/* Learner loss (bp_learner_loss_f32): any violation in the batch also makes the total loss NaN,
 * so bp_rmsprop_clip_f32(reject_if_nonfinite = &losses[3]) rejects the step on every
 * data-parallel rank after the loss all-reduce. */

int bp_abi_version(void);
const char* bp_last_error(void);
/* number of kernels this library has launched in the process (bench evidence) */
unsigned long long bp_launch_count(void);

/* ---------------------------------------------------------------------------
 * V-trace
 * ------------------------------------------------------------------------- */

/* Fused log-softmax x2 + action gather + clipped rho/c + reverse scan + pg
 * advantages.  Replaces action_log_rhos (vtrace.py:51-69) followed by
 * vtrace_targets (vtrace.py:94-128); upstream TorchBeast vtrace.from_logits.
 *   behavior_logits, target_logits: (T, B, A) f32;  actions: (T, B) int64
 *   discounts, rewards, values: (T, B) f32;  bootstrap_value: (B) f32
 *   clip_rho   : rho_bar (delta clip).           INFINITY = no clip (upstream None)
 *   clip_pg_rho: clip for pg advantages.         beastpipe uses clip_rho here
 *   clip_c     : c_bar (trace cut). upstream fixes 1.0
 * Outputs (T, B) f32: vs, pg_advantages, log_rhos, behavior_logp, target_logp
 * (the last three nullable).  A <= 48, T*min(B,16) <= 6144. */
int bp_vtrace_from_logits_f32(const float* behavior_logits, const float* target_logits,
                              const int64_t* actions, const float* discounts,
                              const float* rewards, const float* values,
                              const float* bootstrap_value, int T, int B, int A,
                              float clip_rho, float clip_pg_rho, float clip_c, float* vs,
                              float* pg_advantages, float* log_rhos, float* behavior_logp,
                              float* target_logp, unsigned* status, void* stream);

/* V-trace from given log importance weights.  Replaces vtrace_targets
 * (vtrace.py:94-128); upstream vtrace.from_importance_weights.
 * clipped_rhos (nullable) receives min(clip_rho, exp(log_rho)) (VtraceResult.clipped_rhos). */
int bp_vtrace_from_importance_weights_f32(const float* log_rhos, const float* discounts,
                                          const float* rewards, const float* values,
                                          const float* bootstrap_value, int T, int B,
                                          float clip_rho, float clip_pg_rho, float clip_c,
                                          float* vs, float* pg_advantages,
                                          float* clipped_rhos, unsigned* status, void* stream);

/* ---------------------------------------------------------------------------
 * Fused learner loss: V-trace + policy-gradient / baseline / entropy losses
 * and their exact gradients in one kernel.  Replaces compute_losses
 * (vtrace.py:224-255) = action_log_rhos + vtrace_targets + losses_from_targets
 * (vtrace.py:169-221); upstream learn()'s from_logits + compute_*_loss + autograd.
 *
 *   learner_logits  : (T, B, A) f32  rows 0..T-1 of the network output
 *   learner_baseline: (T+1, B) f32   values = rows 0..T-1, bootstrap = row T
 *   behavior_logits : (T, B, A) f32  already row-aligned by the caller
 *                     (beastpipe: policy_logits[:-1]; TorchBeast: [1:])
 *   actions         : (T, B) int64   aligned like behavior_logits
 *   rewards         : (T, B) f32     reward[1:]
 *   done            : (T, B) uint8   done[1:] (bool storage); discount is
 *                     (float)discount * !done exactly (vtrace.py:246)
 *   reward_clip     : 1 = clamp rewards to [-1, 1] (upstream abs_one)
 * Outputs
 *   d_logits  : (T, B, A) f32   d total / d learner_logits
 *   d_baseline: (T+1, B) f32    d total / d learner_baseline, row T = 0
 *   vs, pg_advantages, clipped_rhos: (T, B) f32, nullable (clipped_rhos = min(rho_bar, rho),
 *               VtraceResult.clipped_rhos vtrace.py:128)
 *   losses    : 4 doubles on device: pg, baseline(0.5*sum sq), entropy(-sum H), total
 *   workspace : bp_learner_loss_workspace_bytes(T, B, A) bytes, zeroed ONCE by
 *               the caller before first use (the kernel leaves it zeroed). */
size_t bp_learner_loss_workspace_bytes(int T, int B, int A);
int bp_learner_loss_f32(const float* learner_logits, const float* learner_baseline,
                        const float* behavior_logits, const int64_t* actions,
                        const float* rewards, const uint8_t* done, int T, int B, int A,
                        float discount, float clip_rho, float clip_pg_rho, float clip_c,
                        float pg_cost, float baseline_cost, float entropy_cost, int reward_clip,
                        float* d_logits, float* d_baseline, float* vs, float* pg_advantages,
                        float* clipped_rhos, double* losses, void* workspace, unsigned* status,
                        void* stream);

/* ---------------------------------------------------------------------------
 * Optimiser: global-norm clip + RMSProp (eps outside the root, no momentum)
 * ------------------------------------------------------------------------- */

/* Sum of squares of n f32 gradients into *sumsq (device double), deterministic.
 * Replaces the norm in clip_global_norm (model.py:224-228). workspace:
 * bp_sumsq_workspace_bytes(n), zeroed once. */
size_t bp_sumsq_workspace_bytes(int64_t n);
int bp_sumsq_f32(const float* x, int64_t n, double* sumsq, void* workspace, void* stream);

/* In-place clip + RMSProp over flat buffers of n elements.  Replaces
 * SharedModel.apply_gradients (pipeline.py:247-251) = clip_global_norm
 * (model.py:224-233) + rmsprop_step (model.py:236-268).
 *   clip_mode 0: beastpipe -- scale = max_norm/norm only if max_norm > 0 and norm > max_norm
 *   clip_mode 1: torch clip_grad_norm_ -- scale = min(1, max_norm/(norm + 1e-6))
 *   clip_mode 2: no clipping
 * The norm is read from *sumsq on the device (no host sync); a non-finite
 * norm rejects the whole step (params untouched, BP_STATUS_NONFINITE_GRAD); so does a
 * non-finite *reject_if_nonfinite (nullable: the step's f64 total loss).
 * square_avg and params are updated in place; grads are overwritten with the
 * clipped gradients when write_clipped_grads != 0 (torch semantics).
 * norm_out (nullable, device f32) receives the pre-clip norm.  lr is read
 * from *lr_dev when non-null (device-side LR schedule), else `lr`.
 * bf16_mirror (nullable, n bf16) receives the updated parameters in bf16 (the
 * GEMM operand copy of BpAtariNet.wbf), fused into the same pass. */
int bp_rmsprop_clip_f32(float* params, float* grads, float* square_avg, int64_t n,
                        const double* sumsq, float max_norm, int clip_mode, float lr,
                        const float* lr_dev, float alpha, float eps, int write_clipped_grads,
                        float* norm_out, void* bf16_mirror, unsigned* status,
                        const double* reject_if_nonfinite, void* stream);

/* ---------------------------------------------------------------------------
 * Loss helpers (north-star: upstream monobeast compute_policy_gradient_loss /
 * compute_baseline_loss / compute_entropy_loss, sum-reduced; in-tree arithmetic
 * beastpipe losses_from_targets vtrace.py:169-221).  Forward: one HBM pass, the f32 loss
 * into *out (and the f64 sum into *out64, nullable), deterministic fixed-order reduction;
 * workspace: bp_loss_workspace_bytes() zeroed bytes, one per concurrently running call.
 * Backward: grad_out is the device f32 upstream gradient of the scalar loss; the result
 * overwrites d_logits [rows][A] / d_advantages [n].
 * pg: logits [rows][A] f32, actions [rows] int64 (out of range -> BP_STATUS_ACTION_RANGE,
 * treated as action 0), advantages [rows] f32 (no gradient, upstream detaches them).
 * ------------------------------------------------------------------------- */
size_t bp_loss_workspace_bytes(void);
int bp_pg_loss_f32(const float* logits, const int64_t* actions, const float* advantages, long long rows,
                   int A, float* out, double* out64, void* workspace, unsigned* status, void* stream);
int bp_baseline_loss_f32(const float* advantages, long long n, float* out, double* out64, void* workspace,
                         void* stream);
int bp_entropy_loss_f32(const float* logits, long long rows, int A, float* out, double* out64,
                        void* workspace, unsigned* status, void* stream);
int bp_pg_loss_bwd_f32(const float* logits, const int64_t* actions, const float* advantages, long long rows,
                       int A, const float* grad_out, float* d_logits, void* stream);
int bp_baseline_loss_bwd_f32(const float* advantages, long long n, const float* grad_out, float* d_advantages,
                             void* stream);
int bp_entropy_loss_bwd_f32(const float* logits, long long rows, int A, const float* grad_out,
                            float* d_logits, void* stream);

/* ---------------------------------------------------------------------------
 * AtariNet (north-star network; replaces the reference network seam
 * mlp_forward / mlp_backward / mlp_forward_backward, model.py:126-203).
 * All dense contractions run on tcgen05 tensor cores (bf16 operands, f32
 * accumulate).  The caller owns every buffer; sizes are given per field for
 * a capacity of `max_frames` frames (N = (T+1)*B rows).
 * ------------------------------------------------------------------------- */
typedef struct BpAtariNet {
  int num_actions; /* A in [1, 31] */
  int max_frames;  /* capacity N */
  int use_lstm;    /* 1: parameter layout with the LSTM core (bp_atari_lstm_*) */
  void* wbf;  /* bf16 mirror of the flat f32 parameters (GEMM operands) */
  void* whf;  /* [32][576] bf16 heads operand: [Wp | bp], [Wv | bv], zero rows */
  /* activations, bf16 */
  void* x0;   /* [N*441][64]  space-to-depth frames           */
  void* x1;   /* [N*100][128] conv1 out (space-to-depth 2)    */
  void* x2;   /* [N*81][64]   conv2 out                       */
  void* x3;   /* [N][3136]    conv3 out, (y, x, c) order      */
  void* core; /* [N][576]     [relu(fc) | clip(r) | onehot(a) | 1 | 0]  */
  /* relu masks (1 bit per activation element, same layout), u32 words */
  void* m1;   /* [N*100*4]  of x1 */
  void* m2;   /* [N*81*2]   of x2 */
  void* m3;   /* [N*98]     of x3 */
  void* mc;   /* [N*18]     of core */
  /* backward temporaries, bf16.  d_pre1/2/3 MUST be zeroed once at
   * allocation: their grid padding rows are never written. */
  void* g;      /* [N][64]      [d_logits | d_baseline | 0]  */
  void* d_fc;   /* [N][512]                                  */
  void* d_pre3; /* [N*81][64]   conv3 pre-activation grad    */
  void* d_pre2; /* [N*100][64]  conv2 pre-activation grad    */
  void* d_pre1; /* [N*441][32]  conv1 pre-activation grad    */
  void* ws;     /* f32 workspace, bp_atari_workspace_bytes()  */
  size_t ws_bytes;
  int flags;    /* BP_NET_* */
  /* nullable cudaEvent_t: the no-LSTM backward records it on the stream right after the fc
   * weight gradient (1.6 M of the 1.69 M parameters) is final in grads, before the conv data /
   * weight gradients -- the data-parallel learner all-reduces that bucket on a side stream
   * while the rest of the backward runs */
  void* fc_grad_ready;
} BpAtariNet;

/* flags: the forward does not materialise the bf16 X0 grid (conv1 reads the u8 frames on
 * chip); the backward then needs the same frame source: bp_atari_backward_frames.
 * (LSTM nets ignore it: bp_atari_lstm_backward reads X0.) */
#define BP_NET_NO_X0 1

/* f32 master parameter layout (flat, upstream AtariNet module order):
 * [0] conv1.weight, [1] conv1.bias, [2] conv2.weight, [3] conv2.bias, [4] conv3.weight,
 * [5] conv3.bias, [6] fc.weight, [7] fc.bias,
 * [8..15] (use_lstm only, else empty) core.weight_ih_l0 [4H][H], core.weight_hh_l0 [4H][H],
 *         core.bias_ih_l0 [4H], core.bias_hh_l0 [4H], the same four for layer 1 (H = 513+A,
 *         torch nn.LSTM layout and gate order i, f, g, o),
 * [16] policy.weight [A][513+A], [17] policy.bias, [18] baseline.weight [1][513+A],
 * [19] baseline.bias; offsets[20] = total count.
 * Conv / fc weights are stored in GEMM layout [Cout][K], K = (tap, channel):
 *   conv1 k = (dy*2+dx)*64 + ci*16 + ry*4 + rx   (ky = 4dy+ry, kx = 4dx+rx)
 *   conv2 k = (dy*2+dx)*128 + (py*2+px)*32 + c    (ky = 2dy+py, kx = 2dx+px)
 *   conv3 k = (dy*3+dx)*64 + c;   fc k = (y*7+x)*64 + c
 * (the Python module converts to / from the torch layouts in state_dicts). */
int64_t bp_atari_param_count(int num_actions, int use_lstm);
int bp_atari_param_offsets(int num_actions, int use_lstm, int64_t* offsets /* 21 */);
size_t bp_atari_workspace_bytes(int num_actions, int max_frames);
/* bf16 mirror of the f32 master parameters (needed after parameters change outside
 * bp_rmsprop_clip_f32 with a mirror output, e.g. after load / init) */
int bp_atari_pack_weights(const BpAtariNet* net, const float* params, void* stream);
/* Forward of n frames: frames u8 [n][4][84][84], reward [n], last_action [n] int64
 * -> logits [n][A] f32, baseline [n] f32.  Keeps the activations for backward. */
int bp_atari_forward(const BpAtariNet* net, int n, const uint8_t* frames, const float* reward,
                     const int64_t* last_action, const float* params, float* logits,
                     float* baseline, void* stream);
/* Debug: the next tcgen05 GEMM launch records per-tile role timestamps (SM clock64 cycles)
 * into buf[(cta * tiles + i) * 16 + event]: 0/1 producer, 2/3 MMA, 4/5 epilogue, 6/7 u8
 * converter (start / end of tile i of that CTA), 8/9 converter loop end / fence end.  buf = null cancels. */
int bp_gemm_trace_next(void* buf, int tiles, int skip);  /* skip: traced launch = the (skip+1)-th */
/* conv1 operand path: 1 (default) builds 128B-swizzled bf16 windows on chip from the u8 frames
 * in shared memory; 2 builds im2col rows in tensor memory (the MMA reads A from TMEM);
 * 0 uses the bf16 X0 space-to-depth grid.  Results are identical.  on < 0 only queries.
 * Returns the previous setting.  (Test / A-B knob, process-global.) */
int bp_atari_set_conv1_u8(int on);
/* Conv weight-gradient path: 1 (default) = window kernel (one X window + dY box per K-block
 * feeds every m-tile of the CTA), 0 = per-tap operand boxes.  Identical sums in the same
 * order per split; the split plan differs.  on < 0 queries.  Returns the previous setting. */
int bp_atari_set_wgrad_window(int on);
/* Forward with frame-stack dedup: the frames are not shipped as [n][4][84][84]
 * but as a plane store planes u8 [num_planes][84][84] (one plane per env step) and
 * plane_index int32 [n][4]: channel c of frame i is planes[plane_index[i*4 + c]]
 * (indices are clamped to [0, num_planes)).  Results are bit-identical to bp_atari_forward
 * on the stacked frames.  Replaces the np.stack of stacked frames at enqueue
 * (rollout.py:116-144); upstream FrameStack semantics are built by
 * rollout.frame_stack_index. */
int bp_atari_forward_planes(const BpAtariNet* net, int n, const uint8_t* planes, const int32_t* plane_index,
                            int num_planes, const float* reward, const int64_t* last_action,
                            const float* params, float* logits, float* baseline, void* stream);
/* Actor inference (the PolyBeast / beastpipe inference loop body, pipeline.py:609-634:
 * mlp_forward + sample_actions): bp_atari_forward / bp_atari_forward_planes (plane_index
 * nullable) whose heads-GEMM epilogue also draws actions [n] int64 (Gumbel-max over the
 * row's logits in registers, same RNG and draws as bp_sample_actions_f32; greedy != 0 ->
 * argmax).  n is any batch size (the dynamic batch k).  seed_state (nullable) makes the
 * key device-resident for CUDA-graph replays: the call first advances *seed_state by one
 * splitmix64 step, then draws with the advanced value (seed is ignored). */
int bp_atari_forward_sample(const BpAtariNet* net, int n, const uint8_t* frames, const int32_t* plane_index,
                            int num_planes, const float* reward, const int64_t* last_action,
                            const float* params, uint64_t seed, uint64_t* seed_state, int greedy, float* logits, float* baseline,
                            int64_t* actions, void* stream);
/* Backward of the last forward: d_logits [n][A], d_baseline [n] -> grads (flat f32,
 * same layout as params; every entry is overwritten). */
int bp_atari_backward(const BpAtariNet* net, int n, const float* d_logits, const float* d_baseline,
                      const float* reward, const int64_t* last_action, float* grads, void* stream);
/* Backward of the last forward given its frame source again (frames, or the plane store +
 * plane index of bp_atari_forward_planes): the conv1 weight gradient converts the u8 frames
 * on chip, so a BP_NET_NO_X0 net never writes or reads the bf16 X0 grid. */
int bp_atari_backward_frames(const BpAtariNet* net, int n, const uint8_t* frames, const int32_t* plane_index,
                             int num_planes, const float* d_logits, const float* d_baseline, float* grads,
                             void* stream);

/* ---------------------------------------------------------------------------
 * LSTM core (AtariNet(use_lstm=True): upstream nn.LSTM(H, H, 2), H = 513 + A,
 * stepped per time row with the done reset core_state = notdone_t * core_state).
 * Input projections and weight / input gradients are tcgen05 GEMMs over all
 * N = T1*B rows.  The recurrence (default) runs on 16-CTA thread-block clusters, one
 * per 8 batch columns: each CTA holds its W_hh slice in registers as bf16 mma.sync
 * fragments and exchanges h / partial W_hh^T dz over DSMEM on mbarriers (bf16 W_hh,
 * h_{t-1} and dz operands, f32 accumulation and cell math).  The fallback
 * (bp_lstm_set_mode(1), or no 16-CTA clusters) is a pair of grid-cooperative kernels
 * with one grid barrier per step and W_hh resident in shared memory in f32.
 * G4 = 4H rounded up to a multiple of 128.  Buffers marked "zeroed once" must be
 * zero at allocation (padding columns are never written).
 * ------------------------------------------------------------------------- */
typedef struct BpLstmCore {
  int hidden;     /* H = 513 + A */
  int max_rows;   /* capacity N = T1 * B */
  void* wih;      /* [2][G4][576] bf16 [W_ih | b_ih + b_hh | 0], rows >= 4H zero   */
  float* gx;      /* [N][G4] input projection of the current layer            */
  float* gates;   /* [2][N][8H] per-step gate records (cluster path: [N][H][8]
                     {i, f, g, o, c, pad} f32; cooperative path: [N][4H] i,f,g,o) */
  float* cseq;    /* [2][N][H] cell states                                   */
  void* hprev;    /* [2][N][576] bf16 [notdone_t h_{t-1} | 1 | 0], zeroed once */
  void* out;      /* [2][N][576] bf16 [h_t | 1 | 0], zeroed once; out[1] feeds the heads */
  float* hx;      /* [2][H][32] recurrent exchange                           */
  float* part;    /* bp_lstm_partial_floats(H): cooperative-path exchange, or the
                     cluster path's packed W_hh fragments (written by the forward,
                     read by the backward of the same step)                */
  void* dgates;   /* [2][N][G4] bf16 pre-activation gate gradients per layer, zeroed once */
  float* dh;      /* [N][576] f32                                            */
  float* dx;      /* [N][576] f32                                            */
  float* wpart;   /* [2][2][G4][576] f32 weight-gradient GEMM outputs (W_ih, W_hh)
                     x (split-K parts)                                        */
} BpLstmCore;
size_t bp_lstm_partial_floats(int hidden);
/* Recurrence implementation: 0 auto (16-CTA cluster kernels with W_hh in registers and
 * DSMEM exchange when available, else the grid-cooperative kernels), 1 cooperative,
 * 2 cluster.  Process-wide; for tests and diagnostics. */
int bp_lstm_set_mode(int mode);
/* Diagnostics: how many 16-CTA recurrence clusters can be co-resident (8 batch columns each;
 * 7 on a 148-SM B200, so B <= 56 runs as one pass). */
int bp_lstm_cluster_capacity(void);
/* 1 if the LSTM recurrence currently runs on the cluster kernels (bf16 recurrent operands),
 * 0 if on the cooperative f32 kernels. */
int bp_lstm_cluster_active(void);
/* Diagnostics: per-step %globaltimer trace of CTA 0 of the recurrent kernels into
 * buf (device u64 [2][T1][4] + 2: forward phases, backward phases, forward start /
 * end of set-up); NULL disables. */
int bp_lstm_trace(void* buf);
/* Forward of T1*B frames through torso + LSTM core + heads.  done [T1*B] u8;
 * h0, c0 [2][B][H] f32 initial state (layer-major, torch (num_layers, B, H));
 * hN, cN [2][B][H] receive the final state.  B is split into recurrent passes of <= 32. */
int bp_atari_lstm_forward(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                          const uint8_t* frames, const float* reward, const int64_t* last_action,
                          const uint8_t* done, const float* params, const float* h0, const float* c0,
                          float* logits, float* baseline, float* hN, float* cN, void* stream);
/* bp_atari_lstm_forward on a deduplicated plane store (see bp_atari_forward_planes). */
int bp_atari_lstm_forward_planes(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                                 const uint8_t* planes, const int32_t* plane_index, int num_planes,
                                 const float* reward, const int64_t* last_action, const uint8_t* done,
                                 const float* params, const float* h0, const float* c0, float* logits,
                                 float* baseline, float* hN, float* cN, void* stream);
/* bp_atari_lstm_forward (plane_index nullable) with the fused action sampling of
 * bp_atari_forward_sample; T1 = 1 is the actor's per-step core_state update. */
int bp_atari_lstm_forward_sample(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                                 const uint8_t* frames, const int32_t* plane_index, int num_planes,
                                 const float* reward, const int64_t* last_action, const uint8_t* done,
                                 const float* params, const float* h0, const float* c0, uint64_t seed,
                                 uint64_t* seed_state, int greedy, float* logits, float* baseline, float* hN, float* cN,
                                 int64_t* actions, void* stream);
/* Backward of the last bp_atari_lstm_forward (same T1, B, done, c0): d_logits [N][A],
 * d_baseline [N] -> grads (flat, every entry overwritten).  The initial state gets no
 * gradient (upstream learn() feeds the actors' state as a constant). */
int bp_atari_lstm_backward(const BpAtariNet* net, const BpLstmCore* core, int T1, int B,
                           const float* d_logits, const float* d_baseline, const uint8_t* done,
                           const float* params, const float* c0, float* grads, void* stream);

/* Categorical sampling per row (Gumbel-max; Philox4x32-10 keyed by the 64-bit seed,
 * counter (row, column / 4) -> word column % 4, u = ((w >> 8) + 1/2) 2^-24, noise
 * -log(-log u)); greedy != 0 -> argmax.  Replaces sample_actions (model.py:218-221) /
 * upstream torch.multinomial(softmax(logits)).  logits [n][A] f32 -> actions [n] int64.
 * Draws are identical to the fused sampler of bp_atari_forward_sample for the same seed. */
int bp_sample_actions_f32(const float* logits, int n, int A, uint64_t seed, int greedy,
                          int64_t* actions, void* stream);
/* Infeed slot refill (DeviceInfeed.put; the reference stacks rollouts on the host,
 * rollout.py:116-144): on `stream`, wait for wait_event (nullable: the consumer released the
 * slot), copy `bytes` from pinned host src to device dst, record ready_event. */
int bp_infeed_put(void* dst, const void* src, size_t bytes, void* stream, void* wait_event,
                  void* ready_event);
/* Infeed consumer (DeviceInfeed.get / release): on `stream`, record release_event (nullable)
 * after the work enqueued so far, then wait for ready_event (the next slot's copy). */
int bp_infeed_get(void* stream, void* release_event, void* ready_event);
/* Learner-step stats read-back (monobeast learn() stats: losses + episode returns of the
 * finished episodes): packs losses [4] f64, done [tb] u8 and episode_return [tb] f32
 * (nullable) and the status word (nullable; read, then cleared for the next step) into
 * out = [32 B losses | 4 B status | 4 B seq | tb B done | tb * 4 B returns] in one launch.
 * sumsq (nullable): the step's squared gradient norm; a non-finite value with a finite total
 * loss (losses[3]) adds BP_STATUS_NONFINITE_GRAD, the verdict bp_rmsprop_clip_f32 reaches from
 * the same inputs -- so the pack can run concurrently with an update given status = NULL.
 * out may be device memory or pinned host memory (written through its unified-address
 * mapping: the step's result reaches the host without a separate copy).  seq_state
 * (nullable; 2 x u32 device memory, zeroed once) makes the pack publish a completion
 * sequence number in the seq word (1, 2, ... per call) after all its other writes are visible
 * system-wide: the host can spin on it instead of synchronising on an event. */
int bp_pack_stats(const double* losses, const uint8_t* done, const float* episode_return, int tb,
                  unsigned* status, const double* sumsq, unsigned* seq_state, void* out, void* stream);
/* n <= 8 asynchronous copies dsts[i] <- srcs[i] (bytes[i] each; device or mapped pinned memory)
 * on stream as one kernel launch (ActorInference's graph path stages its inputs with it). */
int bp_copy_many(void* const* dsts, const void* const* srcs, const size_t* bytes, int n, void* stream);
/* Host-side wait for a completion word in pinned host memory, e.g. the seq word of
 * bp_pack_stats: returns 0 once (*word - want) mod 2^32 < 2^31, 1 after timeout_us. */
int bp_host_wait_seq(const unsigned* word, unsigned want, long long timeout_us);
/* Shifted-tap GEMM test entry (the convolution form of the engine):
 * C[m][n] = sum_t sum_c A[m + offs[t]][c] * B[n][t*Cin + c]; window_mode 0 = one TMA box
 * per tap, 1 / 2 = one shared window per channel block (descriptor base offset 0 / row&7).
 * trace (nullable, device u64 [grid][trace_tiles][8]): per-tile %globaltimer events
 * (producer start/end, MMA start/end, epilogue start/end). */
int bp_gemm_shift_test(const void* A, const void* B, float* C, int R, int Cin, int N, int taps,
                       const int* offs, int window_mode, void* trace, int trace_tiles, void* stream);
/* Raw tcgen05 GEMM engine (test entry): C[M][N] = A . B^T, bf16 operands
 * (a_mn / b_mn select MN-major storage), f32 output (bf16 if out_bf16), split-K
 * partials at C + s*M*N. */
int bp_gemm_bf16_test(const void* A, const void* B, void* C, int M, int N, int K, int a_mn,
                      int b_mn, int splits, int out_bf16, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BEAST_B200_H_ */
