/*
 * optfuse_b200.h -- C ABI of the B200 (sm_100a) fused-optimizer kernel library.
 *
 * This is the drop-in boundary for the hot path of Optimizer Fusion
 * (arXiv 2104.00237).  The reference (`optfuse`, pure Python/numpy) has no FFI;
 * its plugin boundary is the Python method
 *
 *     OptimizerPolicy.step(param, step_t=None, trace=None)
 *         /root/reference/pkg/src/optfuse/optim.py:74-115  (contract + axpy)
 *         /root/reference/pkg/src/optfuse/optim.py:117-148 (_delta per kind)
 *         /root/reference/pkg/src/optfuse/tensor.py:140-144 (axpy_inplace)
 *
 * and the global-information transform
 *
 *     clip_by_global_norm(graph, max_norm)
 *         /root/reference/pkg/src/optfuse/optim.py:151-172
 *
 * Every entry point below takes plain device pointers, element counts, host
 * scalars and a CUDA stream (as `void*`, i.e. a `cudaStream_t`).  No torch
 * types cross this boundary.  Ownership: the caller owns every buffer; the
 * library never allocates, frees or synchronises.  Errors are returned as an
 * `of_status`; invalid arguments are rejected before anything is launched
 * (mirroring the reference's raise-before-mutate convention), and the
 * contract errors of the reference (SchedulingContractError,
 * GlobalInfoRequired, ConfigError) are raised by the host layer above this ABI
 * before it is called.  Thread-safety: all entry points are reentrant; the
 * only per-thread state is the last error message.
 *
 * Arithmetic contract: for kinds SGD..ADAM every element update performs the
 * exact IEEE-754 operation sequence of the reference's numpy code (one
 * correctly rounded f32/f64 operation per numpy operation, source order, no
 * FMA contraction), so results are bit-identical to the reference on the same
 * inputs.  Host scalars are passed as doubles exactly as Python holds them and
 * are rounded to the tensor precision once, as numpy >= 2 (NEP 50) does.
 */
#ifndef OPTFUSE_B200_H
#define OPTFUSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI 3: grad_scale_dev of of_policy_step_mt is untyped (f32, or f64 with
 * OF_FLAG_SCALE_F64); of_mc_bucket carries dtypes; of_wgrad_step.
 * ABI 4: of_dp_sqnorm_peer (global-norm clipping on the peer transport). */
#define OF_ABI_VERSION 4

typedef enum of_status {
  OF_OK = 0,
  OF_ERR_INVALID = 1,      /* bad argument; nothing was launched */
  OF_ERR_UNSUPPORTED = 2,  /* dtype/kind/flag combination not built */
  OF_ERR_CUDA = 3          /* the CUDA runtime rejected a launch */
} of_status;

typedef enum of_dtype {
  OF_F32 = 0,
  OF_F64 = 1,
  OF_BF16 = 2
} of_dtype;

/* optim.py:22 KINDS (minus "newton", which has no per-parameter step,
 * optim.py:82-83) plus AdamW (decoupled decay, torch.optim.AdamW semantics;
 * not in the reference). */
typedef enum of_kind {
  OF_SGD = 0,           /* optim.py:119-120 */
  OF_SGD_MOMENTUM = 1,  /* optim.py:121-125 */
  OF_ADAGRAD = 2,       /* optim.py:126-129 */
  OF_RMSPROP = 3,       /* optim.py:130-133 */
  OF_ADADELTA = 4,      /* optim.py:134-140 */
  OF_ADAM = 5,          /* optim.py:141-148 (coupled weight decay) */
  OF_ADAMW = 6          /* torch.optim.AdamW(foreach=False) formula */
} of_kind;

/* step flags */
#define OF_FLAG_ZERO_GRAD 0x1u   /* write grad = 0 after reading it (optim.py:111) */
#define OF_FLAG_SHADOW_BF16 0x2u /* also write a bf16 copy of the new parameter */
#define OF_FLAG_DEVICE_STEP 0x4u /* read the step index on the device (see of_hparams) */
#define OF_FLAG_SCALE_F64 0x8u   /* grad_scale_dev points to a double (ABI 3) */

/* Hyper-parameters of one policy step (optim.py:42-51).  Scalars are the
 * Python doubles; the library rounds them to the tensor precision. */
typedef struct of_hparams {
  int32_t kind;            /* of_kind */
  int32_t max_ctas;        /* launch at most this many CTAs (0 = fill the GPU): a
                              backward-fusion update on a side stream keeps most
                              SMs free for the backward it overlaps */
  double eta;              /* step size */
  double alpha;            /* momentum decay */
  double weight_decay;     /* coupled for SGD..ADAM (optim.py:102-104), decoupled for ADAMW */
  double epsilon;
  double beta1;
  double beta2;
  double rho;
  double bias_correction1; /* ADAM/ADAMW: 1 - beta1**t, in double (optim.py:145) */
  double bias_correction2; /* ADAM/ADAMW: 1 - beta2**t, in double (optim.py:146) */
  /* OF_FLAG_DEVICE_STEP (ABI 2): the step-dependent scalars are read on the
   * device when the kernel runs, so a launch captured into a CUDA graph stays
   * correct on every replay.  The step index is t = t_base + *step_offset_dev;
   * row t of step_table_dev (step_table_rows rows of 2 doubles) holds the
   * host's {1 - beta1**t, 1 - beta2**t}, and bias_correction1/2 are ignored.
   * Rows outside [1, step_table_rows) are clamped (the host keeps t inside). */
  const int64_t* step_offset_dev;
  const double* step_table_dev;
  int64_t step_table_rows;
  int64_t t_base;
} of_hparams;

/* A list of parameters updated by one launch.  Arrays live in HOST memory and
 * hold DEVICE pointers; they are read during the call only.  History slots
 * follow optim.py:24-31:
 *   SGD: none | SGD_MOMENTUM: state0=momentum | ADAGRAD: state0=sum_sq
 *   RMSPROP: state0=square_avg | ADADELTA: state0=square_avg, state1=acc_delta
 *   ADAM/ADAMW: state0=exp_avg, state1=exp_avg_sq
 * param/state dtype: OF_F32 or OF_F64.  grad dtype: same as param, or OF_BF16
 * with OF_F32 params (bf16 gradients into fp32 master weights). */
typedef struct of_tensor_list {
  int32_t n;               /* number of tensors, >= 0 */
  int32_t param_dtype;     /* of_dtype of param and state slots */
  int32_t grad_dtype;      /* of_dtype of grad */
  int32_t reserved;
  void* const* param;      /* [n] */
  void* const* grad;       /* [n] */
  void* const* state0;     /* [n] or NULL when the kind has no slot */
  void* const* state1;     /* [n] or NULL when the kind has < 2 slots */
  void* const* shadow;     /* [n] bf16 copies, required with OF_FLAG_SHADOW_BF16 */
  const int64_t* numel;    /* [n] element counts (0 allowed: skipped) */
} of_tensor_list;

int of_abi_version(void);
const char* of_status_string(int status);
/* Message of the last error returned on this thread ("" if none). */
const char* of_last_error(void);
/* Number of kernels this library has launched in this process (all threads). */
uint64_t of_launch_count(void);

/* One policy step over every tensor of `list` (OptimizerPolicy.step,
 * optim.py:74-115, applied to several parameters in one multi-tensor launch).
 * grad_scale_dev: NULL, or a device scalar multiplied into every gradient
 * before the update (the global-norm clip factor, optim.py:170): an f32 value,
 * or with OF_FLAG_SCALE_F64 an f64 value rounded once to the parameter
 * precision -- numpy scales f64 gradients by the double factor itself, f32
 * gradients by its f32 rounding, so f64 lists pass the double. */
int of_policy_step_mt(const of_tensor_list* list, const of_hparams* hp,
                      const void* grad_scale_dev, uint32_t flags, void* stream);

/* Convenience wrappers with the kind fixed (same semantics). */
int of_sgdm_mt(const of_tensor_list* list, double eta, double alpha, double weight_decay,
               const void* grad_scale_dev, uint32_t flags, void* stream);
int of_adam_mt(const of_tensor_list* list, double eta, double beta1, double beta2,
               double epsilon, double weight_decay, double bias_correction1,
               double bias_correction2, int decoupled_weight_decay,
               const void* grad_scale_dev, uint32_t flags, void* stream);

/* *step_offset_dev += delta on `stream` (one thread): the first node of a
 * captured iteration, advancing the device step index of OF_FLAG_DEVICE_STEP
 * launches once per replay. */
int of_step_advance(int64_t* step_offset_dev, int64_t delta, void* stream);

/* ---- Data parallel over peer memory (NVLink / NVSwitch) ----------------
 * One bucket of a data-parallel model: every rank holds a flat gradient and a
 * flat parameter buffer of the same padded size, mapped into every peer's
 * address space (e.g. torch symmetric memory).  Rank r owns the elements
 * [shard_begin, shard_begin + shard_len) and their optimizer history. */
#define OF_MAX_PEERS 16

typedef struct of_peer_bucket {
  int32_t world;           /* W, 1 .. OF_MAX_PEERS */
  int32_t rank;            /* this rank */
  int32_t param_dtype;     /* OF_F32 / OF_F64, or OF_BF16 with an fp32 master shard */
  int32_t grad_dtype;      /* same as param_dtype */
  void* const* peer_grad;  /* [W] flat gradient buffers, as mapped on this GPU */
  void* const* peer_param; /* [W] flat parameter buffers, as mapped on this GPU */
  void* master;            /* OF_BF16: fp32 master of the shard; else NULL */
  void* state0;            /* history of the shard (optim.py:24-31 slots) */
  void* state1;
  int64_t shard_begin;     /* multiple of 4 */
  int64_t shard_len;       /* multiple of 4 */
} of_peer_bucket;

/* Reduce-scatter + policy step + all-gather of one bucket in ONE kernel: sums
 * the shard's gradients over the W peers (rank order), multiplies by
 * *grad_scale_dev (1/W; NULL = 1), applies OptimizerPolicy.step to the shard
 * (optim.py:74-148, same arithmetic as of_policy_step_mt), writes the new
 * parameter (bf16 rounding of the master for OF_BF16) into every peer's
 * parameter buffer and zeroes the shard's gradient in every peer.  The caller
 * orders it with a cross-rank barrier before (all gradients complete) and
 * after (all writes landed).  flags: 0 or OF_FLAG_DEVICE_STEP. */
int of_dp_step_peer(const of_peer_bucket* bucket, const of_hparams* hp,
                    const float* grad_scale_dev, uint32_t flags, void* stream);

/* Global-norm clipping for the peer transport (optim.py:151-172 under data
 * parallel): Sum over this rank's shard of (Sum_w grad_w)^2 -- the peers'
 * gradients summed in rank order exactly as of_dp_step_peer sums them --
 * accumulated in f64 with a fixed reduction order into *out_dev (added to it
 * when accumulate != 0).  The caller all-reduces the scalar over the ranks and
 * turns it into the clip factor with of_clip_coef.  Same barrier contract as
 * of_dp_step_peer (every peer's gradients complete); workspace as
 * of_sqnorm_mt.  Only world, rank, grad_dtype, peer_grad, shard_begin and
 * shard_len of the bucket are read. */
int of_dp_sqnorm_peer(const of_peer_bucket* bucket, double* workspace_dev, int64_t workspace_len,
                      double* out_dev, int accumulate, void* stream);

/* EXPERIMENTAL (not used by the data-parallel host layer; its numerics have
 * not run on a multi-GPU box yet).
 * The same bucket step over NVLink SHARP (NVLS) multicast: the shard's gradient is
 * read once through the multicast address with an in-switch sum
 * (multimem.ld_reduce), the new parameters and the zeroed gradient are written
 * once to every peer through multicast stores (multimem.st).  fp32 only.  The
 * switch's summation order is its own: bitwise equal to of_dp_step_peer at
 * world 1, tolerance-equal beyond.  Same barriers, flags and errors as
 * of_dp_step_peer (replaces the same reduce-scatter/all-gather pair). */
typedef struct of_mc_bucket {
  int32_t world;           /* W, 1 .. OF_MAX_PEERS */
  int32_t rank;
  int32_t param_dtype;     /* must be OF_F32 (anything else: OF_ERR_UNSUPPORTED) */
  int32_t grad_dtype;      /* must be OF_F32 */
  void* mc_grad;           /* multicast address of the flat gradient buffer */
  void* mc_param;          /* multicast address of the flat parameter buffer */
  void* local_param;       /* this rank's flat parameter buffer (unicast) */
  void* state0;            /* history of the shard */
  void* state1;
  int64_t shard_begin;     /* multiple of 4 */
  int64_t shard_len;       /* multiple of 4 */
} of_mc_bucket;

int of_dp_step_multicast(const of_mc_bucket* bucket, const of_hparams* hp,
                         const float* grad_scale_dev, uint32_t flags, void* stream);

/* dst[i] <- src[i] (nbytes[i] bytes each) for n tensors in one launch per 256
 * (multi-tensor copy; CUDA-graph forward fusion routes each replay's gradients
 * to the buffers the next replay's updates read with it). */
int of_copy_mt(void* const* dst, const void* const* src, const int64_t* nbytes, int n, void* stream);

/* Parity-harness helper (not on the update path): out[M][N] = a[M][K] @ b[K][N]
 * (row-major, contiguous) with the reference engine's fixed accumulation order
 * (tensor.py:91-105 matmul_arrays: out = 0; out += a[:, k] * b[k, :] for k ascending, every
 * product and sum correctly rounded), so the synthetic graphs' gradients are
 * bit-identical to the reference's.  dtype: OF_F32 or OF_F64; M <= 65535. */
int of_exact_matmul(const void* a, const void* b, void* out, int64_t M, int64_t K, int64_t N,
                    int dtype, void* stream);

/* ---- Consumer-fused backward fusion: weight-gradient GEMM + update --------
 * For a Linear layer y = x W^T (W: [out_features][in_features]) whose
 * backward has the output gradient dY [tokens][out_features] and the input X
 * [tokens][in_features] (bf16, row-major, 16-byte aligned), ONE kernel
 * computes dW = dY^T X on the tensor cores (tcgen05, fp32 accumulator in
 * TMEM) and applies OptimizerPolicy.step (optim.py:74-148; hp->kind, same
 * functors as of_policy_step_mt) to the fp32 parameter/master and history
 * tile by tile from the accumulator: the gradient is never written to memory
 * (unless grad_dump is given).  With OF_FLAG_SHADOW_BF16 the new parameter is
 * also written as bf16 to `shadow` (the module's weight).  The caller orders
 * the layer's input-gradient GEMM (the last reader of the old W) before it on
 * the same stream (Appendix B.2).  in_features must be a multiple of 32,
 * out_features of 8.  flags: OF_FLAG_SHADOW_BF16 | OF_FLAG_DEVICE_STEP. */
typedef struct of_wgrad_args {
  int64_t out_features;    /* M: rows of W */
  int64_t in_features;     /* N: columns of W */
  int64_t tokens;          /* T: rows of dY and X (the reduction) */
  const void* grad_out_rows; /* dY, bf16 [T][M] */
  const void* input;       /* X, bf16 [T][N] */
  void* param;             /* fp32 [M][N]: the parameter, or the master of a bf16 module */
  void* state0;            /* fp32 [M][N] history slots (optim.py:24-31) */
  void* state1;
  void* shadow;            /* bf16 [M][N], with OF_FLAG_SHADOW_BF16 */
  void* grad_dump;         /* NULL, or fp32 [M][N]: also store dW (parity checks) */
} of_wgrad_args;

int of_wgrad_step(const of_wgrad_args* args, const of_hparams* hp, uint32_t flags, void* stream);

/* Sum of squares of every grad in `list`, accumulated in f64 with a fixed
 * (deterministic) reduction order (optim.py:160-164).  Uses `workspace_dev`
 * (>= of_sqnorm_workspace_len() doubles).  Writes *out_dev = sum, or
 * *out_dev += sum when accumulate != 0 (stream-ordered, so chained calls over
 * several lists are deterministic). */
int64_t of_sqnorm_workspace_len(void);
int of_sqnorm_mt(const of_tensor_list* list, double* workspace_dev, int64_t workspace_len,
                 double* out_dev, int accumulate, void* stream);

/* norm = sqrt(*sqnorm_dev); factor = norm <= max_norm ? 1 : max_norm / norm
 * (optim.py:165-168, in double); *coef_dev = (float)factor (the f32 multiplier
 * numpy applies at optim.py:170); *factor_dev = factor when non-NULL. */
int of_clip_coef(const double* sqnorm_dev, double max_norm, float* coef_dev,
                 double* factor_dev, void* stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* OPTFUSE_B200_H */
