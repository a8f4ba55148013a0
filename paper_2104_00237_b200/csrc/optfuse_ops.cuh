// optfuse_ops.cuh -- the update functors shared by every kernel of
// liboptfuse_b200.so (the multi-tensor step, the data-parallel peer and
// multicast steps, and the wgrad GEMM's fused epilogue).
//
// Each functor mirrors one branch of OptimizerPolicy._delta
// (/root/reference/pkg/src/optfuse/optim.py:117-148) plus the shared
// prologue/epilogue of OptimizerPolicy.step (optim.py:74-115): one correctly
// rounded IEEE operation per numpy operation, in numpy's order, no FMA
// contraction (the library is built with --fmad=false), constants rounded once
// to the tensor precision (NEP 50) -- so f32/f64 results are bit-identical to
// the reference.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>

#include "../../include/optfuse_b200.h"

namespace ofk {

// library-internal (defined in optfuse_kernels.cu)
extern std::atomic<uint64_t> g_launches;
extern thread_local char g_err[512];
int fail(int status, const char* fmt, ...);
int check_launch(const char* what);
int sm_count();

// ---------------------------------------------------------------------------
// Correctly rounded scalar ops (one IEEE operation per numpy operation).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float o_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float o_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float o_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float o_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float o_sqrt(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ float o_fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double o_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double o_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double o_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double o_div(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double o_sqrt(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ double o_fma(double a, double b, double c) { return __fma_rn(a, b, c); }

// ---------------------------------------------------------------------------
// Update functors.  Each mirrors one branch of OptimizerPolicy._delta plus the
// shared prologue/epilogue of OptimizerPolicy.step.  Constants are held in the
// tensor precision T (host rounds the Python double once, NEP 50).
// ---------------------------------------------------------------------------
template <class T>
struct CoupledWd {
  T wd;
  bool on;  // optim.py:103 `if self.weight_decay > 0`
  __device__ __forceinline__ T apply(T g, T p) const {
    return on ? o_add(g, o_mul(wd, p)) : g;  // g + wd * theta (new temp, optim.py:104)
  }
};

// Step-dependent scalars read on the device (OF_FLAG_DEVICE_STEP); only the
// Adam kinds have any.
struct StepSrc {
  const int64_t* offset;   // nullptr: host mode (constants already in the functor)
  const double* table;     // [rows][2] = {1 - beta1**t, 1 - beta2**t}
  int64_t rows;
  int64_t t_base;
};

template <class T>
struct SgdOp {  // optim.py:119-120
  static constexpr int kSlots = 0;
  __device__ __forceinline__ void set_step(double, double) {}  // step-independent
  CoupledWd<T> wd;
  T neg_eta;
  __device__ __forceinline__ void operator()(T& p, T g, T&, T&) const {
    g = wd.apply(g, p);
    p = o_add(p, o_mul(neg_eta, g));  // axpy_inplace(theta, 1.0, -eta*g)
  }
};

template <class T>
struct SgdMomentumOp {  // optim.py:121-125
  static constexpr int kSlots = 1;
  __device__ __forceinline__ void set_step(double, double) {}  // step-independent
  CoupledWd<T> wd;
  T neg_eta, alpha;
  __device__ __forceinline__ void operator()(T& p, T g, T& buf, T&) const {
    g = wd.apply(g, p);
    buf = o_mul(buf, alpha);        // buf *= alpha
    buf = o_add(buf, g);            // buf += g
    p = o_add(p, o_mul(neg_eta, buf));
  }
};

template <class T>
struct AdagradOp {  // optim.py:126-129
  static constexpr int kSlots = 1;
  __device__ __forceinline__ void set_step(double, double) {}  // step-independent
  CoupledWd<T> wd;
  T neg_eta, eps;
  __device__ __forceinline__ void operator()(T& p, T g, T& acc, T&) const {
    g = wd.apply(g, p);
    acc = o_add(acc, o_mul(g, g));
    p = o_add(p, o_div(o_mul(neg_eta, g), o_add(o_sqrt(acc), eps)));
  }
};

template <class T>
struct RmspropOp {  // optim.py:130-133
  static constexpr int kSlots = 1;
  __device__ __forceinline__ void set_step(double, double) {}  // step-independent
  CoupledWd<T> wd;
  T neg_eta, eps, rho, one_minus_rho;
  __device__ __forceinline__ void operator()(T& p, T g, T& sq, T&) const {
    g = wd.apply(g, p);
    sq = o_add(o_mul(rho, sq), o_mul(one_minus_rho, o_mul(g, g)));
    p = o_add(p, o_div(o_mul(neg_eta, g), o_add(o_sqrt(sq), eps)));
  }
};

template <class T>
struct AdadeltaOp {  // optim.py:134-140
  static constexpr int kSlots = 2;
  __device__ __forceinline__ void set_step(double, double) {}  // step-independent
  CoupledWd<T> wd;
  T neg_eta, eps, rho, one_minus_rho;
  __device__ __forceinline__ void operator()(T& p, T g, T& sq, T& acc) const {
    g = wd.apply(g, p);
    sq = o_add(o_mul(rho, sq), o_mul(one_minus_rho, o_mul(g, g)));
    T dx = o_mul(o_div(o_sqrt(o_add(acc, eps)), o_sqrt(o_add(sq, eps))), g);
    acc = o_add(o_mul(rho, acc), o_mul(one_minus_rho, o_mul(dx, dx)));
    p = o_add(p, o_mul(neg_eta, dx));
  }
};

template <class T>
struct AdamOp {  // optim.py:141-148
  static constexpr int kSlots = 2;
  CoupledWd<T> wd;
  T neg_eta, eps, beta1, beta2, one_minus_beta1, one_minus_beta2, bc1, bc2;
  __device__ __forceinline__ void operator()(T& p, T g, T& m, T& v) const {
    g = wd.apply(g, p);
    m = o_add(o_mul(beta1, m), o_mul(one_minus_beta1, g));
    v = o_add(o_mul(beta2, v), o_mul(one_minus_beta2, o_mul(g, g)));
    const T m_hat = o_div(m, bc1);
    const T v_hat = o_div(v, bc2);
    p = o_add(p, o_div(o_mul(neg_eta, m_hat), o_add(o_sqrt(v_hat), eps)));
  }
  // the host rounds the same doubles once (static_cast<T>)
  __device__ __forceinline__ void set_step(double c1, double c2) { bc1 = T(c1); bc2 = T(c2); }
};

// AdamW is not in the reference (SPEC.md:244 puts decoupled decay out of
// scope).  It follows torch.optim.AdamW(foreach=False) step by step:
//   param.mul_(1 - lr*wd); exp_avg.lerp_(grad, 1-beta1);
//   exp_avg_sq.mul_(beta2).addcmul_(grad, grad, value=1-beta2);
//   denom = exp_avg_sq.sqrt() / sqrt(bc2) + eps; param.addcdiv_(exp_avg, denom, -lr/bc1)
template <class T>
struct AdamWOp {
  static constexpr int kSlots = 2;
  T decay, w1, beta2, one_minus_beta2, bc2_sqrt, eps, neg_step;
  bool decay_on, w1_small;
  double eta;
  // same double expressions as the host side (sqrt and division are
  // correctly rounded on both), then one rounding to T
  __device__ __forceinline__ void set_step(double c1, double c2) {
    bc2_sqrt = T(__dsqrt_rn(c2));
    neg_step = T(-__ddiv_rn(eta, c1));
  }
  __device__ __forceinline__ void operator()(T& p, T g, T& m, T& v) const {
    if (decay_on) p = o_mul(p, decay);
    const T diff = o_sub(g, m);
    m = w1_small ? o_fma(w1, diff, m)                        // lerp, weight < 0.5
                 : o_fma(o_sub(w1, T(1)), diff, g);          // lerp, weight >= 0.5
    v = o_add(o_mul(v, beta2), o_mul(o_mul(one_minus_beta2, g), g));
    const T denom = o_add(o_div(o_sqrt(v), bc2_sqrt), eps);
    p = o_add(p, o_div(o_mul(neg_step, m), denom));
  }
};


template <class T>
CoupledWd<T> coupled(const of_hparams* hp) {
  return CoupledWd<T>{static_cast<T>(hp->weight_decay), hp->weight_decay > 0.0};
}

// Builds the functor of hp->kind (constants rounded once to T, as numpy does)
// and hands it to f.
template <class T, class F>
int with_op(const of_hparams* hp, F&& f) {
  const T neg_eta = static_cast<T>(-hp->eta);
  switch (hp->kind) {
    case OF_SGD: return f(SgdOp<T>{coupled<T>(hp), neg_eta});
    case OF_SGD_MOMENTUM: return f(SgdMomentumOp<T>{coupled<T>(hp), neg_eta, static_cast<T>(hp->alpha)});
    case OF_ADAGRAD: return f(AdagradOp<T>{coupled<T>(hp), neg_eta, static_cast<T>(hp->epsilon)});
    case OF_RMSPROP:
      return f(RmspropOp<T>{coupled<T>(hp), neg_eta, static_cast<T>(hp->epsilon),
                            static_cast<T>(hp->rho), static_cast<T>(1.0 - hp->rho)});
    case OF_ADADELTA:
      return f(AdadeltaOp<T>{coupled<T>(hp), neg_eta, static_cast<T>(hp->epsilon),
                             static_cast<T>(hp->rho), static_cast<T>(1.0 - hp->rho)});
    case OF_ADAM:
      return f(AdamOp<T>{coupled<T>(hp), neg_eta, static_cast<T>(hp->epsilon),
                         static_cast<T>(hp->beta1), static_cast<T>(hp->beta2),
                         static_cast<T>(1.0 - hp->beta1), static_cast<T>(1.0 - hp->beta2),
                         static_cast<T>(hp->bias_correction1), static_cast<T>(hp->bias_correction2)});
    case OF_ADAMW: {
      const double w1 = 1.0 - hp->beta1;
      return f(AdamWOp<T>{static_cast<T>(1.0 - hp->eta * hp->weight_decay), static_cast<T>(w1),
                          static_cast<T>(hp->beta2), static_cast<T>(1.0 - hp->beta2),
                          static_cast<T>(std::sqrt(hp->bias_correction2)), static_cast<T>(hp->epsilon),
                          static_cast<T>(-(hp->eta / hp->bias_correction1)),
                          hp->weight_decay != 0.0, std::fabs(w1) < 0.5, hp->eta});
    }
    default:
      return fail(OF_ERR_INVALID, "unknown optimizer kind %d", hp->kind);
  }
}

inline StepSrc step_source(const of_hparams* hp, uint32_t flags) {
  if (flags & OF_FLAG_DEVICE_STEP)
    return StepSrc{hp->step_offset_dev, hp->step_table_dev, hp->step_table_rows, hp->t_base};
  return StepSrc{nullptr, nullptr, 0, 0};
}


}  // namespace ofk
