// optfuse_kernels.cu -- sm_100a multi-tensor optimizer-update kernels behind the
// C ABI declared in include/optfuse_b200.h.
//
// What this replaces in the reference (/root/reference/pkg/src/optfuse):
//   OptimizerPolicy.step   optim.py:74-115   (coupled wd, _delta, grad reset, axpy)
//   OptimizerPolicy._delta optim.py:117-148  (one functor per kind below)
//   axpy_inplace           tensor.py:140-144 (theta += 1.0 * delta, fused)
//   clip_by_global_norm    optim.py:151-172  (sum of squares + factor; the factor
//                                             is folded into the update as a
//                                             device scalar, no second grad pass)
//
// Design (B200): the update is purely HBM-bound (20-28 algorithmic bytes per
// element, ~0.5 flop/byte), so the kernel is a grid-stride loop over fixed
// 4096-element tiles of a list of tensors whose pointers travel in the kernel
// parameter block (__grid_constant__, no metadata copy).  Each thread moves
// 128-bit vectors of every stream (theta, grad, history slots), issuing all of
// its loads for kUnroll vectors before any math so that each SM keeps tens of
// KB in flight.  The grid is sized to the SM count x resident CTAs.  Arithmetic
// uses explicit round-to-nearest intrinsics (no FMA contraction) in the exact
// order numpy evaluates the reference's expressions, so the result is
// bit-identical to the reference for f32 and f64.
#include "../../include/optfuse_b200.h"
#include "optfuse_ops.cuh"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace ofk {
std::atomic<uint64_t> g_launches{0};
thread_local char g_err[512] = "";

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int check_launch(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(OF_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return OF_OK;
}

int sm_count() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}
}  // namespace ofk

namespace {
using namespace ofk;

constexpr int kThreads = 256;
constexpr int kVec = 4;
#ifndef OF_UNROLL
#define OF_UNROLL 4
#endif
#ifndef OF_MIN_BLOCKS
#define OF_MIN_BLOCKS 1
#endif
#ifndef OF_UNROLL_BF16
#define OF_UNROLL_BF16 2
#endif
#ifndef OF_MIN_BLOCKS_BF16
#define OF_MIN_BLOCKS_BF16 4
#endif
#ifndef OF_CS
#define OF_CS 0
#endif
constexpr int kUnroll = OF_UNROLL;
constexpr int kTile = kThreads * kVec * kUnroll;  // elements per tile
constexpr int kCtasPerSm = 8;
constexpr int kCapMax = 256;                      // tensors per launch (param block)
constexpr int kSqnormWorkspace = 148 * 8 * 4;      // >= any sqnorm grid we launch


// ---------------------------------------------------------------------------
// Tensor-list parameter block.
// ---------------------------------------------------------------------------
template <int CAP>
struct MTParams {
  void* p[CAP];
  void* g[CAP];
  void* s0[CAP];
  void* s1[CAP];
  void* sh[CAP];
  int64_t n[CAP];
  int32_t tile_end[CAP];  // inclusive prefix sum of tiles per tensor
  int32_t count;
};

// Index of the tensor owning `tile`: binary search over the inclusive tile
// prefix sum, starting at `from` (tiles visited by one CTA only increase).
// With up to 256 tensors per launch a linear scan from 0 would cost a CTA
// hundreds of dependent parameter-bank loads before its first byte moves.
template <int CAP>
__device__ __forceinline__ int find_tensor(const MTParams<CAP>& mp, int from, int tile) {
  int lo = from, hi = mp.count - 1;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (tile < mp.tile_end[mid]) hi = mid; else lo = mid + 1;
  }
  return lo;
}

// 4-element vector loads/stores.
__device__ __forceinline__ void ld4(const float* p, float (&v)[4]) {
  const float4 t = *reinterpret_cast<const float4*>(p);
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void st4(float* p, const float (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const double2 b = reinterpret_cast<const double2*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void st4(double* p, const double (&v)[4]) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
}
__device__ __forceinline__ void ld4(const __nv_bfloat16* p, float (&v)[4]) {
  const uint2 t = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t.y));
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void st4_bf16(__nv_bfloat16* p, const float (&v)[4]) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
  __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
  uint2 t;
  t.x = *reinterpret_cast<uint32_t*>(&a);
  t.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = t;
}
__device__ __forceinline__ void st4_bf16(__nv_bfloat16* p, const double (&v)[4]) {
  const float f[4] = {(float)v[0], (float)v[1], (float)v[2], (float)v[3]};
  st4_bf16(p, f);
}
__device__ __forceinline__ void st4_zero(float* p) { *reinterpret_cast<float4*>(p) = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void st4_zero(double* p) {
  reinterpret_cast<double2*>(p)[0] = make_double2(0.0, 0.0);
  reinterpret_cast<double2*>(p)[1] = make_double2(0.0, 0.0);
}
__device__ __forceinline__ void st4_zero(__nv_bfloat16* p) { *reinterpret_cast<uint2*>(p) = make_uint2(0u, 0u); }

// Read-once streams (gradient, history) with the evict-first hint when
// OF_CS=1: they are not reused by anything that follows the update.
#if OF_CS
__device__ __forceinline__ void ld4s(const float* p, float (&v)[4]) {
  const float4 t = __ldcs(reinterpret_cast<const float4*>(p));
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void ld4s(const double* p, double (&v)[4]) {
  const double2 a = __ldcs(reinterpret_cast<const double2*>(p));
  const double2 b = __ldcs(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void ld4s(const __nv_bfloat16* p, float (&v)[4]) {
  const uint2 t = __ldcs(reinterpret_cast<const uint2*>(p));
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&t.y));
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
__device__ __forceinline__ void st4s(float* p, const float (&v)[4]) {
  __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
}
__device__ __forceinline__ void st4s(double* p, const double (&v)[4]) {
  __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
  __stcs(reinterpret_cast<double2*>(p) + 1, make_double2(v[2], v[3]));
}
#else
template <class P, class V> __device__ __forceinline__ void ld4s(const P* p, V (&v)[4]) { ld4(p, v); }
template <class P, class V> __device__ __forceinline__ void st4s(P* p, const V (&v)[4]) { st4(p, v); }
#endif

template <class T> __device__ __forceinline__ T ld1(const T* p) { return *p; }

// The gradient scale (global-norm clip factor, optim.py:170): an f32 device
// scalar, or with OF_FLAG_SCALE_F64 the f64 factor itself, rounded once to T
// (numpy multiplies an f64 gradient by the Python-double factor, an f32 one by
// its f32 rounding).
template <class T>
__device__ __forceinline__ T load_scale(const void* gscale, uint32_t flags) {
  if (gscale == nullptr) return T(1);
  if (flags & OF_FLAG_SCALE_F64) return static_cast<T>(*static_cast<const double*>(gscale));
  return static_cast<T>(*static_cast<const float*>(gscale));
}
__device__ __forceinline__ float ld1(const __nv_bfloat16* p) { return __bfloat162float(*p); }
template <class G> __device__ __forceinline__ void st1_zero(G* p) { *p = G(0); }
__device__ __forceinline__ void st1_zero(__nv_bfloat16* p) { *p = __float2bfloat16_rn(0.f); }

template <class T> struct GradVal { using type = T; };
template <> struct GradVal<__nv_bfloat16> { using type = float; };

__host__ __device__ __forceinline__ bool aligned(const void* p, unsigned a) {
  return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0;
}

// Per gradient type: vectors per thread per tile and the CTAs per SM the
// register budget must allow.  fp32/f64 gradients: 4 vectors in flight per
// thread at 2 CTAs/SM (measured best for VGG-16 / BERT); bf16 gradients (fp32
// master + bf16 shadow, 8 streams per element): 2 vectors at 4 CTAs/SM -- the
// 4-vector build needs 108 registers and stalls at 16 warps/SM (ncu: 52% of
// DRAM peak on ResNet-50), the 2-vector one reaches 0.80 of the copy peak.
template <class G> struct Tune {
  static constexpr int kUnr = OF_UNROLL;
  static constexpr int kMinBlocks = OF_MIN_BLOCKS;
};
template <> struct Tune<__nv_bfloat16> {
  static constexpr int kUnr = OF_UNROLL_BF16;
  static constexpr int kMinBlocks = OF_MIN_BLOCKS_BF16;
};

// One multi-tensor policy step.  T: param/state type; G: grad type; UNR:
// vectors per thread per tile (tile = 256 * 4 * UNR elements).  Small lists
// use UNR=1 so that even a few MB spread over more CTAs than there are SMs.
template <class Op, class T, class G, int CAP, int UNR>
__global__ void __launch_bounds__(kThreads, Tune<G>::kMinBlocks)
mt_step_kernel(const __grid_constant__ MTParams<CAP> mp, const Op op_in,
               const void* __restrict__ gscale, uint32_t flags, const StepSrc step) {
  using GV = typename GradVal<G>::type;
  Op op = op_in;
  if (step.offset != nullptr) {  // OF_FLAG_DEVICE_STEP: this replay's step index
    int64_t t = step.t_base + *step.offset;
    t = t < 1 ? 1 : (t >= step.rows ? step.rows - 1 : t);
    op.set_step(step.table[2 * t], step.table[2 * t + 1]);
  }
  constexpr int kTileU = kThreads * kVec * UNR;
  constexpr int kRoundMax = sizeof(T) == 8 ? 2 : 4;
  constexpr int kRound = UNR < kRoundMax ? UNR : kRoundMax;  // vectors in flight per thread
  const int total = mp.tile_end[mp.count - 1];
  const bool zero_grad = (flags & OF_FLAG_ZERO_GRAD) != 0;
  const bool shadow = (flags & OF_FLAG_SHADOW_BF16) != 0;
  const bool has_scale = gscale != nullptr;
  const T scale = load_scale<T>(gscale, flags);
  int ti = 0;
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    ti = find_tensor(mp, ti, tile);
    const int tfirst = ti ? mp.tile_end[ti - 1] : 0;
    const int64_t base = static_cast<int64_t>(tile - tfirst) * kTileU;
    const int64_t rem = mp.n[ti] - base;
    const int len = rem < kTileU ? static_cast<int>(rem) : kTileU;
    T* p = static_cast<T*>(mp.p[ti]) + base;
    G* g = static_cast<G*>(mp.g[ti]) + base;
    T* s0 = Op::kSlots >= 1 ? static_cast<T*>(mp.s0[ti]) + base : nullptr;
    T* s1 = Op::kSlots >= 2 ? static_cast<T*>(mp.s1[ti]) + base : nullptr;
    __nv_bfloat16* sh = shadow ? static_cast<__nv_bfloat16*>(mp.sh[ti]) + base : nullptr;
    const bool vec_ok = aligned(p, 16) && aligned(g, 4 * sizeof(G)) &&
                        (Op::kSlots < 1 || aligned(s0, 16)) && (Op::kSlots < 2 || aligned(s1, 16)) &&
                        (!shadow || aligned(sh, 8));
    int scalar_from = 0;
    if (vec_ok) {
      const int nvec = len / kVec;
#pragma unroll
      for (int r = 0; r < UNR; r += kRound) {
        T vp[kRound][4], v0[kRound][4], v1[kRound][4];
        GV vg[kRound][4];
#pragma unroll
        for (int u = 0; u < kRound; ++u) {
          const int j = threadIdx.x + (r + u) * kThreads;
          if (j < nvec) {
            ld4(p + 4 * j, vp[u]);
            ld4s(g + 4 * j, vg[u]);
            if (Op::kSlots >= 1) ld4s(s0 + 4 * j, v0[u]);
            if (Op::kSlots >= 2) ld4s(s1 + 4 * j, v1[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < kRound; ++u) {
          const int j = threadIdx.x + (r + u) * kThreads;
          if (j < nvec) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              T gk = static_cast<T>(vg[u][k]);
              if (has_scale) gk = o_mul(gk, scale);  // grad *= clip factor (optim.py:170)
              op(vp[u][k], gk, v0[u][k], v1[u][k]);
            }
            st4(p + 4 * j, vp[u]);
            if (Op::kSlots >= 1) st4s(s0 + 4 * j, v0[u]);
            if (Op::kSlots >= 2) st4s(s1 + 4 * j, v1[u]);
            if (zero_grad) st4_zero(g + 4 * j);
            if (shadow) st4_bf16(sh + 4 * j, vp[u]);
          }
        }
      }
      scalar_from = nvec * kVec;
    }
    for (int e = scalar_from + threadIdx.x; e < len; e += kThreads) {
      T pv = p[e];
      T a = Op::kSlots >= 1 ? s0[e] : T(0);
      T b = Op::kSlots >= 2 ? s1[e] : T(0);
      T gk = static_cast<T>(ld1(g + e));
      if (has_scale) gk = o_mul(gk, scale);
      op(pv, gk, a, b);
      p[e] = pv;
      if (Op::kSlots >= 1) s0[e] = a;
      if (Op::kSlots >= 2) s1[e] = b;
      if (zero_grad) st1_zero(g + e);
      if (shadow) sh[e] = __float2bfloat16_rn(static_cast<float>(pv));
    }
  }
}

// Sum of squares, per-CTA f64 partials (deterministic order within a CTA).
template <class G, int CAP>
__global__ void __launch_bounds__(kThreads)
mt_sqnorm_kernel(const __grid_constant__ MTParams<CAP> mp, double* __restrict__ partials) {
  const int total = mp.tile_end[mp.count - 1];
  double acc = 0.0;
  int ti = 0;
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    ti = find_tensor(mp, ti, tile);
    const int tfirst = ti ? mp.tile_end[ti - 1] : 0;
    const int64_t base = static_cast<int64_t>(tile - tfirst) * kTile;
    const int64_t rem = mp.n[ti] - base;
    const int len = rem < kTile ? static_cast<int>(rem) : kTile;
    const G* g = static_cast<const G*>(mp.g[ti]) + base;
    for (int e = threadIdx.x; e < len; e += kThreads) {
      const double x = static_cast<double>(ld1(g + e));
      acc = __dadd_rn(acc, __dmul_rn(x, x));
    }
  }
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
  }
}

__global__ void __launch_bounds__(kThreads)
sqnorm_finalize_kernel(const double* __restrict__ partials, int n, double* out, int accumulate) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += kThreads) acc = __dadd_rn(acc, partials[i]);
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s = __dadd_rn(s, red[w]);
    *out = accumulate ? __dadd_rn(*out, s) : s;
  }
}

__global__ void clip_coef_kernel(const double* sq, double max_norm, float* coef, double* factor_out) {
  const double norm = __dsqrt_rn(*sq);                       // optim.py:165
  const double factor = norm <= max_norm ? 1.0 : __ddiv_rn(max_norm, norm);  // optim.py:166-168
  *coef = __double2float_rn(factor);                         // numpy casts the factor to f32
  if (factor_out) *factor_out = factor;
}

__global__ void step_advance_kernel(int64_t* offset, int64_t delta) { *offset += delta; }

// Multi-tensor byte copy (dst[i] <- src[i]): one launch for a whole gradient
// set.  MTParams carries dst in p, src in g and the byte count in n; tiles of
// kCopyTile bytes, 16-byte vectors where both sides allow, bytes otherwise.
constexpr int kCopyTile = 16384;
template <int CAP>
__global__ void __launch_bounds__(kThreads)
mt_copy_kernel(const __grid_constant__ MTParams<CAP> mp) {
  const int total = mp.tile_end[mp.count - 1];
  int ti = 0;
  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    ti = find_tensor(mp, ti, tile);
    const int tfirst = ti ? mp.tile_end[ti - 1] : 0;
    const int64_t base = static_cast<int64_t>(tile - tfirst) * kCopyTile;
    const int64_t rem = mp.n[ti] - base;
    const int len = rem < kCopyTile ? static_cast<int>(rem) : kCopyTile;
    char* d = static_cast<char*>(mp.p[ti]) + base;
    const char* s = static_cast<const char*>(mp.g[ti]) + base;
    int from = 0;
    if (aligned(d, 16) && aligned(s, 16)) {
      const int nv = len / 16;
      for (int j = threadIdx.x; j < nv; j += kThreads)
        reinterpret_cast<uint4*>(d)[j] = reinterpret_cast<const uint4*>(s)[j];
      from = nv * 16;
    }
    for (int j = from + threadIdx.x; j < len; j += kThreads) d[j] = s[j];
  }
}

// Fixed-order matmul of the synthetic parity graphs (tensor.py's
// accumulation: out = 0; for k ascending: out = out + a[:, k] * b[k, :], every
// product and sum separately rounded): one thread per output element.
template <class T>
__global__ void __launch_bounds__(kThreads)
exact_matmul_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                    int64_t M, int64_t K, int64_t N) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= N || i >= M) return;
  T acc = T(0);
  for (int64_t k = 0; k < K; ++k) acc = o_add(acc, o_mul(a[i * K + k], b[k * N + j]));
  out[i * N + j] = acc;
}

// ---------------------------------------------------------------------------
// Host side: validation, packing, dispatch.
// ---------------------------------------------------------------------------
int slots_of(int kind) {
  switch (kind) {
    case OF_SGD: return 0;
    case OF_SGD_MOMENTUM: case OF_ADAGRAD: case OF_RMSPROP: return 1;
    case OF_ADADELTA: case OF_ADAM: case OF_ADAMW: return 2;
    default: return -1;
  }
}

int validate_list(const of_tensor_list* l, int slots, bool need_shadow, bool grads_only) {
  if (!l) return fail(OF_ERR_INVALID, "tensor list is NULL");
  if (l->n < 0) return fail(OF_ERR_INVALID, "tensor list has n=%d < 0", l->n);
  if (l->n == 0) return OF_OK;
  if (l->param_dtype != OF_F32 && l->param_dtype != OF_F64)
    return fail(OF_ERR_UNSUPPORTED, "param dtype %d not supported (f32, f64)", l->param_dtype);
  if (!(l->grad_dtype == l->param_dtype || (l->grad_dtype == OF_BF16 && l->param_dtype == OF_F32)))
    return fail(OF_ERR_UNSUPPORTED, "grad dtype %d with param dtype %d not supported",
                l->grad_dtype, l->param_dtype);
  if (!l->numel || !l->grad || (!grads_only && !l->param))
    return fail(OF_ERR_INVALID, "tensor list is missing the param/grad/numel arrays");
  if (!grads_only) {
    if (slots >= 1 && !l->state0) return fail(OF_ERR_INVALID, "kind needs state0 (history slot 0)");
    if (slots >= 2 && !l->state1) return fail(OF_ERR_INVALID, "kind needs state1 (history slot 1)");
    if (need_shadow && !l->shadow) return fail(OF_ERR_INVALID, "OF_FLAG_SHADOW_BF16 needs shadow pointers");
  }
  for (int i = 0; i < l->n; ++i) {
    if (l->numel[i] < 0) return fail(OF_ERR_INVALID, "tensor %d has numel %lld < 0", i, (long long)l->numel[i]);
    if (l->numel[i] == 0) continue;
    if (!l->grad[i]) return fail(OF_ERR_INVALID, "tensor %d has a NULL grad", i);
    if (grads_only) continue;
    if (!l->param[i]) return fail(OF_ERR_INVALID, "tensor %d has a NULL param", i);
    if (slots >= 1 && !l->state0[i]) return fail(OF_ERR_INVALID, "tensor %d has a NULL state0", i);
    if (slots >= 2 && !l->state1[i]) return fail(OF_ERR_INVALID, "tensor %d has a NULL state1", i);
    if (need_shadow && !l->shadow[i]) return fail(OF_ERR_INVALID, "tensor %d has a NULL shadow", i);
  }
  return OF_OK;
}

// Packs tensors [first, first+count) into a parameter block; returns total tiles.
template <int CAP>
int64_t pack(const of_tensor_list* l, int first, int count, MTParams<CAP>& mp, int tile = kTile) {
  int64_t tiles = 0;
  mp.count = count;
  for (int i = 0; i < count; ++i) {
    const int k = first + i;
    mp.p[i] = l->param ? l->param[k] : nullptr;
    mp.g[i] = l->grad[k];
    mp.s0[i] = l->state0 ? l->state0[k] : nullptr;
    mp.s1[i] = l->state1 ? l->state1[k] : nullptr;
    mp.sh[i] = l->shadow ? l->shadow[k] : nullptr;
    mp.n[i] = l->numel[k];
    tiles += (l->numel[k] + tile - 1) / tile;
    mp.tile_end[i] = static_cast<int32_t>(tiles);
  }
  return tiles;
}

template <class Op, class T, class G, int CAP>
int launch_step_chunk(const of_tensor_list* l, int first, int count, const Op& op,
                      const void* gscale, uint32_t flags, const StepSrc& step, int max_ctas,
                      cudaStream_t s) {
  constexpr int U = Tune<G>::kUnr;
  MTParams<CAP> mp;
  int64_t tiles = pack<CAP>(l, first, count, mp, kThreads * kVec * U);
  if (tiles == 0) return OF_OK;
  int64_t cap = static_cast<int64_t>(sm_count()) * kCtasPerSm;
  if (max_ctas > 0 && max_ctas < cap) cap = max_ctas;
  if (tiles < 2 * static_cast<int64_t>(sm_count()) && max_ctas == 0) {
    // small launch: 1024-element tiles, 4x the CTAs for the same bytes
    tiles = pack<CAP>(l, first, count, mp, kThreads * kVec);
    const int grid = static_cast<int>(tiles < cap ? tiles : cap);
    mt_step_kernel<Op, T, G, CAP, 1><<<grid, kThreads, 0, s>>>(mp, op, gscale, flags, step);
    return check_launch("mt_step_kernel");
  }
  if (tiles > INT32_MAX) return fail(OF_ERR_INVALID, "tensor list too large for one launch");
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  mt_step_kernel<Op, T, G, CAP, U><<<grid, kThreads, 0, s>>>(mp, op, gscale, flags, step);
  return check_launch("mt_step_kernel");
}

template <class Op, class T, class G>
int launch_step(const of_tensor_list* l, const Op& op, const void* gscale, uint32_t flags,
                const StepSrc& step, int max_ctas, cudaStream_t s) {
  int first = 0;
  while (first < l->n) {
    const int left = l->n - first;
    int st;
    if (left <= 4) {
      st = launch_step_chunk<Op, T, G, 4>(l, first, left, op, gscale, flags, step, max_ctas, s);
      first += left;
    } else if (left <= 16) {
      st = launch_step_chunk<Op, T, G, 16>(l, first, left, op, gscale, flags, step, max_ctas, s);
      first += left;
    } else if (left <= 64) {
      st = launch_step_chunk<Op, T, G, 64>(l, first, left, op, gscale, flags, step, max_ctas, s);
      first += left;
    } else {
      // up to 256 tensors in one launch: a 13 KB parameter block (CUDA >= 12.1
      // accepts up to 32 KB), so a whole CNN's parameter set is one kernel
      const int c = left < kCapMax ? left : kCapMax;
      st = launch_step_chunk<Op, T, G, kCapMax>(l, first, c, op, gscale, flags, step, max_ctas, s);
      first += c;
    }
    if (st != OF_OK) return st;
  }
  return OF_OK;
}

template <class T, class G>
int dispatch_kind(const of_tensor_list* l, const of_hparams* hp, const void* gscale,
                  uint32_t flags, cudaStream_t s) {
  const StepSrc step = step_source(hp, flags);
  flags &= ~OF_FLAG_DEVICE_STEP;
  return with_op<T>(hp, [&](auto op) {
    return launch_step<decltype(op), T, G>(l, op, gscale, flags, step, hp->max_ctas, s);
  });
}

// ---------------------------------------------------------------------------
// Data-parallel fused step over peer memory (NVLink / NVSwitch).
//
// Rank r owns the shard [begin, begin + len) of a flat bucket.  One kernel
// replaces reduce-scatter -> update -> all-gather: each thread loads its
// gradient vector from every peer's buffer (peer-mapped pointers, fixed rank
// order, so the sum is deterministic), applies the policy step to the local
// parameter (or fp32 master) and history, stores the new parameter (or its
// bf16 shadow) into every peer's parameter buffer and zeroes the gradient
// vector it read in every peer.  Each gradient element is read and zeroed by
// exactly one rank (its shard owner), so there is no write-write race; the
// caller brackets the launch with a cross-rank barrier (gradients complete
// before, writes visible after).
// ---------------------------------------------------------------------------
struct PeerParams {
  void* grad[OF_MAX_PEERS];
  void* param[OF_MAX_PEERS];
  void* master;            // fp32 master shard (mixed) or nullptr
  void* s0;                // history shards
  void* s1;
  int64_t begin, len;      // shard, in elements of the flat buffers (multiples of 4)
  int32_t world, rank;
};

template <class Op, class T, class G, bool kMixed>
__global__ void __launch_bounds__(kThreads)
peer_step_kernel(const __grid_constant__ PeerParams pp, const Op op_in,
                 const float* __restrict__ gscale, const StepSrc step) {
  using GV = typename GradVal<G>::type;
  Op op = op_in;
  if (step.offset != nullptr) {
    int64_t t = step.t_base + *step.offset;
    t = t < 1 ? 1 : (t >= step.rows ? step.rows - 1 : t);
    op.set_step(step.table[2 * t], step.table[2 * t + 1]);
  }
  const bool has_scale = gscale != nullptr;
  const T scale = has_scale ? T(*gscale) : T(1);
  const int64_t nvec = pp.len / kVec;
  const int W = pp.world;
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; v < nvec;
       v += static_cast<int64_t>(gridDim.x) * kThreads) {
    const int64_t e = pp.begin + kVec * v;   // flat-buffer element
    const int64_t o = kVec * v;              // shard element
    GV acc[4], tmp[4];
    ld4(static_cast<const G*>(pp.grad[0]) + e, acc);
    for (int w = 1; w < W; ++w) {
      ld4(static_cast<const G*>(pp.grad[w]) + e, tmp);
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = o_add(acc[k], tmp[k]);
    }
    T p[4], a[4], b[4];
    if (kMixed) ld4(static_cast<const T*>(pp.master) + o, p);
    else ld4(static_cast<const T*>(pp.param[pp.rank]) + e, p);
    if (Op::kSlots >= 1) ld4(static_cast<const T*>(pp.s0) + o, a);
    if (Op::kSlots >= 2) ld4(static_cast<const T*>(pp.s1) + o, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      T gk = static_cast<T>(acc[k]);
      if (has_scale) gk = o_mul(gk, scale);   // 1/W (and the clip factor)
      op(p[k], gk, a[k], b[k]);
    }
    if (Op::kSlots >= 1) st4(static_cast<T*>(pp.s0) + o, a);
    if (Op::kSlots >= 2) st4(static_cast<T*>(pp.s1) + o, b);
    if (kMixed) st4(static_cast<T*>(pp.master) + o, p);
    for (int w = 0; w < W; ++w) {
      if (kMixed) st4_bf16(static_cast<__nv_bfloat16*>(pp.param[w]) + e, p);
      else st4(static_cast<T*>(pp.param[w]) + e, p);
      st4_zero(static_cast<G*>(pp.grad[w]) + e);
    }
  }
}

// Sum of squares of the peer-summed gradient shard (of_dp_sqnorm_peer): the
// same rank-order sum as peer_step_kernel, squared and accumulated in f64;
// per-CTA partials in a fixed order, then sqnorm_finalize_kernel.
template <class G>
__global__ void __launch_bounds__(kThreads)
peer_sqnorm_kernel(const __grid_constant__ PeerParams pp, double* __restrict__ partials) {
  using GV = typename GradVal<G>::type;
  const int64_t nvec = pp.len / kVec;
  const int W = pp.world;
  double acc2 = 0.0;
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; v < nvec;
       v += static_cast<int64_t>(gridDim.x) * kThreads) {
    const int64_t e = pp.begin + kVec * v;
    GV acc[4], tmp[4];
    ld4(static_cast<const G*>(pp.grad[0]) + e, acc);
    for (int w = 1; w < W; ++w) {
      ld4(static_cast<const G*>(pp.grad[w]) + e, tmp);
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = o_add(acc[k], tmp[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double x = static_cast<double>(acc[k]);
      acc2 = __dadd_rn(acc2, __dmul_rn(x, x));
    }
  }
  __shared__ double red[kThreads / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc2 = __dadd_rn(acc2, __shfl_down_sync(0xffffffffu, acc2, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc2;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < kThreads / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
    if (threadIdx.x == 0) partials[blockIdx.x] = v;
  }
}

template <class T, class G, bool kMixed>
int dispatch_peer(const PeerParams& pp, const of_hparams* hp, const float* gscale, uint32_t flags,
                  cudaStream_t s) {
  const StepSrc step = step_source(hp, flags);
  const int64_t nvec = pp.len / kVec;
  if (nvec == 0) return OF_OK;
  int64_t grid = (nvec + kThreads - 1) / kThreads;
  int64_t cap = static_cast<int64_t>(sm_count()) * kCtasPerSm;
  if (hp->max_ctas > 0 && hp->max_ctas < cap) cap = hp->max_ctas;
  if (grid > cap) grid = cap;
  return with_op<T>(hp, [&](auto op) {
    peer_step_kernel<decltype(op), T, G, kMixed><<<static_cast<int>(grid), kThreads, 0, s>>>(
        pp, op, gscale, step);
    return check_launch("peer_step_kernel");
  });
}

// ---------------------------------------------------------------------------
// The peer step over NVLS multicast (of_dp_step_multicast): one in-switch
// reduced load of the shard's gradient, one multicast store of the new
// parameters and of the zeroed gradient, whatever the world size.
// ---------------------------------------------------------------------------
struct McParams {
  float* mc_grad;
  float* mc_param;
  const float* local_param;
  float* s0;
  float* s1;
  int64_t begin, len;
};

__device__ __forceinline__ float4 mc_ld_reduce_add4(const float* p) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p) : "memory");
  return r;
}

__device__ __forceinline__ void mc_st4(float* p, float a, float b, float c, float d) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
               :: "l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

template <class Op>
__global__ void __launch_bounds__(kThreads)
mc_step_kernel(const __grid_constant__ McParams mp, const Op op_in,
               const float* __restrict__ gscale, const StepSrc step) {
  Op op = op_in;
  if (step.offset != nullptr) {
    int64_t t = step.t_base + *step.offset;
    t = t < 1 ? 1 : (t >= step.rows ? step.rows - 1 : t);
    op.set_step(step.table[2 * t], step.table[2 * t + 1]);
  }
  const bool has_scale = gscale != nullptr;
  const float scale = has_scale ? *gscale : 1.f;
  const int64_t nvec = mp.len / kVec;
  for (int64_t v = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; v < nvec;
       v += static_cast<int64_t>(gridDim.x) * kThreads) {
    const int64_t e = mp.begin + kVec * v;
    const int64_t o = kVec * v;
    const float4 g4 = mc_ld_reduce_add4(mp.mc_grad + e);
    const float g[4] = {g4.x, g4.y, g4.z, g4.w};
    float p[4], a[4], b[4];
    ld4(mp.local_param + e, p);
    if (Op::kSlots >= 1) ld4(mp.s0 + o, a);
    if (Op::kSlots >= 2) ld4(mp.s1 + o, b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float gk = g[k];
      if (has_scale) gk = o_mul(gk, scale);
      op(p[k], gk, a[k], b[k]);
    }
    if (Op::kSlots >= 1) st4(mp.s0 + o, a);
    if (Op::kSlots >= 2) st4(mp.s1 + o, b);
    mc_st4(mp.mc_param + e, p[0], p[1], p[2], p[3]);
    mc_st4(mp.mc_grad + e, 0.f, 0.f, 0.f, 0.f);
  }
}

template <class G, int CAP>
int launch_sqnorm_chunk(const of_tensor_list* l, int first, int count, double* ws, int64_t ws_len,
                        double* out, int accumulate, cudaStream_t s) {
  MTParams<CAP> mp;
  const int64_t tiles = pack<CAP>(l, first, count, mp);
  if (tiles == 0) {
    if (!accumulate) {
      if (cudaMemsetAsync(out, 0, sizeof(double), s) != cudaSuccess)
        return fail(OF_ERR_CUDA, "cudaMemsetAsync failed");
    }
    return OF_OK;
  }
  int64_t cap = static_cast<int64_t>(sm_count()) * 4;
  if (cap > ws_len) cap = ws_len;
  const int grid = static_cast<int>(tiles < cap ? tiles : cap);
  mt_sqnorm_kernel<G, CAP><<<grid, kThreads, 0, s>>>(mp, ws);
  int st = check_launch("mt_sqnorm_kernel");
  if (st != OF_OK) return st;
  sqnorm_finalize_kernel<<<1, kThreads, 0, s>>>(ws, grid, out, accumulate);
  return check_launch("sqnorm_finalize_kernel");
}

template <class G>
int launch_sqnorm(const of_tensor_list* l, double* ws, int64_t ws_len, double* out, int accumulate,
                  cudaStream_t s) {
  int first = 0;
  do {
    const int left = l->n - first;
    const int c = left < kCapMax ? left : kCapMax;
    const int st = launch_sqnorm_chunk<G, kCapMax>(l, first, c, ws, ws_len, out, accumulate, s);
    if (st != OF_OK) return st;
    accumulate = 1;
    first += c;
  } while (first < l->n);
  return OF_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

int of_abi_version(void) { return OF_ABI_VERSION; }

const char* of_status_string(int status) {
  switch (status) {
    case OF_OK: return "ok";
    case OF_ERR_INVALID: return "invalid argument";
    case OF_ERR_UNSUPPORTED: return "unsupported combination";
    case OF_ERR_CUDA: return "CUDA launch error";
    default: return "unknown status";
  }
}

const char* of_last_error(void) { return g_err; }

uint64_t of_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int of_policy_step_mt(const of_tensor_list* list, const of_hparams* hp,
                      const void* grad_scale_dev, uint32_t flags, void* stream) {
  g_err[0] = '\0';
  if (!hp) return fail(OF_ERR_INVALID, "hparams is NULL");
  const int slots = slots_of(hp->kind);
  if (slots < 0) return fail(OF_ERR_INVALID, "unknown optimizer kind %d", hp->kind);
  if (flags & ~(OF_FLAG_ZERO_GRAD | OF_FLAG_SHADOW_BF16 | OF_FLAG_DEVICE_STEP | OF_FLAG_SCALE_F64))
    return fail(OF_ERR_INVALID, "unknown flags 0x%x", flags);
  if ((flags & OF_FLAG_SCALE_F64) && !grad_scale_dev)
    return fail(OF_ERR_INVALID, "OF_FLAG_SCALE_F64 without a grad_scale_dev");
  if (!(hp->eta > 0.0)) return fail(OF_ERR_INVALID, "step size must be > 0, got %g", hp->eta);
  if (flags & OF_FLAG_DEVICE_STEP) {
    if (!hp->step_offset_dev || !hp->step_table_dev)
      return fail(OF_ERR_INVALID, "OF_FLAG_DEVICE_STEP needs step_offset_dev and step_table_dev");
    if (hp->step_table_rows < 2)
      return fail(OF_ERR_INVALID, "step table needs >= 2 rows, got %lld", (long long)hp->step_table_rows);
  } else if ((hp->kind == OF_ADAM || hp->kind == OF_ADAMW) &&
             (hp->bias_correction1 == 0.0 || hp->bias_correction2 == 0.0)) {
    return fail(OF_ERR_INVALID, "adam bias corrections must be non-zero (step index t >= 1)");
  }
  int st = validate_list(list, slots, (flags & OF_FLAG_SHADOW_BF16) != 0, false);
  if (st != OF_OK || list->n == 0) return st;
  if (hp->max_ctas < 0) return fail(OF_ERR_INVALID, "max_ctas must be >= 0, got %d", hp->max_ctas);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (list->param_dtype == OF_F64) return dispatch_kind<double, double>(list, hp, grad_scale_dev, flags, s);
  if (list->grad_dtype == OF_BF16) return dispatch_kind<float, __nv_bfloat16>(list, hp, grad_scale_dev, flags, s);
  return dispatch_kind<float, float>(list, hp, grad_scale_dev, flags, s);
}

int of_sgdm_mt(const of_tensor_list* list, double eta, double alpha, double weight_decay,
               const void* grad_scale_dev, uint32_t flags, void* stream) {
  of_hparams hp;
  memset(&hp, 0, sizeof(hp));
  hp.kind = OF_SGD_MOMENTUM;
  hp.eta = eta;
  hp.alpha = alpha;
  hp.weight_decay = weight_decay;
  return of_policy_step_mt(list, &hp, grad_scale_dev, flags, stream);
}

int of_adam_mt(const of_tensor_list* list, double eta, double beta1, double beta2, double epsilon,
               double weight_decay, double bias_correction1, double bias_correction2,
               int decoupled_weight_decay, const void* grad_scale_dev, uint32_t flags,
               void* stream) {
  of_hparams hp;
  memset(&hp, 0, sizeof(hp));
  hp.kind = decoupled_weight_decay ? OF_ADAMW : OF_ADAM;
  hp.eta = eta;
  hp.beta1 = beta1;
  hp.beta2 = beta2;
  hp.epsilon = epsilon;
  hp.weight_decay = weight_decay;
  hp.bias_correction1 = bias_correction1;
  hp.bias_correction2 = bias_correction2;
  return of_policy_step_mt(list, &hp, grad_scale_dev, flags, stream);
}

int of_step_advance(int64_t* step_offset_dev, int64_t delta, void* stream) {
  g_err[0] = '\0';
  if (!step_offset_dev) return fail(OF_ERR_INVALID, "step_offset_dev is NULL");
  step_advance_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(step_offset_dev, delta);
  return check_launch("step_advance_kernel");
}

int of_exact_matmul(const void* a, const void* b, void* out, int64_t M, int64_t K, int64_t N,
                    int dtype, void* stream) {
  g_err[0] = '\0';
  if (!a || !b || !out) return fail(OF_ERR_INVALID, "exact_matmul: NULL operand");
  if (M < 0 || K < 0 || N < 0 || M > 65535)
    return fail(OF_ERR_INVALID, "exact_matmul: bad shape %lld x %lld x %lld", (long long)M,
                (long long)K, (long long)N);
  if (M == 0 || N == 0) return OF_OK;
  const dim3 grid(static_cast<unsigned>((N + kThreads - 1) / kThreads), static_cast<unsigned>(M));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == OF_F32)
    exact_matmul_kernel<float><<<grid, kThreads, 0, s>>>(static_cast<const float*>(a),
        static_cast<const float*>(b), static_cast<float*>(out), M, K, N);
  else if (dtype == OF_F64)
    exact_matmul_kernel<double><<<grid, kThreads, 0, s>>>(static_cast<const double*>(a),
        static_cast<const double*>(b), static_cast<double*>(out), M, K, N);
  else
    return fail(OF_ERR_UNSUPPORTED, "exact_matmul: dtype %d", dtype);
  return check_launch("exact_matmul_kernel");
}

int of_copy_mt(void* const* dst, const void* const* src, const int64_t* nbytes, int n, void* stream) {
  g_err[0] = '\0';
  if (n < 0 || (n > 0 && (!dst || !src || !nbytes))) return fail(OF_ERR_INVALID, "copy_mt: bad list");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int first = 0; first < n; first += kCapMax) {
    const int count = n - first < kCapMax ? n - first : kCapMax;
    MTParams<kCapMax> mp;
    memset(&mp, 0, sizeof(mp));
    int64_t tiles = 0;
    mp.count = count;
    for (int i = 0; i < count; ++i) {
      const int k = first + i;
      if (nbytes[k] < 0) return fail(OF_ERR_INVALID, "copy_mt: tensor %d has %lld bytes", k,
                                     (long long)nbytes[k]);
      if (nbytes[k] > 0 && (!dst[k] || !src[k])) return fail(OF_ERR_INVALID, "copy_mt: NULL tensor %d", k);
      mp.p[i] = dst[k];
      mp.g[i] = const_cast<void*>(src[k]);
      mp.n[i] = nbytes[k];
      tiles += (nbytes[k] + kCopyTile - 1) / kCopyTile;
      mp.tile_end[i] = static_cast<int32_t>(tiles);
    }
    if (tiles == 0) continue;
    const int64_t cap = static_cast<int64_t>(sm_count()) * kCtasPerSm;
    const int grid = static_cast<int>(tiles < cap ? tiles : cap);
    mt_copy_kernel<kCapMax><<<grid, kThreads, 0, s>>>(mp);
    const int st = check_launch("mt_copy_kernel");
    if (st != OF_OK) return st;
  }
  return OF_OK;
}

int64_t of_sqnorm_workspace_len(void) { return kSqnormWorkspace; }

int of_sqnorm_mt(const of_tensor_list* list, double* workspace_dev, int64_t workspace_len,
                 double* out_dev, int accumulate, void* stream) {
  g_err[0] = '\0';
  if (!workspace_dev || workspace_len < 1) return fail(OF_ERR_INVALID, "sqnorm needs a workspace");
  if (!out_dev) return fail(OF_ERR_INVALID, "sqnorm output pointer is NULL");
  int st = validate_list(list, 0, false, true);
  if (st != OF_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (list->n == 0) {
    if (!accumulate && cudaMemsetAsync(out_dev, 0, sizeof(double), s) != cudaSuccess)
      return fail(OF_ERR_CUDA, "cudaMemsetAsync failed");
    return OF_OK;
  }
  switch (list->grad_dtype) {
    case OF_F32: return launch_sqnorm<float>(list, workspace_dev, workspace_len, out_dev, accumulate, s);
    case OF_F64: return launch_sqnorm<double>(list, workspace_dev, workspace_len, out_dev, accumulate, s);
    case OF_BF16: return launch_sqnorm<__nv_bfloat16>(list, workspace_dev, workspace_len, out_dev, accumulate, s);
    default: return fail(OF_ERR_UNSUPPORTED, "grad dtype %d", list->grad_dtype);
  }
}

int of_clip_coef(const double* sqnorm_dev, double max_norm, float* coef_dev, double* factor_dev,
                 void* stream) {
  g_err[0] = '\0';
  if (!sqnorm_dev || !coef_dev) return fail(OF_ERR_INVALID, "clip_coef needs sqnorm and coef pointers");
  if (!(max_norm >= 0.0)) return fail(OF_ERR_INVALID, "max_norm must be >= 0, got %g", max_norm);
  clip_coef_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(sqnorm_dev, max_norm, coef_dev, factor_dev);
  return check_launch("clip_coef_kernel");
}

int of_dp_step_peer(const of_peer_bucket* b, const of_hparams* hp, const float* grad_scale_dev,
                    uint32_t flags, void* stream) {
  g_err[0] = '\0';
  if (!b || !hp) return fail(OF_ERR_INVALID, "bucket or hparams is NULL");
  const int slots = slots_of(hp->kind);
  if (slots < 0) return fail(OF_ERR_INVALID, "unknown optimizer kind %d", hp->kind);
  if (flags & ~(OF_FLAG_DEVICE_STEP))
    return fail(OF_ERR_INVALID, "flags 0x%x not supported by the peer step (gradients are always "
                "zeroed; bf16 parameters follow from param_dtype)", flags);
  if (!(hp->eta > 0.0)) return fail(OF_ERR_INVALID, "step size must be > 0, got %g", hp->eta);
  if (flags & OF_FLAG_DEVICE_STEP) {
    if (!hp->step_offset_dev || !hp->step_table_dev || hp->step_table_rows < 2)
      return fail(OF_ERR_INVALID, "OF_FLAG_DEVICE_STEP needs step_offset_dev and a step table");
  } else if ((hp->kind == OF_ADAM || hp->kind == OF_ADAMW) &&
             (hp->bias_correction1 == 0.0 || hp->bias_correction2 == 0.0)) {
    return fail(OF_ERR_INVALID, "adam bias corrections must be non-zero (step index t >= 1)");
  }
  if (b->world < 1 || b->world > OF_MAX_PEERS)
    return fail(OF_ERR_INVALID, "world %d outside [1, %d]", b->world, OF_MAX_PEERS);
  if (b->rank < 0 || b->rank >= b->world)
    return fail(OF_ERR_INVALID, "rank %d outside [0, %d)", b->rank, b->world);
  if (b->shard_begin < 0 || b->shard_len < 0 || (b->shard_begin % 4) || (b->shard_len % 4))
    return fail(OF_ERR_INVALID, "shard [%lld, +%lld) must be non-negative multiples of 4",
                (long long)b->shard_begin, (long long)b->shard_len);
  if (!b->peer_grad || !b->peer_param) return fail(OF_ERR_INVALID, "peer pointer arrays are NULL");
  PeerParams pp;
  memset(&pp, 0, sizeof(pp));
  for (int w = 0; w < b->world; ++w) {
    if (!b->peer_grad[w] || !b->peer_param[w])
      return fail(OF_ERR_INVALID, "peer %d has a NULL grad or param buffer", w);
    pp.grad[w] = b->peer_grad[w];
    pp.param[w] = b->peer_param[w];
  }
  const bool mixed = b->param_dtype == OF_BF16;
  if (mixed && (b->grad_dtype != OF_BF16 || !b->master))
    return fail(OF_ERR_INVALID, "bf16 parameters need bf16 gradients and an fp32 master shard");
  if (!mixed && b->grad_dtype != b->param_dtype)
    return fail(OF_ERR_UNSUPPORTED, "grad dtype %d with param dtype %d", b->grad_dtype, b->param_dtype);
  if (slots >= 1 && !b->state0) return fail(OF_ERR_INVALID, "kind needs state0");
  if (slots >= 2 && !b->state1) return fail(OF_ERR_INVALID, "kind needs state1");
  pp.master = b->master;
  pp.s0 = b->state0;
  pp.s1 = b->state1;
  pp.begin = b->shard_begin;
  pp.len = b->shard_len;
  pp.world = b->world;
  pp.rank = b->rank;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mixed) return dispatch_peer<float, __nv_bfloat16, true>(pp, hp, grad_scale_dev, flags, s);
  if (b->param_dtype == OF_F32) return dispatch_peer<float, float, false>(pp, hp, grad_scale_dev, flags, s);
  if (b->param_dtype == OF_F64) return dispatch_peer<double, double, false>(pp, hp, grad_scale_dev, flags, s);
  return fail(OF_ERR_UNSUPPORTED, "param dtype %d", b->param_dtype);
}

int of_dp_sqnorm_peer(const of_peer_bucket* b, double* workspace_dev, int64_t workspace_len,
                      double* out_dev, int accumulate, void* stream) {
  g_err[0] = '\0';
  if (!b) return fail(OF_ERR_INVALID, "bucket is NULL");
  if (!workspace_dev || workspace_len < 1) return fail(OF_ERR_INVALID, "sqnorm needs a workspace");
  if (!out_dev) return fail(OF_ERR_INVALID, "sqnorm output pointer is NULL");
  if (b->world < 1 || b->world > OF_MAX_PEERS)
    return fail(OF_ERR_INVALID, "world %d outside [1, %d]", b->world, OF_MAX_PEERS);
  if (b->rank < 0 || b->rank >= b->world)
    return fail(OF_ERR_INVALID, "rank %d outside [0, %d)", b->rank, b->world);
  if (b->shard_begin < 0 || b->shard_len < 0 || (b->shard_begin % 4) || (b->shard_len % 4))
    return fail(OF_ERR_INVALID, "shard [%lld, +%lld) must be non-negative multiples of 4",
                (long long)b->shard_begin, (long long)b->shard_len);
  if (!b->peer_grad) return fail(OF_ERR_INVALID, "peer gradient pointer array is NULL");
  PeerParams pp;
  memset(&pp, 0, sizeof(pp));
  for (int w = 0; w < b->world; ++w) {
    if (!b->peer_grad[w]) return fail(OF_ERR_INVALID, "peer %d has a NULL grad buffer", w);
    pp.grad[w] = b->peer_grad[w];
  }
  pp.begin = b->shard_begin;
  pp.len = b->shard_len;
  pp.world = b->world;
  pp.rank = b->rank;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t nvec = pp.len / kVec;
  if (nvec == 0) {
    if (!accumulate && cudaMemsetAsync(out_dev, 0, sizeof(double), s) != cudaSuccess)
      return fail(OF_ERR_CUDA, "cudaMemsetAsync failed");
    return OF_OK;
  }
  int64_t grid = (nvec + kThreads - 1) / kThreads;
  int64_t cap = static_cast<int64_t>(sm_count()) * 4;
  if (cap > workspace_len) cap = workspace_len;
  if (grid > cap) grid = cap;
  switch (b->grad_dtype) {
    case OF_F32: peer_sqnorm_kernel<float><<<static_cast<int>(grid), kThreads, 0, s>>>(pp, workspace_dev); break;
    case OF_F64: peer_sqnorm_kernel<double><<<static_cast<int>(grid), kThreads, 0, s>>>(pp, workspace_dev); break;
    case OF_BF16: peer_sqnorm_kernel<__nv_bfloat16><<<static_cast<int>(grid), kThreads, 0, s>>>(pp, workspace_dev); break;
    default: return fail(OF_ERR_UNSUPPORTED, "grad dtype %d", b->grad_dtype);
  }
  const int st = check_launch("peer_sqnorm_kernel");
  if (st != OF_OK) return st;
  sqnorm_finalize_kernel<<<1, kThreads, 0, s>>>(workspace_dev, static_cast<int>(grid), out_dev, accumulate);
  return check_launch("sqnorm_finalize_kernel");
}

int of_dp_step_multicast(const of_mc_bucket* b, const of_hparams* hp, const float* grad_scale_dev,
                         uint32_t flags, void* stream) {
  g_err[0] = '\0';
  if (!b || !hp) return fail(OF_ERR_INVALID, "bucket or hparams is NULL");
  const int slots = slots_of(hp->kind);
  if (slots < 0) return fail(OF_ERR_INVALID, "unknown optimizer kind %d", hp->kind);
  if (flags & ~(OF_FLAG_DEVICE_STEP))
    return fail(OF_ERR_INVALID, "flags 0x%x not supported by the multicast step", flags);
  if (!(hp->eta > 0.0)) return fail(OF_ERR_INVALID, "step size must be > 0, got %g", hp->eta);
  if (flags & OF_FLAG_DEVICE_STEP) {
    if (!hp->step_offset_dev || !hp->step_table_dev || hp->step_table_rows < 2)
      return fail(OF_ERR_INVALID, "OF_FLAG_DEVICE_STEP needs step_offset_dev and a step table");
  } else if ((hp->kind == OF_ADAM || hp->kind == OF_ADAMW) &&
             (hp->bias_correction1 == 0.0 || hp->bias_correction2 == 0.0)) {
    return fail(OF_ERR_INVALID, "adam bias corrections must be non-zero (step index t >= 1)");
  }
  if (b->world < 1 || b->world > OF_MAX_PEERS)
    return fail(OF_ERR_INVALID, "world %d outside [1, %d]", b->world, OF_MAX_PEERS);
  if (b->rank < 0 || b->rank >= b->world)
    return fail(OF_ERR_INVALID, "rank %d outside [0, %d)", b->rank, b->world);
  if (b->shard_begin < 0 || b->shard_len < 0 || (b->shard_begin % 4) || (b->shard_len % 4))
    return fail(OF_ERR_INVALID, "shard [%lld, +%lld) must be non-negative multiples of 4",
                (long long)b->shard_begin, (long long)b->shard_len);
  if (b->param_dtype != OF_F32 || b->grad_dtype != OF_F32)
    return fail(OF_ERR_UNSUPPORTED, "multicast step: fp32 parameters and gradients only "
                "(param dtype %d, grad dtype %d)", b->param_dtype, b->grad_dtype);
  if (!b->mc_grad || !b->mc_param || !b->local_param)
    return fail(OF_ERR_INVALID, "multicast or local buffer is NULL");
  if ((reinterpret_cast<uintptr_t>(b->mc_grad) | reinterpret_cast<uintptr_t>(b->mc_param) |
       reinterpret_cast<uintptr_t>(b->local_param)) & 15)
    return fail(OF_ERR_INVALID, "multicast buffers must be 16-byte aligned");
  if (slots >= 1 && !b->state0) return fail(OF_ERR_INVALID, "kind needs state0");
  if (slots >= 2 && !b->state1) return fail(OF_ERR_INVALID, "kind needs state1");
  McParams mp;
  mp.mc_grad = static_cast<float*>(b->mc_grad);
  mp.mc_param = static_cast<float*>(b->mc_param);
  mp.local_param = static_cast<const float*>(b->local_param);
  mp.s0 = static_cast<float*>(b->state0);
  mp.s1 = static_cast<float*>(b->state1);
  mp.begin = b->shard_begin;
  mp.len = b->shard_len;
  const StepSrc step = step_source(hp, flags);
  const int64_t nvec = mp.len / kVec;
  if (nvec == 0) return OF_OK;
  int64_t grid = (nvec + kThreads - 1) / kThreads;
  int64_t cap = static_cast<int64_t>(sm_count()) * kCtasPerSm;
  if (hp->max_ctas > 0 && hp->max_ctas < cap) cap = hp->max_ctas;
  if (grid > cap) grid = cap;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return with_op<float>(hp, [&](auto op) {
    mc_step_kernel<decltype(op)><<<static_cast<int>(grid), kThreads, 0, s>>>(mp, op, grad_scale_dev, step);
    return check_launch("mc_step_kernel");
  });
}

}  // extern "C"
