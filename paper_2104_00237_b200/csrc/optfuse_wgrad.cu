// optfuse_wgrad.cu -- consumer-fused backward fusion on sm_100a: the weight
// gradient GEMM of a Linear layer whose epilogue applies the optimizer update
// to the weight tile instead of writing the gradient to HBM.
//
// What this replaces in the reference (/root/reference/pkg/src/optfuse):
//   schedule.py:163-207 run_backward_fusion -- "update a parameter as soon as
//   its gradient is complete" -- taken to its limit: the gradient of a tile of
//   W is complete when the tensor cores finish that tile's accumulation, and
//   the update (OptimizerPolicy.step, optim.py:74-148, the same functors as
//   the multi-tensor kernel) runs right there, out of TMEM.  The gradient
//   never exists in HBM: per element the fused kernel moves the update's
//   read/write of theta and history (+ a bf16 shadow) and nothing else, where
//   the unfused pair writes dW, then reads it back (8 bytes per fp32 element).
//
// Appendix B.2 (schedule.py:54-59): W is read by this layer's input-gradient
// GEMM (dX = dY W).  The caller issues that GEMM first on the same stream, so
// every read of the old W precedes the update in stream order.
//
// Kernel (one 128 x BN output tile per cluster of S CTAs, 448 threads per CTA,
// warp-specialised):
//   split-K    the S CTAs of a cluster (S = 1, 2 or 4: enough CTAs to fill the
//              SMs when the layer has few output tiles, e.g. 36 for 768 x 768)
//              each accumulate 1/S of the tokens; after a cluster barrier every
//              CTA sends the rows it does not own to their owner's shared
//              memory (DSMEM), and each owner sums the S partials in rank order
//              and updates its rows -- the gradient still never reaches HBM;
//   warp 0     TMA producer: dY and X tiles (bf16, row-major [tokens][features],
//              i.e. MN-major operands) into a kStages-deep smem ring (6-8
//              stages, ~190 KB), 128B swizzle, completion on an mbarrier per stage;
//   warp 1     allocates TMEM (BN fp32 columns x 128 lanes) and one elected
//              lane issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N=BN,
//              K=16 per instruction) into the TMEM accumulator, releasing each
//              smem stage with tcgen05.commit;
//   warps 2-13 epilogue: during the mainloop, bulk L2 prefetches of the owned
//              theta/history rows; then tcgen05.ld of their TMEM lane quarter
//              (three warps per quarter, a third of the columns each) into the owner's
//              shared memory, and the update over the owned rows, 4 columns per
//              thread (12 warps: the update's division/square-root chains need
//              the warps to hide their latency).
// D[m][n] = sum_t dY[t][m] * X[t][n]  (= dW of y = x W^T, W: [out=M][in=N]).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cooperative_groups.h>
#include <cstring>
#include <utility>

#include "../../include/optfuse_b200.h"
#include "optfuse_ops.cuh"

namespace {
using namespace ofk;

constexpr int kBM = 128;          // UMMA_M: TMEM lane = output row
constexpr int kBK = 64;           // tokens per stage (one 128-byte swizzle row per token)
#ifndef OFW_EPI_WARPS
#define OFW_EPI_WARPS 12
#endif
constexpr int kEpiThreads = 32 * OFW_EPI_WARPS;  // 12 epilogue warps: enough to hide the update's latency chains
constexpr int kWThreads = 64 + kEpiThreads;   // warp 0 TMA, warp 1 MMA, warps 2.. epilogue
constexpr int kBox = 64;          // features per TMA box (64 bf16 = 128 B, the swizzle span)
#ifndef OFW_MAX_SPLIT
#define OFW_MAX_SPLIT 4
#endif
#ifndef OFW_RING_BYTES
#define OFW_RING_BYTES 196608
#endif
#ifndef OFW_MAX_BN      // widest output tile (256, 128)
#define OFW_MAX_BN 256
#endif
#ifndef OFW_NO_UPDATE   // 1: probe builds skip the epilogue's global traffic (mainloop timing)
#define OFW_NO_UPDATE 0
#endif
constexpr int kMaxSplit = OFW_MAX_SPLIT;   // CTAs per cluster (split-K ways)

template <int BN>
struct Layout {
  static constexpr int kA = kBM * kBK * 2;          // dY tile, bytes
  static constexpr int kB = BN * kBK * 2;           // X tile, bytes
  static constexpr int kStage = kA + kB;
  // the deepest ring that fits ~190 KB: 8 x 24 KB (BN 64), 6 x 32 KB (BN 128)
  static constexpr int kStages = OFW_RING_BYTES / kStage;
  static constexpr int kBoxBytes = kBox * kBK * 2;  // one [kBK][64] box = the MN stride (LBO)
  static constexpr int kSmem = kStages * kStage + 1024 /* 1024-B alignment slack */;
  static constexpr uint32_t kTmemCols = BN;         // power of two >= 32
  // epilogue staging (reuses the ring once every CTA's MMAs are done): S slots
  // of 128/S rows, i.e. always 128 padded rows of fp32
  static_assert(kBM * (BN + 4) * 4 <= kStages * kStage, "epilogue staging exceeds the ring");
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
               " selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}

// Bounded wait: a lost transaction traps (the launch fails) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t tries = 0;
  while (!mbar_try_wait(bar, parity))
    if (++tries > (1u << 26)) __trap();
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];"
      :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1),
         "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor, MN-major operand, 128-byte swizzle
// (cute::UMMA::SmemDescriptor): start address, LBO = byte stride between
// 64-element MN chunks (the TMA boxes), SBO = byte stride between 8-row
// groups along K (1024 B), version 1, layout type 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t umma_desc_mn_sw128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}

// Instruction descriptor of kind::f16: bf16 x bf16 -> f32, both operands
// MN-major (cute::UMMA::InstrDescriptor).
template <int BN>
__host__ __device__ constexpr uint32_t umma_idesc_bf16_mn() {
  return (1u << 4)                            // c_format F32
         | (1u << 7)                          // a_format BF16
         | (1u << 10)                         // b_format BF16
         | (1u << 15)                         // a_major MN
         | (1u << 16)                         // b_major MN
         | (static_cast<uint32_t>(BN >> 3) << 17)
         | (static_cast<uint32_t>(kBM >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
      :: "r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
               :: "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32"
      " {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
      " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct WgradParams {
  int M, N, T;            // out features, in features, tokens
  float* param;           // fp32 parameter or master [M][N]
  float* s0;              // history slots [M][N] (kind-dependent)
  float* s1;
  __nv_bfloat16* shadow;  // bf16 copy of the new parameter (OF_FLAG_SHADOW_BF16) or null
  float* grad_out;        // optional fp32 dump of the gradient (parity / debugging)
};

template <class Op, int BN>
__global__ void __launch_bounds__(kWThreads, 1)
wgrad_step_kernel(const __grid_constant__ CUtensorMap map_dy, const __grid_constant__ CUtensorMap map_x,
                  const WgradParams wp, const Op op_in, const StepSrc step) {
  using L = Layout<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  constexpr int kStages = L::kStages;
  __shared__ __align__(8) uint64_t full[kStages];
  __shared__ __align__(8) uint64_t empty[kStages];
  __shared__ __align__(8) uint64_t acc_full;
  __shared__ uint32_t tmem_base;

  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * kBM;
  const int n0 = blockIdx.x * BN;
  const int kblocks = (wp.T + kBK - 1) / kBK;
  // split-K: this CTA's token blocks [kb0, kb1) (the host keeps every split non-empty)
  const int S = static_cast<int>(gridDim.z);
  const int rank = static_cast<int>(blockIdx.z);
  const int kb_per = (kblocks + S - 1) / S;
  const int kb0 = rank * kb_per;
  const int kb1 = kb0 + kb_per < kblocks ? kb0 + kb_per : kblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {   // TMEM: BN columns x 128 lanes of fp32 accumulator
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(&tmem_base)), "r"(L::kTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;

  if (warp == 0) {
    if (lane == 0) {   // ===== TMA producer =====
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_dy)) : "memory");
      asm volatile("prefetch.tensormap [%0];" :: "l"(reinterpret_cast<uint64_t>(&map_x)) : "memory");
      for (int kb = kb0; kb < kb1; ++kb) {
        const int i = kb - kb0;
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        unsigned char* a = smem + s * L::kStage;
        unsigned char* b = a + L::kA;
        mbar_expect_tx(&full[s], L::kStage);
#pragma unroll
        for (int i = 0; i < kBM / kBox; ++i)
          tma_load_2d(a + i * L::kBoxBytes, &map_dy, m0 + i * kBox, kb * kBK, &full[s]);
#pragma unroll
        for (int i = 0; i < BN / kBox; ++i)
          tma_load_2d(b + i * L::kBoxBytes, &map_x, n0 + i * kBox, kb * kBK, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ===== MMA issuer =====
      constexpr uint32_t idesc = umma_idesc_bf16_mn<BN>();
      for (int kb = kb0; kb < kb1; ++kb) {
        const int i = kb - kb0;
        const int s = i % kStages;
        mbar_wait(&full[s], (i / kStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t a = smem_u32(smem + s * L::kStage);
        const uint32_t b = a + L::kA;
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {   // 16 tokens = 16 swizzle rows = 2048 B
          const uint64_t da = umma_desc_mn_sw128(a + k * 2048, L::kBoxBytes, 1024);
          const uint64_t db = umma_desc_mn_sw128(b + k * 2048, L::kBoxBytes, 1024);
          umma_bf16(tmem, da, db, idesc, (i | k) != 0);
        }
        umma_commit(&empty[s]);                 // stage free once these MMAs have read it
      }
      umma_commit(&acc_full);                   // accumulator complete
    }
  }
  // ===== epilogue =====
  // 1. every epilogue warp copies its 32-lane TMEM quarter (this CTA's partial
  //    of 32 rows) into the shared memory of the quarter's owner -- its own
  //    CTA unless split -- as [slot = rank][owned row][BN + 4 padding] fp32
  //    (16-byte rows: the 128-bit stores of 8 rows and the 128-bit loads of
  //    one row both hit 32 distinct banks);
  // 2. barrier (cluster-wide when split): all partials delivered;
  // 3. the owner's 384 epilogue threads sum each owned element's S partials in
  //    rank order and apply the update to 4 consecutive columns per thread, so
  //    the theta / history / shadow rows move as coalesced runs of BN * 4 bytes.
  constexpr int kPitch = BN + 4;
  const int q = warp & 3;                        // TMEM lane quarter this warp may access
  const int owner = (q * S) >> 2;                // the cluster rank that updates quarter q
  const int rows_owned = kBM / S;
  float* recv = reinterpret_cast<float*>(smem);  // the ring is free once the MMAs are done
  if (warp >= 2) {
    // While the tensor cores run, pull this CTA's owned rows of theta and
    // history into L2 (one bulk prefetch per row and stream), so the update
    // below reads them from L2 instead of waiting on HBM after the mainloop.
    if (!OFW_NO_UPDATE) {
      const int et = threadIdx.x - 64;
      const int ncols = (n0 + BN <= wp.N ? BN : wp.N - n0);
      for (int r = et; r < rows_owned * 3; r += kEpiThreads) {
        const int m = m0 + rank * rows_owned + r / 3;
        if (m >= wp.M || ncols <= 0) continue;
        const int which = r % 3;
        const float* base = which == 0 ? wp.param : which == 1 ? wp.s0 : wp.s1;
        if (base == nullptr) continue;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                     :: "l"(base + static_cast<int64_t>(m) * wp.N + n0), "r"(ncols * 4) : "memory");
      }
    }
    mbar_wait(&acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  __syncwarp();
  namespace cg = cooperative_groups;
  if (S > 1) cg::this_cluster().sync();          // every ring in the cluster is free
  if (warp >= 2) {
    const int orow = (q - (owner * 4) / S) * 32 + lane;   // row within the owner's rows
    float* base = recv + (static_cast<size_t>(rank) * rows_owned + orow) * kPitch;
    float* dst = S > 1 ? cg::this_cluster().map_shared_rank(base, owner) : base;
    const uint32_t tq = tmem + (static_cast<uint32_t>(q * 32) << 16);
    constexpr int kPerQuarter = kEpiThreads / 128;   // warps per lane quarter: they split the columns
    const int half = (warp - 2) >> 2;
#pragma unroll 1
    for (int c = half; c < BN / 32; c += kPerQuarter) {
      float g[32];
      tmem_ld_32x32b_x32(tq + c * 32, g);
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dst + c * 32 + j) = make_float4(g[j], g[j + 1], g[j + 2], g[j + 3]);
    }
  }
  if (S > 1) cg::this_cluster().sync();          // partials delivered
  else __syncthreads();
  if (warp >= 2) {
    Op op = op_in;
    if (step.offset != nullptr) {
      int64_t t = step.t_base + *step.offset;
      t = t < 1 ? 1 : (t >= step.rows ? step.rows - 1 : t);
      op.set_step(step.table[2 * t], step.table[2 * t + 1]);
    }
    const int et = threadIdx.x - 64;             // 0 .. kEpiThreads - 1
    constexpr int kQuads = BN / 4;               // float4 columns per row
    constexpr int kRowsPerPass = kEpiThreads / kQuads;   // 12 (BN 128) or 24 (BN 64)
    const int col = (et % kQuads) * 4;
    const int n = n0 + col;
    const int row_base = rank * rows_owned;      // first owned row of the tile
    constexpr int R = 4;                         // rows in flight per thread: all loads first
    float* __restrict__ P = wp.param;
    float* __restrict__ A = wp.s0;
    float* __restrict__ B = wp.s1;
#pragma unroll 1
    for (int r0 = et / kQuads; r0 < rows_owned; r0 += kRowsPerPass * R) {
      float g[R][4], pp[R][4], aa[R][4], bb[R][4];
      int64_t off[R];
      bool ok[R];
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int r = r0 + u * kRowsPerPass;
        const int m = m0 + row_base + r;
        ok[u] = r < rows_owned && m < wp.M && n < wp.N && !OFW_NO_UPDATE;
        off[u] = static_cast<int64_t>(m) * wp.N + n;
        if (!ok[u]) continue;
        const float4 g4 = *reinterpret_cast<const float4*>(recv + static_cast<size_t>(r) * kPitch + col);
        g[u][0] = g4.x; g[u][1] = g4.y; g[u][2] = g4.z; g[u][3] = g4.w;
        for (int k = 1; k < S; ++k) {            // the S partials in rank order
          const float4 h = *reinterpret_cast<const float4*>(
              recv + (static_cast<size_t>(k) * rows_owned + r) * kPitch + col);
          g[u][0] = __fadd_rn(g[u][0], h.x);
          g[u][1] = __fadd_rn(g[u][1], h.y);
          g[u][2] = __fadd_rn(g[u][2], h.z);
          g[u][3] = __fadd_rn(g[u][3], h.w);
        }
        const float4 pv = *reinterpret_cast<const float4*>(P + off[u]);
        pp[u][0] = pv.x; pp[u][1] = pv.y; pp[u][2] = pv.z; pp[u][3] = pv.w;
        if (Op::kSlots >= 1) {
          const float4 a = *reinterpret_cast<const float4*>(A + off[u]);
          aa[u][0] = a.x; aa[u][1] = a.y; aa[u][2] = a.z; aa[u][3] = a.w;
        }
        if (Op::kSlots >= 2) {
          const float4 b = *reinterpret_cast<const float4*>(B + off[u]);
          bb[u][0] = b.x; bb[u][1] = b.y; bb[u][2] = b.z; bb[u][3] = b.w;
        }
      }
#pragma unroll
      for (int u = 0; u < R; ++u) {
        if (!ok[u]) continue;
#pragma unroll
        for (int e = 0; e < 4; ++e) op(pp[u][e], g[u][e], aa[u][e], bb[u][e]);
        *reinterpret_cast<float4*>(P + off[u]) = make_float4(pp[u][0], pp[u][1], pp[u][2], pp[u][3]);
        if (Op::kSlots >= 1) *reinterpret_cast<float4*>(A + off[u]) = make_float4(aa[u][0], aa[u][1], aa[u][2], aa[u][3]);
        if (Op::kSlots >= 2) *reinterpret_cast<float4*>(B + off[u]) = make_float4(bb[u][0], bb[u][1], bb[u][2], bb[u][3]);
        if (wp.shadow) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(pp[u][0], pp[u][1]);
          __nv_bfloat162 hi = __floats2bfloat162_rn(pp[u][2], pp[u][3]);
          uint2 w;
          w.x = *reinterpret_cast<uint32_t*>(&lo);
          w.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(wp.shadow + off[u]) = w;
        }
        if (wp.grad_out)
          *reinterpret_cast<float4*>(wp.grad_out + off[u]) = make_float4(g[u][0], g[u][1], g[u][2], g[u][3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;"
                 :: "r"(tmem), "r"(L::kTmemCols) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// [rows][cols] bf16 row-major, boxes of 64 columns x kBK rows, 128-byte swizzle
int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols) {
  auto fn = encode_fn();
  if (!fn) return fail(OF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBox), static_cast<cuuint32_t>(kBK)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(OF_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return OF_OK;
}

template <class Op, int BN>
int launch_wgrad(const CUtensorMap& mdy, const CUtensorMap& mx, const WgradParams& wp, const Op& op,
                 const StepSrc& step, int split, cudaStream_t s) {
  using L = Layout<BN>;
  static bool configured = false;
  if (!configured) {
    if (cudaFuncSetAttribute(wgrad_step_kernel<Op, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             L::kSmem) != cudaSuccess)
      return fail(OF_ERR_CUDA, "cudaFuncSetAttribute(wgrad smem %d)", L::kSmem);
    configured = true;
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  cfg.blockDim = dim3(kWThreads);
  cfg.dynamicSmemBytes = L::kSmem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int tiles = ((wp.N + BN - 1) / BN) * ((wp.M + kBM - 1) / kBM);
  // every cluster must be resident at once (one CTA per SM, clusters confined
  // to a GPC): halve the split until the tiles' clusters fit in one wave
  static int fit_cache[kMaxSplit + 1] = {0};   // resident clusters per split (queried once)
  for (; split > 1; split /= 2) {
    attr[0].val.clusterDim.z = split;
    cfg.gridDim = dim3((wp.N + BN - 1) / BN, (wp.M + kBM - 1) / kBM, split);
    if (fit_cache[split] == 0) {
      int fit = 0;
      if (cudaOccupancyMaxActiveClusters(&fit, wgrad_step_kernel<Op, BN>, &cfg) != cudaSuccess || fit < 1)
        fit = -1;
      fit_cache[split] = fit;
    }
    if (tiles <= fit_cache[split]) break;
  }
  attr[0].val.clusterDim.z = split;
  cfg.gridDim = dim3((wp.N + BN - 1) / BN, (wp.M + kBM - 1) / kBM, split);
  cudaLaunchKernelEx(&cfg, wgrad_step_kernel<Op, BN>, mdy, mx, wp, op, step);
  return check_launch("wgrad_step_kernel");
}

}  // namespace

extern "C" int of_wgrad_step(const of_wgrad_args* a, const of_hparams* hp, uint32_t flags,
                             void* stream) {
  g_err[0] = '\0';
  if (!a || !hp) return fail(OF_ERR_INVALID, "wgrad: args or hparams is NULL");
  const int slots = hp->kind == OF_SGD ? 0
                    : (hp->kind == OF_SGD_MOMENTUM || hp->kind == OF_ADAGRAD || hp->kind == OF_RMSPROP) ? 1
                    : (hp->kind >= OF_ADADELTA && hp->kind <= OF_ADAMW) ? 2 : -1;
  if (slots < 0) return fail(OF_ERR_INVALID, "unknown optimizer kind %d", hp->kind);
  if (flags & ~(OF_FLAG_SHADOW_BF16 | OF_FLAG_DEVICE_STEP))
    return fail(OF_ERR_INVALID, "wgrad: flags 0x%x not supported (the gradient never exists in "
                "memory, so there is nothing to zero)", flags);
  if (!(hp->eta > 0.0)) return fail(OF_ERR_INVALID, "step size must be > 0, got %g", hp->eta);
  if (flags & OF_FLAG_DEVICE_STEP) {
    if (!hp->step_offset_dev || !hp->step_table_dev || hp->step_table_rows < 2)
      return fail(OF_ERR_INVALID, "OF_FLAG_DEVICE_STEP needs step_offset_dev and a step table");
  } else if ((hp->kind == OF_ADAM || hp->kind == OF_ADAMW) &&
             (hp->bias_correction1 == 0.0 || hp->bias_correction2 == 0.0)) {
    return fail(OF_ERR_INVALID, "adam bias corrections must be non-zero (step index t >= 1)");
  }
  if (a->out_features <= 0 || a->in_features <= 0 || a->tokens <= 0)
    return fail(OF_ERR_INVALID, "wgrad: empty problem %lld x %lld x %lld", (long long)a->out_features,
                (long long)a->in_features, (long long)a->tokens);
  if (a->in_features % 32 || a->out_features % 8)
    return fail(OF_ERR_UNSUPPORTED, "wgrad: in_features must be a multiple of 32 and out_features "
                "of 8 (got %lld, %lld)", (long long)a->in_features, (long long)a->out_features);
  if (a->out_features > (1 << 30) || a->in_features > (1 << 30) || a->tokens > (1 << 30))
    return fail(OF_ERR_UNSUPPORTED, "wgrad: dimension beyond 2^30");
  if (!a->grad_out_rows || !a->input || !a->param)
    return fail(OF_ERR_INVALID, "wgrad: dY, X and the parameter are required");
  if (slots >= 1 && !a->state0) return fail(OF_ERR_INVALID, "kind needs state0");
  if (slots >= 2 && !a->state1) return fail(OF_ERR_INVALID, "kind needs state1");
  if ((flags & OF_FLAG_SHADOW_BF16) && !a->shadow) return fail(OF_ERR_INVALID, "OF_FLAG_SHADOW_BF16 needs shadow");
  const uintptr_t al = reinterpret_cast<uintptr_t>(a->grad_out_rows) | reinterpret_cast<uintptr_t>(a->input) |
                       reinterpret_cast<uintptr_t>(a->param) | reinterpret_cast<uintptr_t>(a->state0) |
                       reinterpret_cast<uintptr_t>(a->state1) | reinterpret_cast<uintptr_t>(a->grad_dump);
  if (al & 15) return fail(OF_ERR_INVALID, "wgrad: buffers must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(a->shadow) & 7) return fail(OF_ERR_INVALID, "wgrad: shadow must be 8-byte aligned");
  CUtensorMap mdy, mx;
  int st = make_map(&mdy, a->grad_out_rows, a->tokens, a->out_features);
  if (st != OF_OK) return st;
  st = make_map(&mx, a->input, a->tokens, a->in_features);
  if (st != OF_OK) return st;
  WgradParams wp;
  wp.M = static_cast<int>(a->out_features);
  wp.N = static_cast<int>(a->in_features);
  wp.T = static_cast<int>(a->tokens);
  wp.param = static_cast<float*>(a->param);
  wp.s0 = static_cast<float*>(a->state0);
  wp.s1 = static_cast<float*>(a->state1);
  wp.shadow = (flags & OF_FLAG_SHADOW_BF16) ? static_cast<__nv_bfloat16*>(a->shadow) : nullptr;
  wp.grad_out = static_cast<float*>(a->grad_dump);
  const StepSrc step = (flags & OF_FLAG_DEVICE_STEP)
                           ? StepSrc{hp->step_offset_dev, hp->step_table_dev, hp->step_table_rows, hp->t_base}
                           : StepSrc{nullptr, nullptr, 0, 0};
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // The widest tile the columns allow (a 128 x 256 tile reads 25% fewer L2
  // bytes per flop than 128 x 128: the mainloop is L2-bandwidth-bound);
  // split-K across a cluster of 2 or 4 CTAs while that still fits the SMs and
  // leaves each split >= 4 token blocks
  const int kblocks = (wp.T + kBK - 1) / kBK;
  auto split_for = [&](int bn_) {
    const int64_t tiles = static_cast<int64_t>((wp.M + kBM - 1) / kBM) * ((wp.N + bn_ - 1) / bn_);
    int sp = 1;
    while (sp < kMaxSplit && tiles * sp * 2 <= sm_count() && kblocks >= 4 * sp * 2) sp *= 2;
    return std::make_pair(sp, tiles * sp);   // (split, CTAs)
  };
  int bn = wp.N % 128 == 0 ? 128 : 64;
  // 256-wide only where it still fills ~all SMs (768 x 768 would halve them)
  if (wp.N % 256 == 0 && OFW_MAX_BN >= 256 && split_for(256).second * 10 >= sm_count() * 9) bn = 256;
  const int split = split_for(bn).first;
  return with_op<float>(hp, [&](auto op) {
    if (bn == 256) return launch_wgrad<decltype(op), 256>(mdy, mx, wp, op, step, split, s);
    if (bn == 128) return launch_wgrad<decltype(op), 128>(mdy, mx, wp, op, step, split, s);
    return launch_wgrad<decltype(op), 64>(mdy, mx, wp, op, step, split, s);
  });
}
