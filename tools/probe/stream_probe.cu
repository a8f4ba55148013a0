// HBM streaming probe (diagnostic, not product): pure copies with the update
// kernel's access pattern -- R read streams and W write streams of float4, a
// grid-stride loop issuing every load of UNR vectors before any store -- to
// see what the memory system gives each pattern on this B200.
#include <cuda_runtime.h>
#include <cstdint>

template <int R, int W, int UNR>
__global__ void __launch_bounds__(256) stream_kernel(const float4* __restrict__ i0, const float4* __restrict__ i1,
                                                      const float4* __restrict__ i2, const float4* __restrict__ i3,
                                                      float4* __restrict__ o0, float4* __restrict__ o1,
                                                      float4* __restrict__ o2, int64_t nvec) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * 256 * UNR;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * 256 * UNR + threadIdx.x; base < nvec; base += stride) {
    float4 a[UNR][4];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        a[u][0] = i0[j];
        if (R > 1) a[u][1] = i1[j];
        if (R > 2) a[u][2] = i2[j];
        if (R > 3) a[u][3] = i3[j];
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t j = base + u * 256;
      if (j < nvec) {
        float4 s = a[u][0];
        if (R > 1) { s.x += a[u][1].x; s.y += a[u][1].y; s.z += a[u][1].z; s.w += a[u][1].w; }
        if (R > 2) { s.x += a[u][2].x; s.y += a[u][2].y; s.z += a[u][2].z; s.w += a[u][2].w; }
        if (R > 3) { s.x += a[u][3].x; s.y += a[u][3].y; s.z += a[u][3].z; s.w += a[u][3].w; }
        o0[j] = s;
        if (W > 1) o1[j] = a[u][R > 1 ? 1 : 0];
        if (W > 2) o2[j] = a[u][R > 2 ? 2 : 0];
      }
    }
  }
}

extern "C" int probe_stream(int r, int w, int unr, int grid, const void* i0, const void* i1, const void* i2,
                            const void* i3, void* o0, void* o1, void* o2, int64_t nvec, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto I0 = static_cast<const float4*>(i0), I1 = static_cast<const float4*>(i1);
  auto I2 = static_cast<const float4*>(i2), I3 = static_cast<const float4*>(i3);
  auto O0 = static_cast<float4*>(o0), O1 = static_cast<float4*>(o1), O2 = static_cast<float4*>(o2);
#define L(R_, W_, U_) if (r == R_ && w == W_ && unr == U_) { stream_kernel<R_, W_, U_><<<grid, 256, 0, s>>>(I0, I1, I2, I3, O0, O1, O2, nvec); return cudaGetLastError(); }
  L(1, 1, 4) L(1, 1, 8) L(4, 3, 2) L(4, 3, 4) L(3, 2, 4) L(2, 2, 4)
#undef L
  return -1;
}
