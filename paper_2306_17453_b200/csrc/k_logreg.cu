// k_logreg.cu — local SGD of the softmax-regression workload (BASELINE configs[0]).
// The model (7,850 parameters, 31 KB) fits in shared memory, so one CTA runs a client's
// whole ClientUpdate: every SGD step of every epoch, with the
// weights resident on chip, reading its batches through the wave sample table.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fl_internal.h"

namespace flb {
namespace {

constexpr int D = 784, NC = 10;

__global__ void __launch_bounds__(256) k_logreg(const float* __restrict__ xpack, const int32_t* __restrict__ ypack,
                                                const int32_t* __restrict__ sidx_all,
                                                const int64_t* __restrict__ slot_off, const int32_t* __restrict__ steps,
                                                int B, float lr, const float* __restrict__ theta_g, float* slots,
                                                int64_t P_pad) {
  extern __shared__ float sm[];
  float* W = sm;                 // [NC][D] then bias [NC]
  float* xs = W + NC * D + NC;   // [B][D]
  float* dz = xs + B * D;        // [B][NC]
  const int e = blockIdx.x, nsteps = steps[e];
  for (int i = threadIdx.x; i < NC * D + NC; i += blockDim.x) W[i] = theta_g[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = 0; t < nsteps; ++t) {
    const int32_t* sid = sidx_all + slot_off[t] + (int64_t)e * B;
    int b = 0;
    while (b < B && sid[b] >= 0) ++b;
    __syncthreads();  // previous step's update of W is complete
    for (int i = threadIdx.x; i < b * D; i += blockDim.x) {
      const int r = i / D, f = i - r * D;
      xs[i] = xpack[(int64_t)sid[r] * D + f];
    }
    __syncthreads();
    for (int idx = warp; idx < b * NC; idx += nw) {  // z = W x + b
      const int r = idx / NC, q = idx - r * NC;
      float s = 0.f;
      for (int f = lane; f < D; f += 32) s = fmaf(W[q * D + f], xs[r * D + f], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) dz[r * NC + q] = s + W[NC * D + q];
    }
    __syncthreads();
    if (threadIdx.x < b) {  // dz = (softmax(z) − onehot(y)) / |b|
      float* zr = dz + threadIdx.x * NC;
      const int y = ypack[sid[threadIdx.x]];
      float mx = zr[0];
      for (int q = 1; q < NC; ++q) mx = fmaxf(mx, zr[q]);
      float s = 0.f;
      for (int q = 0; q < NC; ++q) s += expf(zr[q] - mx);
      const float inv = 1.f / (float)b;
      for (int q = 0; q < NC; ++q) zr[q] = (expf(zr[q] - mx) / s - (q == y ? 1.f : 0.f)) * inv;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < NC * D; i += blockDim.x) {  // W <- W − η Σ_r dz_r x_rᵀ
      const int q = i / D, f = i - q * D;
      float g = 0.f;
      for (int r = 0; r < b; ++r) g = fmaf(dz[r * NC + q], xs[r * D + f], g);
      W[i] -= lr * g;
    }
    if (threadIdx.x < NC) {
      float g = 0.f;
      for (int r = 0; r < b; ++r) g += dz[r * NC + threadIdx.x];
      W[NC * D + threadIdx.x] -= lr * g;
    }
  }
  __syncthreads();
  float* out = slots + (int64_t)e * P_pad;
  for (int i = threadIdx.x; i < NC * D + NC; i += blockDim.x) out[i] = W[i];
}

}  // namespace

int logreg_train(const Layout& L, const WaveSched& ws, int n_local, int B, float lr, const float* xpack,
                 const int32_t* ypack, const float* theta_g, float* slots, const int32_t* steps_dev,
                 const int64_t* wave_slot_off_dev, cudaStream_t st) {
  if (n_local <= 0) return 0;
  size_t sm = sizeof(float) * (size_t)(NC * D + NC + B * D + B * NC);
  if (sm > 48 * 1024) cudaFuncSetAttribute(k_logreg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k_logreg<<<n_local, 256, sm, st>>>(xpack, ypack, ws.d_sidx, wave_slot_off_dev, steps_dev, B, lr, theta_g, slots,
                                     L.P_pad);
  return 1;
}

}  // namespace flb
