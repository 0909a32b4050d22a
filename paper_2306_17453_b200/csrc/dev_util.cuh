// dev_util.cuh — small device helpers shared by the SIMT and tensor-core kernels.
#pragma once
#include <stdint.h>

namespace flb {

// Σ_{i<n} p[i*stride] summed strictly in index order (deterministic), with the loads of each
// batch of 8 issued before any add so a latency-bound reduction makes one round trip per 8.
__device__ __forceinline__ float ordered_sum(const float* __restrict__ p, int n, int64_t stride) {
  float g = 0.f;
  int i = 0;
  for (; i + 8 <= n; i += 8) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldg(p + (int64_t)(i + j) * stride);
#pragma unroll
    for (int j = 0; j < 8; ++j) g += v[j];
  }
  for (; i < n; ++i) g += __ldg(p + (int64_t)i * stride);
  return g;
}

// Programmatic dependent launch (kernels launched with launch_pdl): let the next kernel in
// the stream start its prologue / block until the previous kernel's writes are visible.
// Both are no-ops for a kernel launched without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

}  // namespace flb
