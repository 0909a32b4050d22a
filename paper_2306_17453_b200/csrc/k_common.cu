// k_common.cu — HBM-streaming kernels of the round: fused per-GPU FedAvg accumulation
// (K1, Eq. 1-2 in delta form), finalize (K2), the ragged-pack
// gather (K3) and parameter layout permutes.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fl_internal.h"

namespace flb {

static inline int grid_for(int64_t n, int threads, int cap = 148 * 16) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)(g < cap ? g : cap);
}

// Streaming 16-byte load that does not allocate in L1 (each client slot is read once).
__device__ __forceinline__ float4 ld_stream4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------------
// K1: per GPU, S[p] = Σ_k n_k·(θ_k[p] − θ_g[p]) in fp64, clients in fixed order k = 0..K-1.
// One thread owns 4 consecutive parameters (16-byte loads); the client loop is unrolled
// by 8 so each thread keeps 8 independent 16-byte loads in flight.  Algorithmic bytes:
// 4·P·(K+1) read + (4 or 8)·P written.
// FINAL (world_size 1): fuses K2, out = fp32_rn(θ_g + S/N) (reading A2/A20).
// ---------------------------------------------------------------------------------
template <bool FINAL>
__global__ void __launch_bounds__(256) k_fedavg4(const float* __restrict__ slots, int64_t stride,
                                                 const int64_t* __restrict__ n, int K, int64_t P4,
                                                 const float* theta_g, double N, float* out, double* S) {
  // partial (world > 1): S[4·P4] = N_g, written by the kernel itself so no host value has
  // to outlive an asynchronous copy (N is N_local here)
  if (!FINAL && blockIdx.x == 0 && threadIdx.x == 0) S[4 * P4] = N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 g = reinterpret_cast<const float4*>(theta_g)[i];
    const double gx = g.x, gy = g.y, gz = g.z, gw = g.w;
    double ax = 0.0, ay = 0.0, az = 0.0, aw = 0.0;
    int k = 0;
    for (; k + 8 <= K; k += 8) {
      float4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = ld_stream4(reinterpret_cast<const float4*>(slots + (int64_t)(k + j) * stride) + i);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double w = (double)__ldg(n + k + j);
        ax = fma(w, (double)v[j].x - gx, ax);
        ay = fma(w, (double)v[j].y - gy, ay);
        az = fma(w, (double)v[j].z - gz, az);
        aw = fma(w, (double)v[j].w - gw, aw);
      }
    }
    for (; k < K; ++k) {
      const float4 v = ld_stream4(reinterpret_cast<const float4*>(slots + (int64_t)k * stride) + i);
      const double w = (double)__ldg(n + k);
      ax = fma(w, (double)v.x - gx, ax);
      ay = fma(w, (double)v.y - gy, ay);
      az = fma(w, (double)v.z - gz, az);
      aw = fma(w, (double)v.w - gw, aw);
    }
    if (FINAL) {
      float4 o;
      o.x = (float)(gx + ax / N);
      o.y = (float)(gy + ay / N);
      o.z = (float)(gz + az / N);
      o.w = (float)(gw + aw / N);
      reinterpret_cast<float4*>(out)[i] = o;
    } else {
      double2* s2 = reinterpret_cast<double2*>(S) + 2 * i;
      s2[0] = make_double2(ax, ay);
      s2[1] = make_double2(az, aw);
    }
  }
}

// Scalar variant for vectors whose length or stride is not a multiple of 4.
template <bool FINAL>
__global__ void k_fedavg1(const float* __restrict__ slots, int64_t stride, const int64_t* __restrict__ n, int K,
                          int64_t P, const float* theta_g, double N, float* out, double* S) {
  if (!FINAL && blockIdx.x == 0 && threadIdx.x == 0) S[P] = N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const double g = theta_g[i];
    double a = 0.0;
    for (int k = 0; k < K; ++k) a = fma((double)n[k], (double)slots[(int64_t)k * stride + i] - g, a);
    if (FINAL) out[i] = (float)(g + a / N);
    else S[i] = a;
  }
}

int fedavg_accum_final(const float* slots, int64_t stride, const int64_t* n, int K, int64_t P,
                       const float* theta_g, double N, float* out, cudaStream_t st) {
  bool vec = (P % 4 == 0) && (stride % 4 == 0) && ((uintptr_t)slots % 16 == 0) && ((uintptr_t)theta_g % 16 == 0) &&
             ((uintptr_t)out % 16 == 0);
  if (vec) {
    int64_t P4 = P / 4;
    k_fedavg4<true><<<grid_for(P4, 256, 1 << 20), 256, 0, st>>>(slots, stride, n, K, P4, theta_g, N, out, nullptr);
  } else {
    k_fedavg1<true><<<grid_for(P, 256), 256, 0, st>>>(slots, stride, n, K, P, theta_g, N, out, nullptr);
  }
  return 1;
}

// S[0..P) = Σ_k n_k(θ_k − θ_g) and S[P] = N_local (the [S_g ‖ N_g] vector of the allreduce).
int fedavg_accum_partial(const float* slots, int64_t stride, const int64_t* n, int K, int64_t P,
                         const float* theta_g, double N_local, double* S, cudaStream_t st) {
  bool vec = (P % 4 == 0) && (stride % 4 == 0) && ((uintptr_t)slots % 16 == 0) && ((uintptr_t)theta_g % 16 == 0);
  if (vec) {
    int64_t P4 = P / 4;
    k_fedavg4<false><<<grid_for(P4, 256, 1 << 20), 256, 0, st>>>(slots, stride, n, K, P4, theta_g, N_local, nullptr, S);
  } else {
    k_fedavg1<false><<<grid_for(P, 256), 256, 0, st>>>(slots, stride, n, K, P, theta_g, N_local, nullptr, S);
  }
  return 1;
}

int fedavg_preload() {
  cudaFuncAttributes a;
  const void* ks[] = {(const void*)k_fedavg4<true>, (const void*)k_fedavg4<false>, (const void*)k_fedavg1<true>,
                      (const void*)k_fedavg1<false>};
  for (const void* k : ks)
    if (cudaFuncGetAttributes(&a, k) != cudaSuccess) return -1;
  return 0;
}

// K2 after the cross-GPU reduce: θ_new = fp32_rn(θ_g + S/N), N = S[P] (exact in fp64).
__global__ void k_finalize(const double* __restrict__ S, int64_t P, const float* theta_g, const double* Ndev,
                           float* out) {
  const double N = *Ndev;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)((double)theta_g[i] + S[i] / N);
}

int fedavg_finalize(const double* S, int64_t P, const float* theta_g, const double* Ndev, float* out,
                    cudaStream_t st) {
  k_finalize<<<grid_for(P, 256), 256, 0, st>>>(S, P, theta_g, Ndev, out);
  return 1;
}

// ---------------------------------------------------------------------------------
// K3: ragged pack.  Packed row r <- population row src_row[r] (identity if null),
// CHW fp32 -> HWC with channels padded to 4 (16-byte pixels).
// ---------------------------------------------------------------------------------
__global__ void k_pack_cnn(const float* __restrict__ x, const int64_t* __restrict__ src_row, int64_t rows, int cin,
                           int HW, float* __restrict__ out, float* __restrict__ planar, int cpad) {
  const int64_t tot = rows * HW;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / HW;
    const int pix = (int)(e - r * HW);
    const int64_t s = src_row ? src_row[r] : r;
    const float* src = x + s * (int64_t)cin * HW + pix;
    if (cpad == 1) {  // one channel, unpadded
      out[e] = src[0];
      continue;
    }
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    v.x = src[0];
    if (cin > 1) v.y = src[HW];
    if (cin > 2) v.z = src[2 * HW];
    if (cin > 3) v.w = src[3 * HW];
    reinterpret_cast<float4*>(out)[e] = v;
  }
}

int pack_cnn(const Layout& L, const float* x_src, const int64_t* src_row, int64_t rows, float* xpack,
             float* xg, cudaStream_t st) {
  if (rows <= 0) return 0;
  int HW = L.d.H0 * L.d.W0;
  k_pack_cnn<<<grid_for(rows * HW, 256, 1 << 20), 256, 0, st>>>(x_src, src_row, rows, L.d.cin, HW, xpack, nullptr,
                                                                  L.d.cpad);
  if (!xg) return 1;
  return 1 + pack_xg(xpack, rows, xg, st);  // conv1 tensor-core window layout
}

__global__ void k_gather_rows(const float* __restrict__ src, const int64_t* __restrict__ src_row, int64_t rows,
                              int64_t dim, float* __restrict__ dst) {
  const int64_t tot = rows * dim;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / dim, c = e - r * dim;
    dst[e] = src[(src_row ? src_row[r] : r) * dim + c];
  }
}

int gather_rows_f32(const float* src, const int64_t* src_row, int64_t rows, int64_t dim, float* dst,
                    cudaStream_t st) {
  if (rows <= 0) return 0;
  k_gather_rows<<<grid_for(rows * dim, 256, 1 << 20), 256, 0, st>>>(src, src_row, rows, dim, dst);
  return 1;
}

__global__ void k_gather_i32(const int32_t* __restrict__ src, const int64_t* __restrict__ src_row, int64_t rows,
                             int32_t* __restrict__ dst) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
    dst[r] = src[src_row ? src_row[r] : r];
}

int gather_i32(const int32_t* src, const int64_t* src_row, int64_t rows, int32_t* dst, cudaStream_t st) {
  if (rows <= 0) return 0;
  k_gather_i32<<<grid_for(rows, 256), 256, 0, st>>>(src, src_row, rows, dst);
  return 1;
}

// ---------------------------------------------------------------------------------
// Canonical (torch state_dict) <-> internal (NHWC-friendly, padded) layouts.
// ---------------------------------------------------------------------------------
__global__ void k_c2i(const float* __restrict__ canon, const int64_t* __restrict__ canon_of, int64_t P_pad,
                      float* __restrict__ internal) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P_pad; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = canon_of[i];
    const float v = canon[c >= 0 ? c : 0];  // always an in-bounds load (padding slots read element 0)
    internal[i] = c >= 0 ? v : 0.f;
  }
}

__global__ void k_i2c(const float* __restrict__ internal, const int64_t* __restrict__ canon_of, int64_t P_pad,
                      float* __restrict__ canon) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P_pad; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = canon_of[i];
    if (c >= 0) canon[c] = internal[i];
  }
}

int canon_to_internal(const float* canon, const int64_t* canon_of, int64_t P_pad, float* internal,
                      cudaStream_t st) {
  k_c2i<<<grid_for(P_pad, 256), 256, 0, st>>>(canon, canon_of, P_pad, internal);
  return 1;
}

int internal_to_canon(const float* internal, const int64_t* canon_of, int64_t P_pad, float* canon,
                      cudaStream_t st) {
  k_i2c<<<grid_for(P_pad, 256), 256, 0, st>>>(internal, canon_of, P_pad, canon);
  return 1;
}

}  // namespace flb
