// k_peer.cu — cross-rank FedAvg over peer memory ("minimising
// server-GPU communication", §4.3 P:321-330 partial aggregation, P:203 / P:221-222 results
// shipped to a server).
//
// FL_AGG_PEER: ONE cooperative kernel per rank replaces partial -> ncclAllReduce -> finalize.
//   Phase A (every tile t of the parameter vector, all CTAs): this rank's fused fp64 partial
//     S_me[t] = Σ_{k local} n_k (θ_k − θ_g) (K1, same arithmetic as k_fedavg4), then a
//     release store of the round's sequence number into the tile OWNER's ready[me][t] word.
//   Phase B (tiles owned by this rank — a contiguous 1/W slice): acquire ready[j][t] for every
//     rank j, read S_j[t] from every peer (NVLink P2P loads; the same HBM when ranks share a
//     GPU), sum in rank order j = 0..W-1 (so every owner's result is the same function of the
//     partials), θ_new = fp32_rn(θ_g + S/N) with N = Σ n_k of the whole cohort (known to every
//     rank from the plan), stored into EVERY rank's θ_g (P2P stores), then done[t] = seq on
//     every rank.  Phase A of later tiles overlaps phase B of earlier ones across CTAs.
//   Phase C: acquire done[t] for every tile: θ_g is complete on this rank when the kernel ends.
//   Traffic per rank: 12·P·(W−1)/W bytes over the links (pull 8 B of S, push 4 B of θ_new per
//   parameter of its slice per peer) instead of shipping K_r models (4·P·K_r).
//   Deadlock freedom: every CTA finishes its phase-A tiles before it waits, and the launch is
//   cooperative (all CTAs co-resident), so a waiting CTA never blocks a tile it waits for; ranks
//   must run concurrently (separate GPUs, or disjoint green-context SM partitions of one GPU).
//
// FL_AGG_UNAGGREGATED (the ablation): every rank pushes each θ_k (fp32) into the server's (rank
// 0's) receive buffer and signals; the server averages all K models (k_fedavg4<true> over the
// receive buffer) and pushes θ_new into every rank.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fl_internal.h"

namespace flb {
namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Bounded spin: a peer that never arrives (a rank that died, or ranks that cannot run
// concurrently) traps after ~30 s instead of hanging the device; the ctx then reports FL_ERR_CUDA.
__device__ __forceinline__ void wait_geq(const unsigned long long* p, unsigned long long seq) {
  long long spins = 0;
  while (ld_acquire_sys(p) < seq) {
    __nanosleep(512);
    if (++spins > (1ll << 26)) __trap();
  }
}
// 16-byte streaming load that does not allocate in L1 (each client slot is read once)
__device__ __forceinline__ float4 ld_stream4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

__global__ void __launch_bounds__(256) k_fedavg_peer(PeerArgs p) {
  const int W = p.W, me = p.me, T = p.T;
  const unsigned long long seq = p.seq;
  unsigned long long* my_sig = p.r[me].sig;
  // ---- phase A: local partial, published to each tile's owner
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    const int64_t i0 = (int64_t)t * p.tile4, i1 = min(i0 + p.tile4, p.P4);
    double2* S = reinterpret_cast<double2*>(p.r[me].S);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const float4 g = reinterpret_cast<const float4*>(p.r[me].theta)[i];
      const double gx = g.x, gy = g.y, gz = g.z, gw = g.w;
      double ax = 0.0, ay = 0.0, az = 0.0, aw = 0.0;
      int k = 0;
      for (; k + 8 <= p.K; k += 8) {
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j)
          v[j] = ld_stream4(reinterpret_cast<const float4*>(p.slots + (int64_t)(k + j) * p.stride) + i);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const double w = (double)__ldg(p.n + k + j);
          ax = fma(w, (double)v[j].x - gx, ax);
          ay = fma(w, (double)v[j].y - gy, ay);
          az = fma(w, (double)v[j].z - gz, az);
          aw = fma(w, (double)v[j].w - gw, aw);
        }
      }
      for (; k < p.K; ++k) {
        const float4 v = ld_stream4(reinterpret_cast<const float4*>(p.slots + (int64_t)k * p.stride) + i);
        const double w = (double)__ldg(p.n + k);
        ax = fma(w, (double)v.x - gx, ax);
        ay = fma(w, (double)v.y - gy, ay);
        az = fma(w, (double)v.z - gz, az);
        aw = fma(w, (double)v.w - gw, aw);
      }
      S[2 * i] = make_double2(ax, ay);
      S[2 * i + 1] = make_double2(az, aw);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(p.r[peer_owner(t, T, W)].sig + (int64_t)me * T + t, seq);
    }
  }
  // ---- phase B: reduce + finalize + all-gather this rank's slice
  const int t0 = peer_slice_begin(me, T, W), t1 = peer_slice_begin(me + 1, T, W);
  for (int t = t0 + blockIdx.x; t < t1; t += gridDim.x) {
    if (threadIdx.x < W) wait_geq(my_sig + (int64_t)threadIdx.x * T + t, seq);
    __syncthreads();
    const int64_t i0 = (int64_t)t * p.tile4, i1 = min(i0 + p.tile4, p.P4);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      double sx = 0.0, sy = 0.0, sz = 0.0, sw = 0.0;
      for (int j = 0; j < W; ++j) {  // fixed rank order: identical on every owner
        const double2* Sj = reinterpret_cast<const double2*>(p.r[j].S);
        const double2 a = __ldcg(Sj + 2 * i), b = __ldcg(Sj + 2 * i + 1);
        sx += a.x, sy += a.y, sz += b.x, sw += b.y;
      }
      const float4 g = reinterpret_cast<const float4*>(p.r[me].theta)[i];
      float4 o;
      o.x = (float)((double)g.x + sx / p.N);
      o.y = (float)((double)g.y + sy / p.N);
      o.z = (float)((double)g.z + sz / p.N);
      o.w = (float)((double)g.w + sw / p.N);
      for (int j = 0; j < W; ++j) __stcg(reinterpret_cast<float4*>(p.r[j].theta) + i, o);
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
    __syncthreads();
    if (threadIdx.x < W) st_release_sys(p.r[threadIdx.x].sig + (int64_t)W * T + t, seq);
  }
  // ---- phase C: every slice of θ_g on this rank is final
  for (int t = blockIdx.x; t < T; t += gridDim.x)
    if (threadIdx.x == 0) wait_geq(my_sig + (int64_t)W * T + t, seq);
}

// Unaggregated ablation, client side: push this rank's slots into the server's receive buffer
// at rows dst_row[e] (plan positions), then (last CTA to finish) signal the server.
__global__ void __launch_bounds__(256) k_unagg_push(const float* __restrict__ slots, int64_t stride,
                                                    const int64_t* __restrict__ dst_row, int K, int64_t P4,
                                                    float* recv, unsigned long long* server_sig, int me,
                                                    unsigned long long seq, unsigned int* done_ctr) {
  const int64_t total = (int64_t)K * P4;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = q / P4, i = q - e * P4;
    const float4 v = ld_stream4(reinterpret_cast<const float4*>(slots + e * stride) + i);
    __stcg(reinterpret_cast<float4*>(recv + dst_row[e] * stride) + i, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(done_ctr, 1u) == gridDim.x - 1) {  // the last CTA: every push is visible
      __threadfence_system();
      *done_ctr = 0;
      st_release_sys(server_sig + me, seq);
    }
  }
}

// Wait until words sig[j·stride] >= seq for j in [j0, j1) (one thread per word).
__global__ void k_wait_flags(const unsigned long long* sig, int j0, int j1, int64_t stride, unsigned long long seq) {
  const int j = j0 + threadIdx.x;
  if (j < j1) wait_geq(sig + (int64_t)j * stride, seq);
}

// Server side after its fedavg: push θ_new into every other rank's θ_g, then signal them.
__global__ void __launch_bounds__(256) k_unagg_bcast(PeerArgs p, unsigned int* done_ctr) {
  const float4* src = reinterpret_cast<const float4*>(p.r[p.me].theta);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p.P4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    for (int j = 0; j < p.W; ++j)
      if (j != p.me) __stcg(reinterpret_cast<float4*>(p.r[j].theta) + i, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    if (atomicAdd(done_ctr, 1u) == gridDim.x - 1) {
      __threadfence_system();
      *done_ctr = 0;
      for (int j = 0; j < p.W; ++j)
        if (j != p.me) st_release_sys(p.r[j].sig + (int64_t)p.W * p.T, p.seq);
    }
  }
}

}  // namespace

// Load every kernel of the cross-rank protocol now: with CUDA's lazy module loading, the first
// launch of a kernel may wait for the device while a peer-waiting kernel spins on it.
int peer_preload() {
  cudaFuncAttributes a;
  const void* ks[] = {(const void*)k_fedavg_peer, (const void*)k_unagg_push, (const void*)k_wait_flags,
                      (const void*)k_unagg_bcast};
  for (const void* k : ks)
    if (cudaFuncGetAttributes(&a, k) != cudaSuccess) return -1;
  return fedavg_preload();
}

int fedavg_peer(const PeerArgs& p, int sms, cudaStream_t st) {
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fedavg_peer, 256, 0) != cudaSuccess || per_sm < 1)
    return -1;
  int grid = sms * (per_sm < 2 ? per_sm : 2);
  if (grid > p.T) grid = p.T;
  PeerArgs a = p;
  void* args[] = {&a};
  // cooperative: all CTAs co-resident, so a CTA waiting in phase B/C never starves a tile
  return cudaLaunchCooperativeKernel((const void*)k_fedavg_peer, dim3(grid), dim3(256), args, 0, st) == cudaSuccess
             ? 1
             : -1;
}

int unagg_push(const float* slots, int64_t stride, const int64_t* dst_row, int K, int64_t P4, float* recv,
               unsigned long long* server_sig, int me, unsigned long long seq, unsigned int* done_ctr, int sms,
               cudaStream_t st) {
  int64_t g = ((int64_t)K * P4 + 255) / 256;
  const int grid = (int)(g < 8 * sms ? (g < 1 ? 1 : g) : 8 * sms);
  k_unagg_push<<<grid, 256, 0, st>>>(slots, stride, dst_row, K, P4, recv, server_sig, me, seq, done_ctr);
  return 1;
}

int wait_flags(const unsigned long long* sig, int j0, int j1, int64_t stride, unsigned long long seq,
               cudaStream_t st) {
  if (j1 <= j0) return 0;
  k_wait_flags<<<1, 32 * ((j1 - j0 + 31) / 32), 0, st>>>(sig, j0, j1, stride, seq);
  return 1;
}

int unagg_bcast(const PeerArgs& p, unsigned int* done_ctr, int sms, cudaStream_t st) {
  int64_t g = (p.P4 + 255) / 256;
  const int grid = (int)(g < 4 * sms ? g : 4 * sms);
  k_unagg_bcast<<<grid, 256, 0, st>>>(p, done_ctr);
  return 1;
}

}  // namespace flb
