// k_fc1_tc.cu — the CNN's fc1 layer (F = 4096 -> HID = 512) on tcgen05 kind::tf32:
// forward, input gradient (with the pool2/ReLU backward fused in its epilogue) and the
// weight gradient with the SGD step fused in its epilogue.
//
// fc1 holds 97% of the CNN's parameters, so every client step streams its 8 MB weight
// matrix twice (forward; fused dX + dW: one read + one write); HBM-bound by design
// and the batch (|b| <= 32) rides in the MMA N dimension ("swap AB"):
//   forward  D[n][r]  = Σ_k W1[n][k] p2[r][k]      A = W1 tile   (K-major, SW128)
//                                                   B = p2 rows   (K-major, SW128)
//            split-K over k when few clients are active (deterministic partial sum).
//   dX       D[k][r]  = Σ_n W1[n][k] dh[r][n]      A = W1ᵀ tile  (MN-major, BASE32B)
//                                                   B = dh rows   (K-major, SW128)
//            epilogue: dp2 -> dY2 through pool2's argmax and ReLU' (writes every dY2 cell).
//   dW+SGD   D[n][k]  = Σ_r dh[r][n] p2[r][k]      A = dhᵀ, B = p2ᵀ (both MN-major), K = |b|
//            epilogue: W1 <- W1 − η·D (θ_g read on the first wave), b1 from Σ_r dh.
// Rows r >= |b| of a client's slots are zero in dh (k_head_fwd writes them) and finite in p2,
// so padding the batch to 32 never changes a sum.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_util.cuh"
#include "fl_internal.h"
#include "tc_common.cuh"

namespace flb {
namespace {

constexpr int NB = 32;   // batch slots per client in the MMA N (or K) dimension

// ------------------------------------------------------------------ forward
// a stage holds FW_KB consecutive 32-wide k-blocks (512-byte runs of every W1 row per TMA box)
constexpr int FW_KB = 4, FW_A = FW_KB * 128 * 128, FW_B = FW_KB * NB * 128, FW_STAGE = FW_A + FW_B, FW_NST = 2;
constexpr int FW_BAR = FW_NST * FW_STAGE, FW_SMEM = FW_BAR + 128 + 1024;

struct FwArgs {
  const int32_t* bs;
  int B, F, HID, wmul, ksplit, kpb;  // kpb: K-blocks (32 k) per split
  const float* bias;
  int64_t bias_stride;
  float* h;       // [S][HID]  (ksplit == 1)
  float* part;    // [A][ksplit][NB][HID] (ksplit > 1)
};

__global__ void __launch_bounds__(192, 1)
    k_fc1_fwd_tc(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX, FwArgs p) {
  static_assert(FW_NST * FW_STAGE + 128 + 1024 <= 227 * 1024, "shared memory");
  constexpr uint32_t IDESC = tc::idesc_tf32(128, NB, 0, 0);
  const int a = blockIdx.y, mt = blockIdx.x / p.ksplit, ks = blockIdx.x % p.ksplit;
  const int bs = p.bs[a];
  if (bs == 0) return;
  const int kb0 = ks * p.kpb, kb1 = min(p.F / 32, kb0 + p.kpb), nkb = (kb1 - kb0) / FW_KB;  // stages
  // PDL: wait for the previous kernel before taking TMEM (a parked CTA holding columns
  // would stall other streams' kernels) or touching anything it writes.
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip would turn every
  // epilogue access into a generic LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FW_BAR);
  uint64_t* empty = full + FW_NST;
  uint64_t* tfull = empty + FW_NST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapW);
      tc::prefetch_tmap(&mapX);
      for (int i = 0; i < FW_NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
      }
      tc::mbar_init(tfull, 1);
      tc::fence_mbar_init();
    }
    __syncwarp();
    tc::tmem_alloc<32>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  if (warp == 0) {
    if (tc::elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int st = i % FW_NST, ph = (i / FW_NST) & 1, kb = kb0 + i * FW_KB;
        tc::mbar_wait(empty + st, ph ^ 1);
        uint8_t* sa = smem + st * FW_STAGE;
        tc::mbar_expect_tx(full + st, FW_STAGE);
        tc::tma_load_4d(sa, &mapW, full + st, 0, 128 * mt, kb, a * p.wmul);  // [kb][128 n][32 k]
        tc::tma_load_3d(sa + FW_A, &mapX, full + st, 0, a * p.B, kb);         // [kb][32 r][32 k]
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      for (int i = 0; i < nkb; ++i) {
        const int st = i % FW_NST, ph = (i / FW_NST) & 1;
        tc::mbar_wait(full + st, ph);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(smem + st * FW_STAGE), sb = sa + FW_A;
#pragma unroll
        for (int k = 0; k < 4 * FW_KB; ++k)
          tc::mma_tf32(tbase, tc::sdesc(sa + (k >> 2) * 16384 + (k & 3) * 32, 0, 1024, tc::kSW128),
                       tc::sdesc(sb + (k >> 2) * 4096 + (k & 3) * 32, 0, 1024, tc::kSW128), IDESC, (i | k) != 0);
        tc::mma_commit(empty + st);
      }
      tc::mma_commit(tfull);
    }
  } else {
    const int qd = warp & 3, n = mt * 128 + qd * 32 + lane;
    tc::mbar_wait(tfull, 0);
    tc::tc_fence_after();
    float v[NB];
    tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16), *reinterpret_cast<float(*)[16]>(v));
    tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + 16, *reinterpret_cast<float(*)[16]>(v + 16));
    if (p.ksplit == 1) {
      const float b = p.bias[(int64_t)a * p.bias_stride * p.wmul + n];
      for (int r = 0; r < bs; ++r) {
        const float x = v[r] + b;
        p.h[((int64_t)a * p.B + r) * p.HID + n] = x > 0.f ? x : 0.f;
      }
    } else {
      float* out = p.part + (((int64_t)a * p.ksplit + ks) * NB) * p.HID + n;
      for (int r = 0; r < bs; ++r) out[(int64_t)r * p.HID] = v[r];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<32>(tbase);
}

// h = ReLU(Σ_splits part + b1), fixed split order.
__global__ void k_fc1_fwd_reduce(const float* __restrict__ part, const int32_t* __restrict__ bs, int B, int HID,
                                 int ksplit, const float* bias, int64_t bias_stride, int wmul, float* h) {
  pdl_wait();  // (PDL) previous kernel's writes visible; the implicit trigger is at exit
  const int a = blockIdx.z, r = blockIdx.y, n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= HID || r >= bs[a]) return;
  float s = 0.f;
  s = ordered_sum(part + (((int64_t)a * ksplit) * NB + r) * HID + n, ksplit, (int64_t)NB * HID);
  s += bias[(int64_t)a * bias_stride * wmul + n];
  h[((int64_t)a * B + r) * HID + n] = s > 0.f ? s : 0.f;
}

constexpr int DW_N = 128;  // W1 tile width in k (fc1_tc_supported requires F % DW_N == 0)

// ------------------------------------------------------------------ fused dX + dW + SGD
// Persistent over (client, 128-column k panel of W1) tiles; a panel is streamed in 4 chunks
// of 128 rows (n).  Each chunk (64 KB, SWIZZLE_128B_ATOM_32B, so it is directly the MN-major
// A operand of the dX MMA) is read from HBM once: the dX MMAs accumulate
// dp2[k][r] += Σ_n W1[n][k] dh[r][n] from the OLD values, the dW MMAs produce
// G[n][k] = Σ_r dh[r][n] p2[r][k] into a double-buffered TMEM tile, and only after both
// complete does the epilogue apply W1 <- W1 − η·G in shared memory and TMA-store the chunk.
// W1 is read once and written once per client step (separate dX / dW kernels read it
// twice).  After a panel's last chunk the epilogue routes dp2 through pool2's argmax / ReLU'
// into dY2.  The stage ring, the G buffers and the two dX accumulators run across tiles.
constexpr int BW_W = 4 * 128 * 128;               // 4 k-chunks x [128 n][32 k]
// dh, 4 chunks [32 r][32 n] in the SWIZZLE_128B_ATOM_32B layout, used twice: as the MN-major A
// of dW (n contiguous) and as the K-major B of dX (descriptor layout BASE32B, SBO = 512 —
// probed in scripts/tc_probe.cu), so one copy serves both MMAs
constexpr int BW_DHT = 4 * NB * 128;
constexpr int BW_STAGE = BW_W + BW_DHT;           // 80 KB
constexpr int BW_NST = 2;
constexpr int BW_P2B = 4 * NB * 128;              // p2ᵀ panel, 4 chunks [32 r][32 k] (MN-major B of dW)
constexpr int BW_P2 = BW_NST * BW_STAGE;          // two panels (double-buffered across tiles)
constexpr int BW_OUT = BW_P2 + 2 * BW_P2B;        // 2 x 16 KB store buffers: a stage is released as
constexpr int BW_BAR = BW_OUT + 2 * 16384;        // soon as the epilogue has read it, not when stored
constexpr int BW_SMEM = BW_BAR + 256 + 1024;
constexpr uint32_t BW_TCOLS = 512;                // G [0,128) [128,256); dX [256,288) [288,320)
constexpr int BW_EPI = 256;                       // epilogue threads (8 warps)
constexpr int BW_THREADS = 64 + BW_EPI;

struct BwArgs {
  const int32_t* bs;
  int A, B, HID, F, wmul;
  int H2, W2, C2;
  int H1, W1;          // conv2 output plane (pool2 input): 2·H2 x 2·W2, or one odd row / column more
  const float* p2;
  const uint8_t* am2;
  float* dY2;
  const float* bsrc;   // client 0 bias (θ_g on the first wave); client a at + a*bstride
  int64_t bstride;
  float* bdst;         // slot 0 bias; client a at + a*P_pad
  int64_t P_pad;
  const float* dh;     // [S][HID]
  float lr;
};

__global__ void __launch_bounds__(BW_THREADS, 1)
    k_fc1_bwd_tc(const __grid_constant__ CUtensorMap mapWsrc, const __grid_constant__ CUtensorMap mapWdst,
                 const __grid_constant__ CUtensorMap mapDht, const __grid_constant__ CUtensorMap mapX, BwArgs p) {
  constexpr uint32_t IDESC_DX = tc::idesc_tf32(128, NB, 1, 0);   // A (W1ᵀ) MN-major, B (dh) K-major
  constexpr uint32_t IDESC_DW = tc::idesc_tf32(128, 128, 1, 1);  // A (dhᵀ), B (p2ᵀ) MN-major
  const int KT = p.F / 128, T = p.A * KT, nch = p.HID / 128;
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip would turn every
  // epilogue access into a generic LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BW_BAR);
  uint64_t* empty = full + BW_NST;
  uint64_t* gfull = empty + BW_NST;
  uint64_t* gempty = gfull + 2;
  uint64_t* p2full = gempty + 2;    // [2]
  uint64_t* p2empty = p2full + 2;   // [2]
  uint64_t* dxfull = p2empty + 2;   // [2]
  uint64_t* dxempty = dxfull + 2;   // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dxempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapWsrc);
      tc::prefetch_tmap(&mapWdst);
      tc::prefetch_tmap(&mapDht);
      tc::prefetch_tmap(&mapX);
      for (int i = 0; i < BW_NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, BW_EPI);  // every epilogue thread, after its last read of the stage
      }
      for (int i = 0; i < 2; ++i) {
        tc::mbar_init(gfull + i, 1);
        tc::mbar_init(gempty + i, BW_EPI);
        tc::mbar_init(p2full + i, 1);
        tc::mbar_init(p2empty + i, BW_EPI);  // released by the dX epilogue (it reads p2 from the panel)
        tc::mbar_init(dxfull + i, 1);
        tc::mbar_init(dxempty + i, BW_EPI);
      }
      tc::fence_mbar_init();
    }
    __syncwarp();
    tc::tmem_alloc<BW_TCOLS>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  if (warp == 0) {
    // ---------------- producer
    if (tc::elect_one()) {
      int it = 0, ti = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int a = t / KT, kt = t % KT;
        if (p.bs[a] == 0) continue;
        const int pb = ti & 1, pph = (ti >> 1) & 1;
        ++ti;
        tc::mbar_wait(p2empty + pb, pph ^ 1);
        tc::mbar_expect_tx(p2full + pb, BW_P2B);
        tc::tma_load_3d(smem + BW_P2 + pb * BW_P2B, &mapX, p2full + pb, 0, a * p.B, 4 * kt);
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it % BW_NST, ph = (it / BW_NST) & 1;
          tc::mbar_wait(empty + st, ph ^ 1);
          uint8_t* sw = smem + st * BW_STAGE;
          tc::mbar_expect_tx(full + st, BW_STAGE);
          for (int j = 0; j < 4; ++j)
            tc::tma_load_3d(sw + j * 16384, &mapWsrc, full + st, 128 * kt + 32 * j, 128 * c, a * p.wmul);
          tc::tma_load_3d(sw + BW_W, &mapDht, full + st, 0, a * p.B, 4 * c);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (tc::elect_one()) {
      int it = 0, ti = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int a = t / KT;
        if (p.bs[a] == 0) continue;
        const int pb = ti & 1, pph = (ti >> 1) & 1;
        ++ti;
        tc::mbar_wait(p2full + pb, pph);
        tc::mbar_wait(dxempty + pb, pph ^ 1);  // dX accumulator pb drained by the epilogue
        const uint32_t up2 = tc::smem_u32(smem + BW_P2 + pb * BW_P2B);
        const uint32_t tdx = tbase + 256 + pb * 32;
        for (int c = 0; c < nch; ++c, ++it) {
          const int st = it % BW_NST, ph = (it / BW_NST) & 1, buf = it & 1, gph = (it >> 1) & 1;
          tc::mbar_wait(full + st, ph);
          tc::mbar_wait(gempty + buf, gph ^ 1);
          tc::tc_fence_after();
          const uint32_t uw = tc::smem_u32(smem + st * BW_STAGE), udht = uw + BW_W;
#pragma unroll
          for (int kk = 0; kk < 16; ++kk)  // dX: K = this chunk's 128 n, 8 per MMA (B = dh, K-major BASE32B)
            tc::mma_tf32(tdx, tc::sdesc(uw + kk * 1024, 16384, 512, tc::kSW128_32B),
                         tc::sdesc(udht + (kk >> 2) * 4096 + (kk & 3) * 32, 0, 512, tc::kSW128_32B), IDESC_DX,
                         (c | kk) != 0);
#pragma unroll
          for (int k = 0; k < 4; ++k)      // dW: K = 32 batch slots
            tc::mma_tf32(tbase + buf * 128, tc::sdesc(udht + k * 1024, NB * 128, 512, tc::kSW128_32B),
                         tc::sdesc(up2 + k * 1024, NB * 128, 512, tc::kSW128_32B), IDESC_DW, k != 0);
          tc::mma_commit(gfull + buf);
        }
        tc::mma_commit(dxfull + pb);
      }
    }
  } else {
    // ---------------- epilogue: 8 warps, two per TMEM lane quarter (warp % 4); half hf of a
    // pair takes columns [16 hf, 16 hf + 16) of every 32-column sub-chunk of G, and batch rows
    // [16 hf, 16 hf + 16) of dX.  Thread = n row of the chunk for G; = k row of the panel for dX.
    const int qd = warp & 3, row = qd * 32 + lane, hf = (warp - 2) >> 2;
    const bool storer = (warp == 2 && lane == 0);  // issues and retires the W stores (bulk groups are per thread)
    int it = 0, ti = 0, oi = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      const int a = t / KT, kt = t % KT;
      const int bs = p.bs[a];
      if (bs == 0) continue;
      const int pb = ti & 1, pph = (ti >> 1) & 1;
      ++ti;
      // pool2 argmax of this thread's dX row and batch half: loaded during the panel's last chunk
      // (few loads in flight while the SGD epilogue runs); p2 itself is read from the panel in smem
      const int k = kt * 128 + row, r0 = 16 * hf;
      uint32_t amb[16];  // pool2 argmax bytes of rows r0.. r0+15 (consumed only in the dX epilogue)
      for (int c = 0; c < nch; ++c, ++it) {
        const int st = it % BW_NST, buf = it & 1, gph = (it >> 1) & 1;
        uint8_t* sw = smem + st * BW_STAGE;
        if (c == nch - 1) {
#pragma unroll
          for (int r = 0; r < 16; ++r) amb[r] = r0 + r < bs ? __ldg(p.am2 + ((int64_t)a * p.B + r0 + r) * p.F + k) : 0u;
        }
        tc::mbar_wait(gfull + buf, gph);
        tc::tc_fence_after();
        if (kt == 0 && hf == 0) {  // bias: b1[n] -= η Σ_r dh[r][n], from the stage's dh chunk (ATOM_32B)
          const int n = 128 * c + row, nn = row & 31;
          const uint8_t* dq = sw + BW_W + (row >> 5) * 4096 + (nn & 7) * 4;
          float g = 0.f;
          for (int r = 0; r < bs; ++r) g += *reinterpret_cast<const float*>(dq + r * 128 + (((nn >> 3) ^ (r & 3)) << 5));
          p.bdst[(int64_t)a * p.P_pad + n] = p.bsrc[(int64_t)a * p.bstride * p.wmul + n] - p.lr * g;
        }
        for (int j = 0; j < 4; ++j, ++oi) {
          uint8_t* ob = smem + BW_OUT + (oi & 1) * 16384;
          float v[16];
          const uint32_t tg = tbase + ((uint32_t)(qd * 32) << 16) + buf * 128 + 32 * j + 16 * hf;
          // the old W1 values (32-byte granule g of the row sits at g ^ (row % 4), ATOM_32B) and the
          // gradient are read before the barrier: both loads overlap the wait for the store buffer
          const uint8_t* rowp = sw + j * 16384 + row * 128;
          float4 wv[2][2];
#pragma unroll
          for (int g2 = 0; g2 < 2; ++g2)
#pragma unroll
            for (int hq = 0; hq < 2; ++hq)
              wv[g2][hq] = reinterpret_cast<const float4*>(rowp + (((2 * hf + g2) ^ (row & 3)) << 5))[hq];
          tc::tmem_ld16(tg, v);
          if (storer) tc::bulk_wait_read<1>();  // the store issued from this buffer two sub-chunks ago has read it
          asm volatile("bar.sync 1, %0;" ::"n"(BW_EPI) : "memory");
          uint8_t* orow = ob + row * 128;
#pragma unroll
          for (int g2 = 0; g2 < 2; ++g2) {
            const int off = ((2 * hf + g2) ^ (row & 3)) << 5;
#pragma unroll
            for (int hq = 0; hq < 2; ++hq) {
              float4 w = wv[g2][hq];
              w.x -= p.lr * v[8 * g2 + 4 * hq];
              w.y -= p.lr * v[8 * g2 + 4 * hq + 1];
              w.z -= p.lr * v[8 * g2 + 4 * hq + 2];
              w.w -= p.lr * v[8 * g2 + 4 * hq + 3];
              reinterpret_cast<float4*>(orow + off)[hq] = w;
            }
          }
          tc::fence_async_smem();  // generic-proxy writes -> TMA store
          asm volatile("bar.sync 1, %0;" ::"n"(BW_EPI) : "memory");
          if (storer) {
            tc::tma_store_3d(&mapWdst, ob, 128 * kt + 32 * j, 128 * c, a);
            tc::bulk_commit();
          }
        }
        tc::tc_fence_before();
        tc::mbar_arrive(gempty + buf);  // G buffer drained
        tc::mbar_arrive(empty + st);    // this thread is done reading the stage
      }
      // dX epilogue: dp2 -> pool2 / ReLU backward -> dY2 (every cell of the 2x2 window written)
      tc::mbar_wait(dxfull + pb, pph);
      tc::tc_fence_after();
      float v[16];
      const uint32_t tdx = tbase + ((uint32_t)(qd * 32) << 16) + 256 + pb * 32 + 16 * hf;
      tc::tmem_ld16(tdx, v);
      tc::tc_fence_before();
      tc::mbar_arrive(dxempty + pb);
      // p2[r][k] from the panel (chunk k/32, row r, SWIZZLE_128B_ATOM_32B), then release it
      float p2v[16];
      {
        const uint8_t* pan = smem + BW_P2 + pb * BW_P2B + (row >> 5) * 4096 + (row & 7) * 4;
        const int g = (row & 31) >> 3;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const int rr = r0 + r;
          p2v[r] = *reinterpret_cast<const float*>(pan + rr * 128 + ((g ^ (rr & 3)) << 5));
        }
      }
      tc::mbar_arrive(p2empty + pb);
      const int cc = k % p.C2, pw = (k / p.C2) % p.W2, ph = k / (p.C2 * p.W2);
      const int W1 = p.W1, H1 = p.H1;  // a trailing odd row / column gets no gradient (floor pooling)
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        if (r0 + r >= bs) break;
        const int64_t s = (int64_t)a * p.B + r0 + r;
        const float g = p2v[r] > 0.f ? v[r] : 0.f;
        const int am = (int)amb[r];
        float* d = p.dY2 + ((s * H1 + 2 * ph) * W1 + 2 * pw) * p.C2 + cc;
        d[0] = am == 0 ? g : 0.f;
        d[p.C2] = am == 1 ? g : 0.f;
        d[(int64_t)W1 * p.C2] = am == 2 ? g : 0.f;
        d[(int64_t)W1 * p.C2 + p.C2] = am == 3 ? g : 0.f;
      }
    }
  }
  if (warp == 2 && lane == 0) tc::bulk_wait_all();  // smem must outlive the last stores
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();
  if (warp == 0) tc::tmem_dealloc<BW_TCOLS>(tbase);
}

template <class K>
void set_smem(K k, int bytes, bool& done) {
  if (!done) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    done = true;
  }
}

}  // namespace

bool fc1_tc_supported(const Layout& L, int B) {
  const CnnDims& d = L.d;
  // B: the slot pitch (the speech model's batch of 20 rides in 32-row slots, rows >= |b| zero)
  return B == NB && d.HID % 128 == 0 && d.F % DW_N == 0 && d.H1 / 2 == d.H2 && d.W1 / 2 == d.W2;
}

int64_t fc1_tc_part_floats(int64_t max_clients, const Layout& L) { return (max_clients + 2 * 148) * 16 * NB * L.d.HID; }

// forward: p2 -> h (split-K + reduce when few clients are active)
int fc1_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wclients, const float* p2,
               int64_t slots, float* h, float* part, int64_t part_floats, cudaStream_t st, int* launches) {
  const CnnDims& d = L.d;
  CUtensorMap mw, mx;
  // W1 viewed as [client][k-block][n][32 k] and p2 as [k-block][slot][32 k]: one box = FW_KB k-blocks
  uint64_t dw[4] = {32, (uint64_t)d.HID, (uint64_t)d.F / 32, (uint64_t)wclients};
  uint64_t sw[3] = {(uint64_t)d.F * 4, 128, (uint64_t)L.P_pad * 4};
  uint32_t bw[4] = {32, 128, FW_KB, 1};
  uint64_t dx[3] = {32, (uint64_t)slots, (uint64_t)d.F / 32};
  uint64_t sx[2] = {(uint64_t)d.F * 4, 128};
  uint32_t bx[3] = {32, NB, FW_KB};
  if (!tmap_encode(&mw, wbase + L.o_f1w, 4, dw, sw, bw, 1) || !tmap_encode(&mx, p2, 3, dx, sx, bx, 1)) return -1;
  const int mtiles = d.HID / 128, nkb = d.F / 32;
  static const int ctas = std::max(1, env_knob("FL_FC1F_CTAS", 2 * 148));
  int ksplit = (ctas + wa.A * mtiles - 1) / (wa.A * mtiles);
  ksplit = ksplit < 1 ? 1 : (ksplit > 16 ? 16 : ksplit);
  while (ksplit > 1 && (int64_t)wa.A * ksplit * NB * d.HID > part_floats) --ksplit;
  const int kpb = (nkb + ksplit * FW_KB - 1) / (ksplit * FW_KB) * FW_KB;  // whole stages per split
  ksplit = (nkb + kpb - 1) / kpb;
  static bool attr = false;
  set_smem(k_fc1_fwd_tc, FW_SMEM, attr);
  const int wmul = wa.first ? 0 : 1;
  FwArgs p{wa.bs, wa.B, d.F, d.HID, wmul, ksplit, kpb, wbase + L.o_f1b, L.P_pad, h, part};
  launch_pdl(wa.pdl, k_fc1_fwd_tc, dim3(mtiles * ksplit, wa.A), 192, FW_SMEM, st, mw, mx, p);
  *launches = 1;
  if (ksplit > 1) {
    launch_pdl(wa.pdl, k_fc1_fwd_reduce, dim3((d.HID + 127) / 128, wa.B, wa.A), 128, 0, st, part, wa.bs, wa.B, d.HID, ksplit,
                                                                       wbase + L.o_f1b, L.P_pad, wmul, h);
    *launches = 2;
  }
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

// fused dX + dW + SGD (one W1 pass): dh -> dY2 (pool2 / ReLU backward), W1, b1 updated
int fc1_bwd_tc(const Layout& L, const WaveArgs& wa, const float* wsrc, int64_t wclients_src, float* slots_w,
               int64_t wclients_dst, const float* dh, const float* p2, const uint8_t* am2, int64_t slots, float* dY2,
               cudaStream_t st) {
  const CnnDims& d = L.d;
  CUtensorMap mws, mwd, mdht, mx;
  uint64_t dws[3] = {(uint64_t)d.F, (uint64_t)d.HID, (uint64_t)wclients_src};
  uint64_t dwd[3] = {(uint64_t)d.F, (uint64_t)d.HID, (uint64_t)wclients_dst};
  uint64_t sww[2] = {(uint64_t)d.F * 4, (uint64_t)L.P_pad * 4};
  uint32_t bww[3] = {32, 128, 1};
  uint64_t dh3[3] = {32, (uint64_t)slots, (uint64_t)d.HID / 32};
  uint64_t sh3[2] = {(uint64_t)d.HID * 4, 128};
  uint32_t bh3[3] = {32, NB, 4};
  uint64_t dx3[3] = {32, (uint64_t)slots, (uint64_t)d.F / 32};
  uint64_t sx3[2] = {(uint64_t)d.F * 4, 128};
  uint32_t bx3[3] = {32, NB, 4};
  if (!tmap_encode(&mws, wsrc + L.o_f1w, 3, dws, sww, bww, 2) || !tmap_encode(&mwd, slots_w + L.o_f1w, 3, dwd, sww, bww, 2) ||
      !tmap_encode(&mdht, dh, 3, dh3, sh3, bh3, 2) ||
      !tmap_encode(&mx, p2, 3, dx3, sx3, bx3, 2))
    return -1;
  static bool attr = false;
  set_smem(k_fc1_bwd_tc, BW_SMEM, attr);
  BwArgs p{wa.bs, wa.A, wa.B, d.HID, d.F, wa.first ? 0 : 1, d.H2, d.W2, d.C2, d.H1, d.W1, p2, am2, dY2,
           wsrc + L.o_f1b, L.P_pad, slots_w + L.o_f1b, L.P_pad, dh, wa.lr};
  const int tiles = wa.A * (d.F / 128);
  launch_pdl(wa.pdl, k_fc1_bwd_tc, dim3(tiles < wa.sms ? tiles : wa.sms), BW_THREADS, BW_SMEM, st, mws, mwd, mdht, mx,
             p);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace flb
