// k_convdw_tc.cu — weight gradient of the CIFAR CNN's 5x5 conv2 on tcgen05 (kind::tf32),
// with the SGD step in a split-K reduction kernel (SURVEY §8 a4 + a7).
//
//   dW2[o][tap][c] = Σ_px dY2[px][o] · p1[px + shift(tap)][c],   db2[o] = Σ_px dY2[px][o]
//
// GEMM with M = (tap, c) = 800 rows, N = o = 64, K = pixels.  One CTA reduces a chunk of
// one client's samples; all 800 rows live in TMEM at once (7 accumulators of 128 x 64 fp32
// plus one for the bias = 512 columns), so every K-block of 32 pixels (two image rows of a
// 16-column patch: CIFAR's 16 x 16 plane has 8 per sample, speech's 20 x 49 plane 10 x 4 with
// the columns past 49 zero-filled by TMA) is loaded exactly once:
//   A: five shifted copies copy_kw[h'][w][c] = p1[h0-2+h'][w+kw-2][c], h' in [0,6) (TMA,
//      zero fill at the borders); tap (kh, kw) is copy_kw shifted down by 16·kh rows.
//      Both operands are MN-major (32-bit MN-major = SWIZZLE_128B_BASE32B layout).
//   M tiles: (kw, kh = 0..3) for kw = 0..4 [LBO = 16 rows], (kh = 4, kw = 0..3) [LBO =
//      copy stride], tap (4,4) alone, and the bias tile: a constant ones operand with
//      LBO = 0, so D = Σ_px dY2 on every row.
//   B: dY2 rows of the block, 64 channels = two 32-wide MN chunks.
// The epilogue writes the chunk's partial [801][64]; k_dw2_reduce_sgd sums the chunks of a
// client and applies W <- W − η·g (θ_g read on the first wave, slot init fused).
#include <cuda.h>

#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_util.cuh"
#include "fl_internal.h"
#include "tc_common.cuh"

namespace flb {
namespace {

constexpr int COPY_ROWS = 6 * 16;                // 96 pixels per shifted copy
constexpr int COPY_BYTES = COPY_ROWS * 128;      // 12288
constexpr int A_BYTES = 5 * COPY_BYTES;          // 61440
constexpr int B_BYTES = 2 * 32 * 128;            // 8192 (dY2: 32 px x 64 ch, two MN chunks)
constexpr int STAGE = A_BYTES + B_BYTES;         // 69632
constexpr int NST = 2;
constexpr int ONES_OFF = NST * STAGE;            // 139264
constexpr int ONES_BYTES = 32 * 128;             // 32 K-rows x 32 ones
constexpr int BAR_OFF = ONES_OFF + ONES_BYTES;
constexpr int SMEM = BAR_OFF + 128 + 1024;
constexpr int NROW = 801;                        // 800 (tap, c) rows + bias
constexpr int NO = 64;

struct DwArgs {
  const int32_t* bpre;  // [A + 1] prefix sums of the wave's batch sizes
  int A, B, G;          // G CTAs split the wave's U k-blocks (kps per sample) evenly
  int64_t U;
  float* part;          // [A + G][64 o][801]: partial of (CTA c, client a) at z = a + c
  int kps, pw;          // k-blocks per sample = (H / 2) row pairs x pw 16-column patches
};

// Largest a in [0, A) with bpre[a] <= x (the client owning concatenated sample x).
__device__ __forceinline__ int client_of(const int32_t* __restrict__ bpre, int A, int64_t x) {
  int lo = 0, hi = A - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bpre[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Balanced split-K: CTA c reduces k-blocks [c·U/G, (c+1)·U/G) of the wave's concatenated
// (client, sample, 2-row block) sequence; each client segment of that range ends with its
// partial written to z = a + c (unique: CTA ranges are monotone in a).  The TMEM
// accumulators are reused across segments (tempty: the epilogue has drained them).
__global__ void __launch_bounds__(192, 1)
    k_conv2_dw_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapD, DwArgs p) {
  constexpr uint32_t IDESC = tc::idesc_tf32(128, NO, 1, 1);  // A and B MN-major
  const int c = blockIdx.x;
  const int64_t u0 = (int64_t)c * p.U / p.G, u1 = (int64_t)(c + 1) * p.U / p.G;
  // PDL: wait for the previous kernel before taking TMEM (a parked CTA holding columns
  // would stall other streams' kernels) or touching anything it writes.
  pdl_wait();
  const int a0 = client_of(p.bpre, p.A, u0 / p.kps);
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip would turn every
  // epilogue access into a generic LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  float* ones = reinterpret_cast<float*>(smem + ONES_OFF);
  for (int i = threadIdx.x; i < ONES_BYTES / 4; i += blockDim.x) ones[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapX);
      tc::prefetch_tmap(&mapD);
      for (int i = 0; i < NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
      }
      tc::mbar_init(tfull, 1);
      tc::mbar_init(tempty, 128);
      tc::fence_mbar_init();
    }
    __syncwarp();
    tc::tmem_alloc<512>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (tc::elect_one()) {
      int it = 0;
      for (int a = a0; a < p.A; ++a) {
        const int64_t kb0 = p.kps * (int64_t)p.bpre[a];
        const int64_t ss = u0 > kb0 ? u0 : kb0, se = min(u1, p.kps * (int64_t)p.bpre[a + 1]);
        if (ss >= u1) break;
        for (int64_t u = ss; u < se; ++u, ++it) {
          const int st = it % NST, ph = (it / NST) & 1;
          const int kk = (int)(u - kb0), s = a * p.B + kk / p.kps, r = kk % p.kps;
          const int h0 = 2 * (r / p.pw), x0 = 16 * (r % p.pw);
          tc::mbar_wait(empty + st, ph ^ 1);
          uint8_t* sa = smem + st * STAGE;
          tc::mbar_expect_tx(full + st, STAGE);
#pragma unroll
          for (int kw = 0; kw < 5; ++kw)
            tc::tma_load_4d(sa + kw * COPY_BYTES, &mapX, full + st, 0, x0 + kw - 2, h0 - 2, s);
          tc::tma_load_4d(sa + A_BYTES, &mapD, full + st, 0, x0, h0, s);
          tc::tma_load_4d(sa + A_BYTES + 4096, &mapD, full + st, 32, x0, h0, s);
        }
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      const uint32_t ones_a = tc::smem_u32(ones);
      int it = 0, si = 0;
      for (int a = a0; a < p.A; ++a, ++si) {
        const int64_t kb0 = p.kps * (int64_t)p.bpre[a];
        const int64_t ss = u0 > kb0 ? u0 : kb0, se = min(u1, p.kps * (int64_t)p.bpre[a + 1]);
        if (ss >= u1) break;
        tc::mbar_wait(tempty, (si & 1) ^ 1);  // previous segment's accumulators drained
        tc::tc_fence_after();
        for (int64_t u = ss; u < se; ++u, ++it) {
          const int st = it % NST, ph = (it / NST) & 1;
          tc::mbar_wait(full + st, ph);
          tc::tc_fence_after();
          const uint32_t sa = tc::smem_u32(smem + st * STAGE);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 8 pixels (K rows) per MMA
            const uint32_t acc = (u != ss || k != 0) ? 1u : 0u;
            const uint64_t bd = tc::sdesc(sb + k * 1024, 4096, 512, tc::kSW128_32B);
#pragma unroll
            for (int kw = 0; kw < 5; ++kw)  // tiles 0-4: taps (kh = 0..3, kw)
              tc::mma_tf32(tbase + kw * NO, tc::sdesc(sa + kw * COPY_BYTES + k * 1024, 2048, 512, tc::kSW128_32B),
                           bd, IDESC, acc);
            // tile 5: taps (kh = 4, kw = 0..3); tile 6: tap (4, 4); tile 7: bias (ones)
            tc::mma_tf32(tbase + 5 * NO, tc::sdesc(sa + 4 * 2048 + k * 1024, COPY_BYTES, 512, tc::kSW128_32B), bd,
                         IDESC, acc);
            tc::mma_tf32(tbase + 6 * NO,
                         tc::sdesc(sa + 4 * COPY_BYTES + 4 * 2048 + k * 1024, 0, 512, tc::kSW128_32B), bd, IDESC,
                         acc);
            tc::mma_tf32(tbase + 7 * NO, tc::sdesc(ones_a + k * 1024, 0, 512, tc::kSW128_32B), bd, IDESC, acc);
          }
          tc::mma_commit(empty + st);
        }
        tc::mma_commit(tfull);
      }
    }
  } else {
    const int qd = warp & 3, i = qd * 32 + lane;  // accumulator row
    int si = 0;
    for (int a = a0; a < p.A; ++a, ++si) {
      const int64_t kb0 = p.kps * (int64_t)p.bpre[a];
      if ((u0 > kb0 ? u0 : kb0) >= u1) break;
      tc::mbar_wait(tfull, si & 1);
      tc::tc_fence_after();
      float* out = p.part + (int64_t)(a + c) * NROW * NO;
#pragma unroll 1
      for (int t = 0; t < 8; ++t) {
        int row;  // partial row = tap*32 + c, or 800 for the bias
        if (t < 5) row = ((i >> 5) * 5 + t) * 32 + (i & 31);
        else if (t == 5) row = (20 + (i >> 5)) * 32 + (i & 31);
        else if (t == 6) row = qd == 0 ? 24 * 32 + lane : -1;
        else row = i == 0 ? 800 : -1;
#pragma unroll
        for (int n0 = 0; n0 < NO; n0 += 16) {
          float v[16];
          tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + t * NO + n0, v);  // warp-collective
          if (row >= 0)  // partial layout [o][row]: a warp's 32 rows are consecutive -> coalesced
#pragma unroll
            for (int j = 0; j < 16; ++j) out[(int64_t)(n0 + j) * NROW + row] = v[j];
        }
      }
      tc::tc_fence_before();
      tc::mbar_arrive(tempty);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

// Σ of a client's partials (CTAs c_first..c_last, in order), then SGD on conv2.w / conv2.b.
__global__ void k_dw2_reduce_sgd(const float* __restrict__ part, const int32_t* __restrict__ bpre, int G,
                                 int64_t U, int kps, const float* wsrc, int64_t wstride, float* dst, int64_t P_pad,
                                 int64_t o_w, int64_t o_b, float lr) {
  pdl_wait();  // (PDL) previous kernel's writes visible; the implicit trigger is at exit
  const int a = blockIdx.y;
  const int64_t v0 = kps * (int64_t)bpre[a], v1 = kps * (int64_t)bpre[a + 1] - 1;  // the client's k-blocks
  const int c0 = (int)(((v0 + 1) * G + U - 1) / U) - 1, c1 = (int)(((v1 + 1) * G + U - 1) / U) - 1;
  const float* pa = part + (int64_t)(a + c0) * NROW * NO;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < NROW * NO; e += gridDim.x * blockDim.x) {
    const float g = ordered_sum(pa + e, c1 - c0 + 1, (int64_t)NROW * NO);
    const int o = e / NROW, row = e - o * NROW;  // [o][row]: consecutive e -> consecutive W[o][tap][c]
    const int64_t idx = row < 800 ? o_w + (int64_t)o * 800 + row : o_b + o;
    dst[(int64_t)a * P_pad + idx] = wsrc[(int64_t)a * wstride + idx] - lr * g;
  }
}

bool make_maps(CUtensorMap* mx, CUtensorMap* md, const float* p1, const float* dY2, int H, int W, int64_t slots) {
  uint64_t dx[4] = {32, (uint64_t)W, (uint64_t)H, (uint64_t)slots};
  uint64_t sx[3] = {32 * 4, (uint64_t)32 * 4 * W, (uint64_t)32 * 4 * W * H};
  uint32_t bx[4] = {32, 16, 6, 1};
  uint64_t dd[4] = {64, (uint64_t)W, (uint64_t)H, (uint64_t)slots};
  uint64_t sd[3] = {64 * 4, (uint64_t)64 * 4 * W, (uint64_t)64 * 4 * W * H};
  uint32_t bd[4] = {32, 16, 2, 1};
  return tmap_encode(mx, p1, 4, dx, sx, bx, 2) && tmap_encode(md, dY2, 4, dd, sd, bd, 2);
}

}  // namespace

int conv2_dw_tc(const Layout& L, const WaveArgs& wa, const float* p1, const float* dY2, int64_t slots, float* part,
                int64_t part_cap, int* g_out, cudaStream_t st) {
  const CnnDims& d = L.d;
  CUtensorMap mx, md;
  if (!make_maps(&mx, &md, p1, dY2, d.H1, d.W1, slots)) return -1;
  // one CTA per SM (512 TMEM columns each), every CTA at least one sample of work
  const int kps = conv2_dw_kps(L), pw = (d.W1 + 15) / 16;
  const int64_t U = (int64_t)kps * wa.sum_bs;
  // at least `mins` samples per CTA (FL_DW2_MINS): each CTA writes a whole [801][64] partial, so
  // in small waves a finer split costs more SM time and traffic than it saves in latency
  static const int mins = std::max(1, env_knob("FL_DW2_MINS", 1));
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(wa.sms, (wa.sum_bs + mins - 1) / mins));
  if ((int64_t)wa.A + G > part_cap) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv2_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  DwArgs p{wa.bpre, wa.A, wa.B, G, U, part, kps, pw};
  launch_pdl(wa.pdl, k_conv2_dw_tc, dim3(G), 192, SMEM, st, mx, md, p);
  *g_out = G;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int conv2_dw_reduce_tc(const Layout& L, const WaveArgs& wa, const float* wsrc, int64_t wsrc_stride, float* dst,
                       const float* part, int G, cudaStream_t st) {
  const int kps = conv2_dw_kps(L);
  launch_pdl(wa.pdl, k_dw2_reduce_sgd, dim3((NROW * NO + 255) / 256, wa.A), 256, 0, st, part, wa.bpre, G,
             (int64_t)kps * wa.sum_bs, kps, wsrc, wsrc_stride, dst, L.P_pad, L.o_c2w, L.o_c2b, wa.lr);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int64_t conv2_dw_tc_part_z(int64_t max_clients) { return max_clients + 2 * 148; }
int conv2_dw_kps(const Layout& L) { return (L.d.H1 / 2) * ((L.d.W1 + 15) / 16); }
int64_t conv2_dw_tc_z_floats() { return (int64_t)NROW * NO; }

}  // namespace flb
