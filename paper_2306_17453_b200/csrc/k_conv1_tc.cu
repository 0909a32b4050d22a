// k_conv1_tc.cu — the CIFAR CNN's first 5x5 conv (3 -> 32 channels, input padded to 4
// channels = one 16-byte pixel) on tcgen05 kind::tf32: forward and weight gradient.
//
// A 4-channel pixel is one 16-byte column of an 8x16B "core matrix", so both kernels use
// the no-swizzle (interleaved) operand layouts, again fed by TMA shifted copies of the
// input plane (zero padding from TMA's out-of-bounds fill):
//
// Forward (M = pixels, N = 32 channels, K = (tap, c)):  one CTA = one half-plane of a
//   sample (512 px = 4 M-tiles of 4 image rows, 4 accumulators x 32 columns).
//   copy_kw[h'][w][c] = x[16*half+h'-2][w+kw-2][c], h' in [0,21).  A of tap (kh, kw) for
//   tile j = copy_kw shifted by
//   (4j+kh) image rows; one MMA (K = 8) pairs taps (kh, kw) and (kh+1, kw) (LBO = one
//   image row); kh = 5 is a zero-weight pad tap.  B = weights per tap as [o][4] (TMA box
//   of the [o][tap][c] tensor, out-of-range taps read as zeros).  Epilogue: + bias -> a1.
//
// Weight gradient (M = (kw, c, kh) = 100 rows + bias, N = o = 32, K = pixels): see below.
//   Split-K over sample chunks -> partial [32][101] -> k_dw_reduce_sgd (SIMT, shared).
#include <cuda.h>

#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fl_internal.h"
#include "tc_common.cuh"

namespace flb {
namespace {

constexpr int H = 32, W = 32, C1 = 32, ROWB = W * 16;  // 512 B per image row of 4-channel pixels

// ------------------------------------------------------------------ forward
// Persistent: CTA b handles tiles t = b, b + grid, ... of the A·B·4 (client, sample,
// quadrant) tiles; a quadrant = 16 image rows x 16 columns = two M=128 tiles of 8 rows x 16
// px.  With a 16-pixel row pitch the 8-pixel core-matrix groups of an M tile are uniformly
// strided (SBO = 128 B), and the 2x2 pool window of accumulator row l lies in lanes l, l^1,
// l^16, l^17 of one warp, so the epilogue pools with shuffles.  Stages (4) hold the 5
// shifted copies of the quadrant's input (+halo) and the client's tap-major weights (one bulk
// copy from the c1wt side buffer the previous step's SGD wrote); TMEM accumulators are
// double-buffered so loads, MMAs and the epilogue of consecutive tiles overlap.
constexpr int Q_ROWS = 16 + 5;                  // 16 output rows + halo + the kh = 5 pad tap
constexpr int Q_ROWB = 16 * 16;                 // 256 B per 16-pixel row
constexpr int Q_COPY = Q_ROWS * Q_ROWB;         // 5376
constexpr int Q_A = 5 * Q_COPY;                 // 26880
constexpr int Q_B = C1WT_FLOATS * 4;            // 15360: [kw][kh = 0..5][32 o][4 c]
constexpr int Q_STAGE = Q_A + Q_B;              // 42240
constexpr int Q_NST = 4;
constexpr int XPITCH = 20;                      // floats per staged row (16 + 4: conflict-free v4 stores)
constexpr int Q_XCH = Q_NST * Q_STAGE;          // 8 epilogue warps x [32 rows][XPITCH]
constexpr int Q_BAR = Q_XCH + 8 * 32 * XPITCH * 4;
constexpr int Q_SMEM = Q_BAR + 128 + 1024;
static_assert(Q_STAGE % 128 == 0, "TMA destinations stay 128-byte aligned");

struct C1Args {
  const int32_t* sidx;
  const int32_t* bs;
  int A, B, wmul;
  const float* wt;    // tap-major weights of client 0; client a at + a*C1WT_FLOATS*wmul
  const float* bias;  // client 0 bias; client a at + a*stride*wmul
  int64_t bias_stride;
  float* p1;          // [S][16][16][32] pooled ReLU output
  uint8_t* am1;       // [S][16][16][32] window argmax
};

// 320 threads: warp 0 producer, warp 1 MMA, warps 2-9 epilogue (two per TMEM lane quarter,
// one per 16-channel half: the epilogue is issue-bound, so it gets the most warps).
constexpr int F_THREADS = 320;
__global__ void __launch_bounds__(F_THREADS, 1)
    k_conv1_fwd_tc(const __grid_constant__ CUtensorMap mapX, C1Args p) {
  constexpr uint32_t IDESC = tc::idesc_tf32(128, C1, 0, 0);
  const int T = p.A * p.B * 4;
  auto valid = [&](int t) { return ((t >> 2) % p.B) < p.bs[t / (4 * p.B)]; };
  // PDL: wait for the previous kernel before taking TMEM (a parked CTA holding columns
  // would stall other streams' kernels) or touching anything it writes.
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip would turn every
  // epilogue access into a generic LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Q_BAR);
  uint64_t* empty = full + Q_NST;
  uint64_t* afull = empty + Q_NST;
  uint64_t* aempty = afull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(aempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapX);
      for (int i = 0; i < Q_NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
      }
      for (int i = 0; i < 2; ++i) {
        tc::mbar_init(afull + i, 1);
        tc::mbar_init(aempty + i, F_THREADS - 64);
      }
      tc::fence_mbar_init();
    }
    __syncwarp();
    tc::tmem_alloc<128>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  if (warp == 0) {
    // ---------------- producer
    if (tc::elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        if (!valid(t)) continue;
        const int a = t / (4 * p.B), s = t >> 2, vh = (t >> 1) & 1, ch = t & 1;
        const int st = it % Q_NST, ph = (it / Q_NST) & 1;
        ++it;
        tc::mbar_wait(empty + st, ph ^ 1);
        uint8_t* sa = smem + st * Q_STAGE;
        tc::mbar_expect_tx(full + st, Q_STAGE);
        const int row = p.sidx[s];
        for (int kw = 0; kw < 5; ++kw)
          tc::tma_load_3d(sa + kw * Q_COPY, &mapX, full + st, 4 * (16 * ch + kw - 2), 16 * vh - 2, row);
        tc::bulk_load(sa + Q_A, p.wt + (int64_t)a * C1WT_FLOATS * p.wmul, Q_B, full + st);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (tc::elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        if (!valid(t)) continue;
        const int st = it % Q_NST, ph = (it / Q_NST) & 1, buf = it & 1, aph = (it >> 1) & 1;
        ++it;
        tc::mbar_wait(aempty + buf, aph ^ 1);
        tc::mbar_wait(full + st, ph);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(smem + st * Q_STAGE), sb = sa + Q_A;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int kw = 0; kw < 5; ++kw)
#pragma unroll
            for (int kp = 0; kp < 3; ++kp) {  // taps (2kp, kw) and (2kp+1, kw): LBO = one image row
              const uint64_t ad = tc::sdesc(sa + kw * Q_COPY + (8 * j + 2 * kp) * Q_ROWB, Q_ROWB, 128, tc::kSWNONE);
              const uint64_t bd = tc::sdesc(sb + (kw * 6 + 2 * kp) * 512, 512, 128, tc::kSWNONE);
              tc::mma_tf32(tbase + buf * 64 + j * C1, ad, bd, IDESC, (kw | kp) != 0);
            }
        tc::mma_commit(empty + st);
        tc::mma_commit(afull + buf);
      }
    }
  } else {
    // ---------------- epilogue: bias + ReLU + 2x2 max-pool (first maximum in row-major
    // window order, reading A13). A warp's 32 accumulator rows are 2 image rows x 16 px, so
    // every pool window lies inside the warp: stage (acc + bias) in a warp-private smem tile,
    // __syncwarp, then lane L pools channels 4(L&3).. of pooled column L>>2 (4 vector loads).
    const int qd = warp & 3, nh = (warp - 2) >> 2, n0 = nh * 16;
    float* xw = reinterpret_cast<float*>(smem + Q_XCH) + (warp - 2) * (32 * XPITCH);
    const int pc = lane >> 2, c4 = lane & 3;
    int it = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      if (!valid(t)) continue;
      const int a = t / (4 * p.B), s = t >> 2, vh = (t >> 1) & 1, ch = t & 1;
      const int buf = it & 1, aph = (it >> 1) & 1;
      ++it;
      const float* bias = p.bias + (int64_t)a * p.bias_stride * p.wmul + n0;
      float bv[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) bv[q] = __ldg(bias + q);
      tc::mbar_wait(afull + buf, aph);
      tc::tc_fence_after();
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float v[16];
        tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + buf * 64 + j * C1 + n0, v);
        float4* xr = reinterpret_cast<float4*>(xw + lane * XPITCH);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          xr[q] = make_float4(v[4 * q] + bv[4 * q], v[4 * q + 1] + bv[4 * q + 1], v[4 * q + 2] + bv[4 * q + 2],
                              v[4 * q + 3] + bv[4 * q + 3]);
        __syncwarp();
        const float4 x00 = *reinterpret_cast<const float4*>(xw + (2 * pc) * XPITCH + 4 * c4);
        const float4 x01 = *reinterpret_cast<const float4*>(xw + (2 * pc + 1) * XPITCH + 4 * c4);
        const float4 x10 = *reinterpret_cast<const float4*>(xw + (2 * pc + 16) * XPITCH + 4 * c4);
        const float4 x11 = *reinterpret_cast<const float4*>(xw + (2 * pc + 17) * XPITCH + 4 * c4);
        __syncwarp();  // the tile is rewritten by the next j
        float r[4];
        uint32_t am = 0;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const float a0 = (&x00.x)[cc], a1 = (&x01.x)[cc], a2 = (&x10.x)[cc], a3 = (&x11.x)[cc];
          float m = a0;
          uint32_t bi = 0;
          if (a1 > m) { m = a1; bi = 1; }
          if (a2 > m) { m = a2; bi = 2; }
          if (a3 > m) { m = a3; bi = 3; }
          r[cc] = m > 0.f ? m : 0.f;
          am |= bi << (8 * cc);
        }
        const int prow = 8 * vh + 4 * j + qd, pcol = 8 * ch + pc;
        const int64_t o = (((int64_t)s * 16 + prow) * 16 + pcol) * C1 + n0 + 4 * c4;
        *reinterpret_cast<float4*>(p.p1 + o) = make_float4(r[0], r[1], r[2], r[3]);
        *reinterpret_cast<uint32_t*>(p.am1 + o) = am;
      }
      tc::tc_fence_before();
      tc::mbar_arrive(aempty + buf);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<128>(tbase);
}

// Tap-major copy of conv1 weights for the forward's B operand: out[(kw*6+kh)*32+o][c] =
// w[o][kh*5+kw][c], zeros for the pad tap kh = 5.
__global__ void k_c1wt_pack(const float* __restrict__ w, float* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= C1WT_FLOATS) return;
  const int c = e & 3, o = (e >> 2) & 31, kk = e >> 7, kw = kk / 6, kh = kk % 6;
  out[e] = kh < 5 ? w[(o * 25 + kh * 5 + kw) * 4 + c] : 0.f;
}

// ------------------------------------------------------------------ weight gradient
// K-block = one image row h0 (32 pixels) of one sample.  A (M = taps x channels, K = px) is
// K-major SW128: row (kw, c, kh) = 32 consecutive pixels of input channel c, row h0+kh-2,
// shifted by kw-2 — one TMA box {32 w, 5 h, 4 c} of the planar (c, h, w) input per kw lands
// as 20 such rows.  Each kw block is padded to 24 rows (3 SW128 atoms); rows 120-127 hold a
// constant ones row (bias) and zeros.  B = dY1 row (32 px x 32 ch), MN-major BASE32B, is
// never read from HBM: TMA brings the pooled row h0/2 of dp1m and pool1's argmax, and the
// four epilogue warps expand it (pool1 backward: dY1 = dp1m at the window's argmax, else 0)
// into the stage's B tile before the MMA consumes it.
constexpr int D_KWB = 24 * 128;          // 3072 B per kw block (20 rows + 4 zero rows)
constexpr int D_A = 128 * 128;           // 16384: 5 kw blocks + constant rows 120..127
constexpr int D_B = 32 * 128;            // 4096
constexpr int D_RAW = 16 * 32 * 4 + 16 * 32;  // pooled-row dp1m (16 px x 32 ch fp32) + its argmax bytes
constexpr int D_STAGE = 23 * 1024;       // A + B + raw, 1024-aligned (SW128 operands)
constexpr int D_NST = 4;
constexpr int D_BAR = D_NST * D_STAGE;
constexpr int D_SMEM = D_BAR + 128 + 1024;
constexpr int D_TX = 5 * 20 * 128 + D_RAW;  // bytes TMA writes per stage (B is built by the expander warps)
static_assert(D_A + D_B + D_RAW <= D_STAGE, "stage layout");
constexpr int NPART = 25 * 4 + 1;        // partial row length per output channel (k_dw_reduce_sgd layout)

struct C1DwArgs {
  const int32_t* sidx;
  const int32_t* bpre;  // [A + 1] prefix sums of the wave's batch sizes
  int A, B, G;          // G CTAs split the wave's U k-blocks (H image rows per sample) evenly
  int64_t U;
  float* part;          // [A + G][32][101]: partial of (CTA c, client a) at z = a + c
};

// Largest a in [0, A) with bpre[a] <= x (the client owning concatenated sample x).
__device__ __forceinline__ int c1_client_of(const int32_t* __restrict__ bpre, int A, int64_t x) {
  int lo = 0, hi = A - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (bpre[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(192, 1)
    k_conv1_dw_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapD,
                  const __grid_constant__ CUtensorMap mapA, C1DwArgs p) {
  constexpr uint32_t IDESC = tc::idesc_tf32(128, C1, 0, 1);  // A K-major, B MN-major
  // Balanced split-K (as conv2's dW): CTA c reduces k-blocks [c·U/G, (c+1)·U/G) of the wave's
  // concatenated (client, sample, image row) sequence; each client segment ends with its
  // partial written to z = a + c.
  const int c = blockIdx.x;
  const int64_t u0 = (int64_t)c * p.U / p.G, u1 = (int64_t)(c + 1) * p.U / p.G;
  pdl_wait();
  const int a0 = c1_client_of(p.bpre, p.A, u0 / H);
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip would turn every
  // epilogue access into a generic LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + D_BAR);
  uint64_t* empty = full + D_NST;
  uint64_t* bready = empty + D_NST;  // B tile expanded (128 arrivals)
  uint64_t* tfull = bready + D_NST;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // constant rows of every stage (never written by TMA): pad rows 20-23 of each kw block = 0,
  // row 120 = ones (bias), rows 121-127 = 0
  for (int st = 0; st < D_NST; ++st) {
    float* sa = reinterpret_cast<float*>(smem + st * D_STAGE);
    for (int i = threadIdx.x; i < 5 * 4 * 32; i += blockDim.x) sa[(i / 128) * (D_KWB / 4) + 20 * 32 + i % 128] = 0.f;
    for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) sa[120 * 32 + i] = i < 32 ? 1.f : 0.f;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapX);
      tc::prefetch_tmap(&mapD);
      tc::prefetch_tmap(&mapA);
      for (int i = 0; i < D_NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
        tc::mbar_init(bready + i, 128);
      }
      tc::mbar_init(tfull, 1);
      tc::mbar_init(tempty, 128);
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
      int it = 0;
      for (int a = a0; a < p.A; ++a) {
        const int64_t kb0 = (int64_t)H * p.bpre[a];
        const int64_t ss = u0 > kb0 ? u0 : kb0, se = min(u1, (int64_t)H * p.bpre[a + 1]);
        if (ss >= u1) break;
        for (int64_t u = ss; u < se; ++u, ++it) {
          const int st = it % D_NST, ph = (it / D_NST) & 1;
          const int kk = (int)(u - kb0), rr = kk / H, h0 = kk % H;
          const int row = p.sidx[a * p.B + rr];
          tc::mbar_wait(empty + st, ph ^ 1);
          uint8_t* sa = smem + st * D_STAGE;
          tc::mbar_expect_tx(full + st, D_TX);
          // tap column kw = shifted copy (kw & 3) read from w' = (kw & 4): x[w + kw - 2]
          for (int kw = 0; kw < 5; ++kw)
            tc::tma_load_5d(sa + kw * D_KWB, &mapX, full + st, kw & 4, h0 - 2, 0, kw & 3, row);
          tc::tma_load_4d(sa + D_A + D_B, &mapD, full + st, 0, 0, h0 >> 1, a * p.B + rr);        // dp1m row
          tc::tma_load_4d(sa + D_A + D_B + 2048, &mapA, full + st, 0, 0, h0 >> 1, a * p.B + rr);  // am1 row
        }
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      int it = 0, si = 0;
      for (int a = a0; a < p.A; ++a, ++si) {
        const int64_t kb0 = (int64_t)H * p.bpre[a];
        const int64_t ss = u0 > kb0 ? u0 : kb0, se = min(u1, (int64_t)H * p.bpre[a + 1]);
        if (ss >= u1) break;
        tc::mbar_wait(tempty, (si & 1) ^ 1);  // previous segment's accumulator drained
        tc::tc_fence_after();
        for (int64_t u = ss; u < se; ++u, ++it) {
          const int st = it % D_NST, ph = (it / D_NST) & 1;
          tc::mbar_wait(bready + st, ph);  // A landed (the expanders waited on full) and B built
          tc::tc_fence_after();
          const uint32_t sa = tc::smem_u32(smem + st * D_STAGE), sb = sa + D_A;
#pragma unroll
          for (int k = 0; k < 4; ++k) {  // 8 pixels per MMA
            const uint64_t ad = tc::sdesc(sa + k * 32, 0, 1024, tc::kSW128);
            const uint64_t bd = tc::sdesc(sb + k * 1024, 4096, 512, tc::kSW128_32B);
            tc::mma_tf32(tbase, ad, bd, IDESC, (u != ss || k != 0) ? 1u : 0u);
          }
          tc::mma_commit(empty + st);
        }
        tc::mma_commit(tfull);
      }
    }
  } else {
    const int qd = warp & 3, m = qd * 32 + lane;  // row = kw*24 + c*5 + kh; 120 = bias
    int n = -1;
    if (m < 120 && (m % 24) < 20) {
      const int kw = m / 24, cc = (m % 24) / 5, kh = (m % 24) % 5;
      n = (kh * 5 + kw) * 4 + cc;
    } else if (m == 120) {
      n = 100;
    }
    int si = 0, it = 0;
    const int t = threadIdx.x - 64, w = t >> 2, q = t & 3;  // B row (pixel) w, channels 8q..8q+7
    for (int a = a0; a < p.A; ++a, ++si) {
      const int64_t kb0 = (int64_t)H * p.bpre[a];
      const int64_t ss = u0 > kb0 ? u0 : kb0, se = min(u1, (int64_t)H * p.bpre[a + 1]);
      if (ss >= u1) break;
      for (int64_t u = ss; u < se; ++u, ++it) {  // pool1 backward into the stage's B tile
        const int st = it % D_NST, ph = (it / D_NST) & 1;
        const int h0 = (int)((u - kb0) % H);
        tc::mbar_wait(full + st, ph);
        uint8_t* stage = smem + st * D_STAGE;
        const float* dp = reinterpret_cast<const float*>(stage + D_A + D_B) + (w >> 1) * 32 + 8 * q;
        const uint2 am = *reinterpret_cast<const uint2*>(stage + D_A + D_B + 2048 + (w >> 1) * 32 + 8 * q);
        const uint32_t code = (uint32_t)(((h0 & 1) << 1) | (w & 1));
        const float4 g0 = *reinterpret_cast<const float4*>(dp), g1 = *reinterpret_cast<const float4*>(dp + 4);
        const float4 o0 = make_float4((am.x & 0xff) == code ? g0.x : 0.f, ((am.x >> 8) & 0xff) == code ? g0.y : 0.f,
                                      ((am.x >> 16) & 0xff) == code ? g0.z : 0.f, (am.x >> 24) == code ? g0.w : 0.f);
        const float4 o1 = make_float4((am.y & 0xff) == code ? g1.x : 0.f, ((am.y >> 8) & 0xff) == code ? g1.y : 0.f,
                                      ((am.y >> 16) & 0xff) == code ? g1.z : 0.f, (am.y >> 24) == code ? g1.w : 0.f);
        // B row w (128 B = 32 channels), 32-byte granule q stored at q ^ (w % 4) (ATOM_32B)
        float4* bw = reinterpret_cast<float4*>(stage + D_A + w * 128 + ((q ^ (w & 3)) << 5));
        bw[0] = o0;
        bw[1] = o1;
        tc::fence_async_smem();  // generic-proxy writes -> tensor-core reads
        tc::mbar_arrive(bready + st);
      }
      tc::mbar_wait(tfull, si & 1);
      tc::tc_fence_after();
      float* out = p.part + (int64_t)(a + c) * C1 * NPART;
#pragma unroll
      for (int n0 = 0; n0 < C1; n0 += 16) {
        float v[16];
        tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + n0, v);
        if (n >= 0)
#pragma unroll
          for (int j = 0; j < 16; ++j) out[(n0 + j) * NPART + n] = v[j];
      }
      tc::tc_fence_before();
      tc::mbar_arrive(tempty);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<32>(tbase);
}

}  // namespace

// conv1 forward (+ bias) on tensor cores: packed input rows -> a1 (pre-activation).
int conv1_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, const float* wt, const float* xpack,
                 int64_t xrows, float* p1, uint8_t* am1, cudaStream_t st) {
  CUtensorMap mx;
  // a 16-pixel row segment (256 B) is the innermost box dimension; a one-pixel shift is a
  // 16-byte-aligned start coordinate (a 16-byte inner box made TMA the bottleneck)
  uint64_t dx[3] = {4 * W, H, (uint64_t)xrows};
  uint64_t sx[2] = {16 * W, 16 * W * H};
  uint32_t bx[3] = {64, Q_ROWS, 1};
  if (!tmap_encode(&mx, xpack, 3, dx, sx, bx, 0)) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv1_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, Q_SMEM);
    attr = true;
  }
  C1Args p{wa.sidx, wa.bs, wa.A, wa.B, wa.first ? 0 : 1, wt, wbase + L.o_c1b, L.P_pad, p1, am1};
  const int tiles = wa.A * wa.B * 4;
  launch_pdl(wa.pdl, k_conv1_fwd_tc, dim3(tiles < wa.sms ? tiles : wa.sms), F_THREADS, Q_SMEM, st, mx, p);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int c1wt_pack(const float* c1w, float* out, cudaStream_t st) {
  k_c1wt_pack<<<(C1WT_FLOATS + 255) / 256, 256, 0, st>>>(c1w, out);
  return 1;
}

// conv1 weight gradient on tensor cores: partials [A*nch][32][101] for k_dw_reduce_sgd.
int conv1_dw_tc(const Layout& L, const WaveArgs& wa, const float* xplanar, int64_t xrows, const float* dp1m,
                const uint8_t* am1, int64_t slots, float* part, int64_t part_cap, int* g_out, cudaStream_t st) {
  CUtensorMap mx, md, ma;
  constexpr int WP = W + 4;  // shifted planar copies [r][s][c][h][W+4]
  uint64_t dx[5] = {WP, H, 4, 4, (uint64_t)xrows};
  uint64_t sx[4] = {4 * WP, 4 * WP * H, 4 * WP * H * 4, 4 * WP * H * 16};
  uint32_t bx[5] = {W, 5, 4, 1, 1};
  // pooled rows of dp1m [S][16][16][32] fp32 and of am1 (u8, viewed as 8 x 4-byte words per pixel)
  uint64_t dd[4] = {32, W / 2, H / 2, (uint64_t)slots};
  uint64_t sd[3] = {128, 128 * (W / 2), 128 * (W / 2) * (H / 2)};
  uint32_t bd[4] = {32, W / 2, 1, 1};
  uint64_t da[4] = {8, W / 2, H / 2, (uint64_t)slots};
  uint64_t sa[3] = {32, 32 * (W / 2), 32 * (W / 2) * (H / 2)};
  uint32_t ba[4] = {8, W / 2, 1, 1};
  if (!tmap_encode(&mx, xplanar, 5, dx, sx, bx, 1) || !tmap_encode(&md, dp1m, 4, dd, sd, bd, 0) ||
      !tmap_encode(&ma, am1, 4, da, sa, ba, 0))
    return -1;
  // two CTAs per SM; at least half a sample (16 image rows) of work per CTA
  const int64_t U = (int64_t)H * wa.sum_bs;
  static const int minr = std::max(1, env_knob("FL_DW1_MINR", 16));
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(2 * wa.sms, U / minr));
  if ((int64_t)wa.A + G > part_cap) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv1_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, D_SMEM);
    attr = true;
  }
  C1DwArgs p{wa.sidx, wa.bpre, wa.A, wa.B, G, U, part};
  launch_pdl(wa.pdl, k_conv1_dw_tc, dim3(G), 192, D_SMEM, st, mx, md, ma, p);
  *g_out = G;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

bool conv1_tc_supported(const Layout& L) {
  return L.model == 1 && L.d.H0 == H && L.d.W0 == W && L.d.cpad == 4 && L.d.C1 == C1;
}

}  // namespace flb
