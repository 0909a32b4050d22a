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
#include <cuda_runtime.h>
#include <stdint.h>

#include "fl_internal.h"
#include "tc_common.cuh"

namespace flb {
namespace {

constexpr int H = 32, W = 32, C1 = 32, ROWB = W * 16;  // 512 B per image row of 4-channel pixels

// ------------------------------------------------------------------ forward
// One CTA = one half-plane (16 image rows = 4 M-tiles) of a sample, so two CTAs fit per SM
// and one's loads / epilogue overlap the other's MMAs.
constexpr int F_ROWS = 16 + 5;                  // output rows + halo + the kh = 5 pad tap
constexpr int F_COPY = F_ROWS * ROWB;           // 10752 B
constexpr int F_A = 5 * F_COPY;                 // 53760
constexpr int F_B = 30 * 512;                   // (kw, kh = 0..5) x [32 o][4 c]
constexpr int F_XCH = F_A + F_B;                // epilogue exchange buffer [4][32][16] fp32
constexpr int F_BAR = F_XCH + 4 * 32 * 16 * 4;
constexpr int F_SMEM = F_BAR + 64 + 1024;

struct C1Args {
  const int32_t* sidx;
  const int32_t* bs;
  int B, wmul;
  const float* bias;  // client 0 bias; client a at + a*stride*wmul
  int64_t bias_stride;
  float* p1;          // [S][16][16][32] pooled ReLU output
  uint8_t* am1;       // [S][16][16][32] window argmax
};

__global__ void __launch_bounds__(192, 2)
    k_conv1_fwd_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW, C1Args p) {
  constexpr uint32_t IDESC = tc::idesc_tf32(128, C1, 0, 0);
  const int r = blockIdx.x >> 1, half = blockIdx.x & 1, a = blockIdx.y;
  if (r >= p.bs[a]) return;
  const int s = a * p.B + r;
  // PDL: wait for the previous kernel before taking TMEM (a parked CTA holding columns
  // would stall other streams' kernels) or touching anything it writes.
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F_BAR);
  uint64_t* tfull = full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::mbar_init(full, 1);
      tc::mbar_init(tfull, 1);
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
    if (tc::elect_one()) {
      const int row = p.sidx[s];
      tc::mbar_expect_tx(full, F_A + F_B);
      for (int kw = 0; kw < 5; ++kw)
        tc::tma_load_4d(smem + kw * F_COPY, &mapX, full, 0, kw - 2, 16 * half - 2, row);
      for (int kw = 0; kw < 5; ++kw)
        for (int kh = 0; kh < 6; ++kh)  // tap 25..29 (kh = 5) is out of range -> zeros
          tc::tma_load_4d(smem + F_A + (kw * 6 + kh) * 512, &mapW, full, 0, kh * 5 + kw, 0, a * p.wmul);
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      tc::mbar_wait(full, 0);
      tc::tc_fence_after();
      const uint32_t sa = tc::smem_u32(smem), sb = sa + F_A;
      for (int j = 0; j < 4; ++j)
        for (int kw = 0; kw < 5; ++kw)
          for (int kp = 0; kp < 3; ++kp) {  // taps (2kp, kw) and (2kp+1, kw)
            const uint64_t ad = tc::sdesc(sa + kw * F_COPY + (4 * j + 2 * kp) * ROWB, ROWB, 128, tc::kSWNONE);
            const uint64_t bd = tc::sdesc(sb + (kw * 6 + 2 * kp) * 512, 512, 128, tc::kSWNONE);
            tc::mma_tf32(tbase + j * C1, ad, bd, IDESC, (kw | kp) != 0);
          }
      tc::mma_commit(tfull);
    }
  } else {
    const int qd = warp & 3;
    tc::mbar_wait(tfull, 0);
    tc::tc_fence_after();
    // bias + ReLU + 2x2 max-pool (first maximum in row-major window order, reading A13).
    // Tile j holds image rows 16*half + 4j..+3, one row per warp; the vertical window partner is
    // in the next warp, so each 16-channel chunk is exchanged through shared memory.
    const float* bias = p.bias + (int64_t)a * p.bias_stride * p.wmul;
    float* xb = reinterpret_cast<float*>(smem + F_XCH);  // [4 rows][32 w][16 c]
    const int t = threadIdx.x - 64;                    // 0..127 over the epilogue warps
    for (int j = 0; j < 4; ++j) {
#pragma unroll 1
      for (int n0 = 0; n0 < C1; n0 += 16) {
        float v[16];
        tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + j * C1 + n0, v);
        float4* xr = reinterpret_cast<float4*>(xb + (qd * 32 + lane) * 16);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          xr[i] = make_float4(v[4 * i] + bias[n0 + 4 * i], v[4 * i + 1] + bias[n0 + 4 * i + 1],
                              v[4 * i + 2] + bias[n0 + 4 * i + 2], v[4 * i + 3] + bias[n0 + 4 * i + 3]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // thread t -> pooled row (t >> 6), pooled column ((t >> 2) & 15), channels 4(t & 3)..+3
        const int pr = t >> 6, pc = (t >> 2) & 15, c4 = t & 3;
        const float* q00 = xb + ((2 * pr) * 32 + 2 * pc) * 16 + 4 * c4;
        float4 r;
        uint32_t am = 0;
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const float x00 = q00[cc], x01 = q00[16 + cc], x10 = q00[32 * 16 + cc], x11 = q00[33 * 16 + cc];
          float bv = x00;
          uint32_t bi = 0;
          if (x01 > bv) { bv = x01; bi = 1; }
          if (x10 > bv) { bv = x10; bi = 2; }
          if (x11 > bv) { bv = x11; bi = 3; }
          reinterpret_cast<float*>(&r)[cc] = bv > 0.f ? bv : 0.f;
          am |= bi << (8 * cc);
        }
        const int64_t o = (((int64_t)s * 16 + 8 * half + 2 * j + pr) * 16 + pc) * C1 + n0 + 4 * c4;
        *reinterpret_cast<float4*>(p.p1 + o) = r;
        *reinterpret_cast<uint32_t*>(p.am1 + o) = am;
        asm volatile("bar.sync 1, 128;" ::: "memory");  // buffer reused by the next chunk
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<128>(tbase);
}

// ------------------------------------------------------------------ weight gradient
// K-block = one image row h0 (32 pixels) of one sample.  A (M = taps x channels, K = px) is
// K-major SW128: row (kw, c, kh) = 32 consecutive pixels of input channel c, row h0+kh-2,
// shifted by kw-2 — one TMA box {32 w, 5 h, 4 c} of the planar (c, h, w) input per kw lands
// as 20 such rows.  Each kw block is padded to 24 rows (3 SW128 atoms); rows 120-127 hold a
// constant ones row (bias) and zeros.  B = dY1 row (32 px x 32 ch), MN-major BASE32B.
constexpr int D_KWB = 24 * 128;          // 3072 B per kw block (20 rows + 4 zero rows)
constexpr int D_A = 128 * 128;           // 16384: 5 kw blocks + constant rows 120..127
constexpr int D_B = 32 * 128;            // 4096
constexpr int D_STAGE = D_A + D_B;       // 20480
constexpr int D_NST = 4;
constexpr int D_BAR = D_NST * D_STAGE;
constexpr int D_SMEM = D_BAR + 128 + 1024;
constexpr int D_TX = 5 * 20 * 128 + D_B; // bytes TMA writes per stage
constexpr int NPART = 25 * 4 + 1;        // partial row length per output channel (k_dw_reduce_sgd layout)

struct C1DwArgs {
  const int32_t* sidx;
  const int32_t* bs;
  int B, nch, rpc;
  float* part;  // [A*nch][32][101]
};

__global__ void __launch_bounds__(192, 1)
    k_conv1_dw_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapD, C1DwArgs p) {
  constexpr uint32_t IDESC = tc::idesc_tf32(128, C1, 0, 1);  // A K-major, B MN-major
  const int ch = blockIdx.x, a = blockIdx.y, z = a * p.nch + ch;
  const int r0 = ch * p.rpc, r1 = min(p.bs[a], r0 + p.rpc);
  if (r0 >= r1) return;
  const int nkb = (r1 - r0) * H;
  // PDL: wait for the previous kernel before taking TMEM (a parked CTA holding columns
  // would stall other streams' kernels) or touching anything it writes.
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + D_BAR);
  uint64_t* empty = full + D_NST;
  uint64_t* tfull = empty + D_NST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
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
      for (int i = 0; i < D_NST; ++i) {
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
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % D_NST, ph = (kb / D_NST) & 1;
        const int rr = r0 + kb / H, h0 = kb % H;
        const int row = p.sidx[a * p.B + rr];
        tc::mbar_wait(empty + st, ph ^ 1);
        uint8_t* sa = smem + st * D_STAGE;
        tc::mbar_expect_tx(full + st, D_TX);
        // tap column kw = shifted copy (kw & 3) read from w' = (kw & 4): x[w + kw - 2]
        for (int kw = 0; kw < 5; ++kw)
          tc::tma_load_5d(sa + kw * D_KWB, &mapX, full + st, kw & 4, h0 - 2, 0, kw & 3, row);
        tc::tma_load_4d(sa + D_A, &mapD, full + st, 0, 0, h0, a * p.B + rr);
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int st = kb % D_NST, ph = (kb / D_NST) & 1;
        tc::mbar_wait(full + st, ph);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(smem + st * D_STAGE), sb = sa + D_A;
#pragma unroll
        for (int k = 0; k < 4; ++k) {  // 8 pixels per MMA
          const uint64_t ad = tc::sdesc(sa + k * 32, 0, 1024, tc::kSW128);
          const uint64_t bd = tc::sdesc(sb + k * 1024, 4096, 512, tc::kSW128_32B);
          tc::mma_tf32(tbase, ad, bd, IDESC, (kb | k) != 0);
        }
        tc::mma_commit(empty + st);
      }
      tc::mma_commit(tfull);
    }
  } else {
    const int qd = warp & 3, m = qd * 32 + lane;  // row = kw*24 + c*5 + kh; 120 = bias
    tc::mbar_wait(tfull, 0);
    tc::tc_fence_after();
    int n = -1;
    if (m < 120 && (m % 24) < 20) {
      const int kw = m / 24, c = (m % 24) / 5, kh = (m % 24) % 5;
      n = (kh * 5 + kw) * 4 + c;
    } else if (m == 120) {
      n = 100;
    }
    float* out = p.part + (int64_t)z * C1 * NPART;
#pragma unroll
    for (int n0 = 0; n0 < C1; n0 += 16) {
      float v[16];
      tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + n0, v);
      if (n >= 0)
#pragma unroll
        for (int j = 0; j < 16; ++j) out[(n0 + j) * NPART + n] = v[j];
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<32>(tbase);
}

}  // namespace

// conv1 forward (+ bias) on tensor cores: packed input rows -> a1 (pre-activation).
int conv1_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wclients, const float* xpack,
                 int64_t xrows, float* p1, uint8_t* am1, cudaStream_t st) {
  CUtensorMap mx, mw;
  uint64_t dx[4] = {4, W, H, (uint64_t)xrows};
  uint64_t sx[3] = {16, 16 * W, 16 * W * H};
  uint32_t bx[4] = {4, W, F_ROWS, 1};
  uint64_t dw[4] = {4, 25, 32, (uint64_t)wclients};  // c1w[o][tap][4] of every client slot
  uint64_t sw[3] = {16, 400, (uint64_t)L.P_pad * 4};
  uint32_t bw[4] = {4, 1, 32, 1};
  if (!tmap_encode(&mx, xpack, 4, dx, sx, bx, 0) || !tmap_encode(&mw, wbase + L.o_c1w, 4, dw, sw, bw, 0)) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv1_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
    attr = true;
  }
  C1Args p{wa.sidx, wa.bs, wa.B, wa.first ? 0 : 1, wbase + L.o_c1b, L.P_pad, p1, am1};
  launch_pdl(wa.pdl, k_conv1_fwd_tc, dim3(2 * wa.B, wa.A), 192, F_SMEM, st, mx, mw, p);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

// conv1 weight gradient on tensor cores: partials [A*nch][32][101] for k_dw_reduce_sgd.
int conv1_dw_tc(const Layout& L, const WaveArgs& wa, const float* xplanar, int64_t xrows, const float* dY1,
                int64_t slots, float* part, int64_t part_cap, int* nch_out, int* rpc_out, cudaStream_t st) {
  CUtensorMap mx, md;
  constexpr int WP = W + 4;  // shifted planar copies [r][s][c][h][W+4]
  uint64_t dx[5] = {WP, H, 4, 4, (uint64_t)xrows};
  uint64_t sx[4] = {4 * WP, 4 * WP * H, 4 * WP * H * 4, 4 * WP * H * 16};
  uint32_t bx[5] = {W, 5, 4, 1, 1};
  uint64_t dd[4] = {32, W, H, (uint64_t)slots};
  uint64_t sd[3] = {128, 128 * W, 128 * W * H};
  uint32_t bd[4] = {32, W, 1, 1};
  if (!tmap_encode(&mx, xplanar, 5, dx, sx, bx, 1) || !tmap_encode(&md, dY1, 4, dd, sd, bd, 2)) return -1;
  int nch = (2 * 148 + wa.A - 1) / wa.A;
  nch = nch < 1 ? 1 : (nch > wa.B ? wa.B : nch);
  const int rpc = (wa.B + nch - 1) / nch;
  nch = (wa.B + rpc - 1) / rpc;
  if ((int64_t)wa.A * nch > part_cap) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv1_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, D_SMEM);
    attr = true;
  }
  C1DwArgs p{wa.sidx, wa.bs, wa.B, nch, rpc, part};
  launch_pdl(wa.pdl, k_conv1_dw_tc, dim3(nch, wa.A), 192, D_SMEM, st, mx, md, p);
  *nch_out = nch;
  *rpc_out = rpc;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

bool conv1_tc_supported(const Layout& L) {
  return L.model == 1 && L.d.H0 == H && L.d.W0 == W && L.d.cpad == 4 && L.d.C1 == C1;
}

}  // namespace flb
