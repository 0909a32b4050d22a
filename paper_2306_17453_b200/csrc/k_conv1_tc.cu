// k_conv1_tc.cu — the CIFAR CNN's first 5x5 conv (3 -> 32 channels, "same" padding) on
// tcgen05 kind::tf32: forward (+ bias, ReLU, 2x2 max-pool, argmax) and weight gradient
// (the McMahan CNN of P:453).
//
// With 32 output channels and 3 input channels the natural implicit GEMM (M = pixels,
// N = 32, K = 75) starves the tensor core: every N = 32 MMA re-reads a 128-row A tile from
// shared memory, so the kernel is shared-memory bound (round 2 ncu: TC + LSU smem wavefronts
// ~96 % busy, tensor pipe 4 %).  Here four horizontally adjacent output pixels share one GEMM
// row instead ("shift in M"):
//
//   window input  xg[y'][j][u][c] = xpad[y'][4j + u][c]   (y' in [0,36), j in [0,8), u in [0,8),
//                                   c in [0,4): 2-pixel zero border, channel 3 zero; 128 B rows)
//   shifted taps  Ws[(o,s)][(dy,u,c)] = W[o][dy][u - s][c]  (0 unless 0 <= u - s < 5), s in [0,4)
//
//   forward   D[(o,s)][(y,j)] = Σ_{dy,u,c} Ws[(o,s)][(dy,u,c)] · xg[y + dy][j][u][c] = conv(x)[o][y][4j + s]
//   dW        G[(o,s)][(dy,u,c)] = Σ_{(y,j)} dY1[y][4j + s][o] · xg[y + dy][j][u][c]
//             dW[o][dy][dx][c] = Σ_s G[(o,s)][(dy, dx + s, c)]
//
// M = (o, s) = 128 rows lives in TMEM as the MMA's A operand (written with tcgen05.st), so the
// tensor core reads only B from shared memory: one TMA box of 20 window rows x 8 windows
// (20 KB) per half sample serves all 5 dy taps (the dy shift is +1 KB on the descriptor).
// Forward: A = Ws (K-major, 160 columns), B = xg K-major SW128, N = 128 (16 rows x 8 windows).
// dW:      A = dY1 expanded from dp1m + pool1's argmax (K = 128 pixels of a half sample),
//          B = xg MN-major (SWIZZLE_128B_BASE32B; N = 160 = 5 dy chunks of 32, LBO = 1 KB).
#include <cuda.h>

#include <algorithm>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fl_internal.h"
#include "tc_common.cuh"

namespace flb {
namespace {

constexpr int H = 32, W = 32, C1 = 32;
constexpr int XG_Y = H + 4;                  // padded rows
constexpr int XG_J = W / 4;                  // 8 windows of 8 pixels per row (stride 4)
constexpr int XG_FLOATS = XG_Y * XG_J * 32;  // 9216 floats per sample
constexpr int BT = 20 * XG_J * 128;          // B tile: 20 window rows (16 outputs + 4 halo) = 20 KB
constexpr int NPART = 25 * 4 + 1;            // dW partial row per output channel (k_dw_reduce*_sgd layout)

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

// Both kernels split the wave's U = 2·Σ|b| half-sample tiles (concatenated over clients in
// order) evenly over G CTAs: CTA c takes [c·U/G, (c+1)·U/G), so it sees few client changes.
// The client's sample range [base, next) stays in registers: no global load per tile.
struct TileWalk {
  const int32_t* bpre;
  int A;
  int a;
  int32_t base, next;
  __device__ TileWalk(const int32_t* b, int A_, int64_t u0) : bpre(b), A(A_), a(client_of(b, A_, u0 >> 1)) {
    base = bpre[a];
    next = bpre[a + 1];
  }
  __device__ int client(int64_t u) {
    while (a + 1 < A && (u >> 1) >= next) {
      ++a;
      base = next;
      next = bpre[a + 1];
    }
    return a;
  }
  __device__ int sample(int64_t u) const { return (int)((u >> 1) - base); }  // index within the client
  __device__ bool last_of_client(int64_t u) const { return ((u + 1) >> 1) >= next; }
};

// ------------------------------------------------------------------ forward
constexpr int F_NST = 6;
constexpr int F_BAR = F_NST * BT;
constexpr int F_SMEM = F_BAR + 256 + 1024;  // > 1/2 of the SM's shared memory: one CTA per SM (TMEM 512)
constexpr uint32_t F_TA = 0, F_TD = 256;    // TMEM columns: Ws [0,160); D double buffer [256,384) [384,512)
constexpr int F_THREADS = 64 + 512;   // producer, MMA, 16 epilogue warps
constexpr int F_EPI = 512;

struct C1Args {
  const int32_t* sidx;
  const int32_t* bpre;
  int A, B, G;
  int64_t U;
  const float* w;      // conv1 weights [32 o][25 taps][4 c] of client 0; client a at + a*wstride
  const float* bias;   // conv1 bias of client 0; client a at + a*wstride
  int64_t wstride;
  float* p1;           // [S][16][16][32] pooled ReLU output
  uint8_t* am1;        // [S][16][16][32] window argmax (row-major window index, first maximum)
};

__global__ void __launch_bounds__(F_THREADS, 1)
    k_conv1_fwd_tc(const __grid_constant__ CUtensorMap mapX, C1Args p) {
  constexpr uint32_t IDESC = tc::idesc_tf32(128, 128, 0, 0);
  const int64_t u0 = (int64_t)blockIdx.x * p.U / p.G, u1 = (int64_t)(blockIdx.x + 1) * p.U / p.G;
  // PDL: wait for the previous kernel before taking TMEM (a parked CTA holding columns
  // would stall other streams' kernels) or touching anything it writes.
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + F_BAR);
  uint64_t* empty = full + F_NST;
  uint64_t* dfull = empty + F_NST;   // [2]
  uint64_t* dempty = dfull + 2;      // [2]
  uint64_t* aready = dempty + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(aready + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapX);
      for (int i = 0; i < F_NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
      }
      for (int i = 0; i < 2; ++i) {
        tc::mbar_init(dfull + i, 1);
        tc::mbar_init(dempty + i, F_EPI);
      }
      tc::mbar_init(aready, F_EPI);
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
    // ---------------- producer: one 20-row window box per half-sample tile
    if (tc::elect_one()) {
      TileWalk tw(p.bpre, p.A, u0);
      int it = 0;
      for (int64_t u = u0; u < u1; ++u, ++it) {
        const int a = tw.client(u);
        const int s = a * p.B + tw.sample(u), h = (int)(u & 1);
        const int st = it % F_NST, ph = (it / F_NST) & 1;
        tc::mbar_wait(empty + st, ph ^ 1);
        tc::mbar_expect_tx(full + st, BT);
        tc::tma_load_4d(smem + st * BT, &mapX, full + st, 0, 0, 16 * h, p.sidx[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (tc::elect_one()) {
      TileWalk tw(p.bpre, p.A, u0);
      int it = 0, cur = -1, aph = 0;
      for (int64_t u = u0; u < u1; ++u, ++it) {
        const int a = tw.client(u);
        if (a != cur) {  // the epilogue warps rebuilt Ws for this client
          tc::mbar_wait(aready, aph);
          aph ^= 1;
          cur = a;
        }
        const int st = it % F_NST, ph = (it / F_NST) & 1, buf = it & 1, dph = (it >> 1) & 1;
        tc::mbar_wait(dempty + buf, dph ^ 1);
        tc::mbar_wait(full + st, ph);
        tc::tc_fence_after();
        const uint32_t sb = tc::smem_u32(smem + st * BT), td = tbase + F_TD + buf * 128;
#pragma unroll
        for (int dy = 0; dy < 5; ++dy)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // 8 of the 32 (u, c) per MMA
            tc::mma_tf32_ts(td, tbase + F_TA + dy * 32 + kk * 8, tc::sdesc(sb + dy * 1024 + kk * 32, 0, 1024, tc::kSW128),
                            IDESC, (dy | kk) != 0);
        tc::mma_commit(empty + st);
        tc::mma_commit(dfull + buf);
      }
    }
  } else {
    // ---------------- epilogue (16 warps, four per TMEM lane quarter): row m = (o, s) = 4o + s;
    // warp part qp owns image rows [4qp, 4qp + 4) of the tile.  Also (re)builds Ws in TMEM at
    // each client change.
    const int q = warp & 3, qp = (warp - 2) >> 2, m = q * 32 + lane, o = m >> 2, s4 = m & 3;
    const uint32_t lrow = (uint32_t)(q * 32) << 16;
    const bool odd = (s4 & 1) != 0;
    TileWalk tw(p.bpre, p.A, u0);
    int it = 0, cur = -1;
    float bo = 0.f;
    for (int64_t u = u0; u < u1; ++u, ++it) {
      const int a = tw.client(u);
      if (a != cur) {
        // Every MMA that read the previous Ws has completed: this thread already waited on the
        // previous tile's dfull, which tcgen05.commit signals after all earlier MMAs.
        const float* wa = p.w + (int64_t)a * p.wstride + o * 100;
#pragma unroll
        for (int i = 0; i < 5; ++i) {  // columns [40 qp + 8 i, +8): (dy, u, c) = k / 32, (k / 4) % 8, k % 4
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int k = 40 * qp + 8 * i + e, dy = k >> 5, uu = (k >> 2) & 7, c = k & 3, dx = uu - s4;
            v[e] = (dx >= 0 && dx < 5) ? __ldg(wa + (dy * 5 + dx) * 4 + c) : 0.f;
          }
          tc::tmem_st8(tbase + lrow + F_TA + 40 * qp + 8 * i, v);
        }
        tc::tmem_wait_st();
        bo = __ldg(p.bias + (int64_t)a * p.wstride + o);
        tc::tc_fence_before();
        tc::mbar_arrive(aready);
        cur = a;
      }
      const int s = a * p.B + tw.sample(u), h = (int)(u & 1);
      const int buf = it & 1, dph = (it >> 1) & 1;
      tc::mbar_wait(dfull + buf, dph);
      tc::tc_fence_after();
      float vv[32];  // both 16-column chunks of this warp's part in one TMEM load
      tc::tmem_ld32(tbase + lrow + F_TD + buf * 128 + qp * 32, vv);
      tc::tc_fence_before();
      tc::mbar_arrive(dempty + buf);  // accumulator drained: the next tile's MMAs may start
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {  // 16 columns = image rows 2·py, 2·py + 1 x 8 windows
        const float* v = vv + 16 * cc;
        const int py = 8 * h + 2 * qp + cc;
        float* prow = p.p1 + (((int64_t)s * 16 + py) * 16) * C1 + o;
        uint8_t* arow = p.am1 + (((int64_t)s * 16 + py) * 16) * C1 + o;
        // The pool window of windows-column j spans pixels 4j + s, 4j + (s ^ 1) (lanes s, s^1) in
        // rows 2py, 2py + 1.  The lane pair splits the 8 windows: the even lane pools j = k, the
        // odd lane j = k + 4, each receiving the partner's two values of its window.  The bias is
        // common to the window, so it is added to the maximum only.
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float mt = odd ? v[k + 4] : v[k], mb = odd ? v[12 + k] : v[8 + k];
          const float st = odd ? v[k] : v[k + 4], sb = odd ? v[8 + k] : v[12 + k];
          const float pt = __shfl_xor_sync(0xffffffffu, st, 1), pb = __shfl_xor_sync(0xffffffffu, sb, 1);
          // row-major window order: (top, even px), (top, odd px), (bottom, even), (bottom, odd)
          const float a0 = odd ? pt : mt, a1 = odd ? mt : pt, a2 = odd ? pb : mb, a3 = odd ? mb : pb;
          const float mx = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
          const uint32_t bi = a0 == mx ? 0u : (a1 == mx ? 1u : (a2 == mx ? 2u : 3u));
          const float r = mx + bo;
          const int px = 2 * (k + (odd ? 4 : 0)) + (s4 >> 1);
          prow[px * C1] = r > 0.f ? r : 0.f;
          arow[px * C1] = (uint8_t)bi;
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

// ------------------------------------------------------------------ weight gradient
constexpr int D_DP = 8 * 16 * C1 * 4;      // pooled gradient dp1m of a half sample [8 py][16 px][32 o]
constexpr int D_AM = 8 * 16 * C1;          // its pool1 argmax bytes
constexpr int D_STAGE = BT + D_DP + D_AM;  // 40 KB
constexpr int D_NST = 4;
constexpr int D_SCR = D_NST * D_STAGE;     // epilogue scratch [128][33] floats + bias [2][32]
constexpr int D_BAR = D_SCR + 128 * 33 * 4 + 8 * 32 * 4;
constexpr int D_SMEM = D_BAR + 256 + 1024;
constexpr uint32_t D_TA = 0, D_TG = 256;   // TMEM columns: dY1 double buffer [0,128) [128,256); G [256,416)
constexpr int D_THREADS = 64 + 256;

struct C1DwArgs {
  const int32_t* sidx;
  const int32_t* bpre;
  int A, B, G;
  int64_t U;
  float* part;  // [A + G][32][101]: partial of (CTA c, client a) at z = a + c
};

__global__ void __launch_bounds__(D_THREADS, 1)
    k_conv1_dw_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapD,
                  const __grid_constant__ CUtensorMap mapA, C1DwArgs p) {
  constexpr uint32_t IDESC = tc::idesc_tf32(128, 160, 0, 1);  // A (TMEM) K-major, B MN-major
  const int c = blockIdx.x;
  const int64_t u0 = (int64_t)c * p.U / p.G, u1 = (int64_t)(c + 1) * p.U / p.G;
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + D_BAR);
  uint64_t* empty = full + D_NST;
  uint64_t* abuilt = empty + D_NST;  // [2]
  uint64_t* aempty = abuilt + 2;     // [2]
  uint64_t* gfull = aempty + 2;
  uint64_t* gempty = gfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(gempty + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapX);
      tc::prefetch_tmap(&mapD);
      tc::prefetch_tmap(&mapA);
      for (int i = 0; i < D_NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
      }
      for (int i = 0; i < 2; ++i) {
        tc::mbar_init(abuilt + i, 256);
        tc::mbar_init(aempty + i, 1);
      }
      tc::mbar_init(gfull, 1);
      tc::mbar_init(gempty, 256);
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
      TileWalk tw(p.bpre, p.A, u0);
      int it = 0;
      for (int64_t u = u0; u < u1; ++u, ++it) {
        const int a = tw.client(u);
        const int s = a * p.B + tw.sample(u), h = (int)(u & 1);
        const int st = it % D_NST, ph = (it / D_NST) & 1;
        tc::mbar_wait(empty + st, ph ^ 1);
        uint8_t* sa = smem + st * D_STAGE;
        tc::mbar_expect_tx(full + st, D_STAGE);
        tc::tma_load_4d(sa, &mapX, full + st, 0, 0, 16 * h, p.sidx[s]);  // 20 window rows (ATOM_32B)
        tc::tma_load_4d(sa + BT, &mapD, full + st, 0, 0, 8 * h, s);          // dp1m rows 8h..8h+7
        tc::tma_load_4d(sa + BT + D_DP, &mapA, full + st, 0, 0, 8 * h, s);   // am1 rows
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      TileWalk tw(p.bpre, p.A, u0);
      int it = 0, gph = 0, prev = -1;
      for (int64_t u = u0; u < u1; ++u, ++it) {
        const int a = tw.client(u);
        const bool seg0 = a != prev;  // first tile of this client's segment in the CTA
        prev = a;
        const bool seg1 = (u + 1 == u1) || tw.last_of_client(u);
        const int st = it % D_NST, ph = (it / D_NST) & 1, ab = it & 1, aph = (it >> 1) & 1;
        tc::mbar_wait(full + st, ph);
        tc::mbar_wait(abuilt + ab, aph);
        if (seg0) tc::mbar_wait(gempty, gph ^ 1);  // G drained by the previous segment's epilogue
        tc::tc_fence_after();
        const uint32_t sb = tc::smem_u32(smem + st * D_STAGE);
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)  // K step = one image row (8 windows); N chunk dy = +1 KB
          tc::mma_tf32_ts(tbase + D_TG, tbase + D_TA + ab * 128 + kk * 8, tc::sdesc(sb + kk * 1024, 1024, 512, tc::kSW128_32B),
                          IDESC, (seg0 && kk == 0) ? 0u : 1u);
        tc::mma_commit(empty + st);
        tc::mma_commit(aempty + ab);
        if (seg1) {
          tc::mma_commit(gfull);
          gph ^= 1;
        }
      }
    }
  } else {
    // ---------------- dY1 builders / epilogue: row m = (s, o) = 32s + o (lane quarter = s, so a
    // warp's dp1m / argmax reads are 32 consecutive channels), half hf of the image rows
    const int q = warp & 3, hf = (warp - 2) >> 2, m = q * 32 + lane, o = lane, s4 = q;
    const uint32_t lrow = (uint32_t)(q * 32) << 16;
    float* scr = reinterpret_cast<float*>(smem + D_SCR);
    float* bscr = scr + 128 * 33;
    const int tid = threadIdx.x - 64;
    TileWalk tw(p.bpre, p.A, u0);
    int it = 0, gph = 0;
    float gsum = 0.f;  // bias gradient share of this row and half
    for (int64_t u = u0; u < u1; ++u, ++it) {
      const int a = tw.client(u);
      const bool seg1 = (u + 1 == u1) || tw.last_of_client(u);
      const int st = it % D_NST, ph = (it / D_NST) & 1, ab = it & 1, aph = (it >> 1) & 1;
      tc::mbar_wait(full + st, ph);
      tc::mbar_wait(aempty + ab, aph ^ 1);  // the MMAs of two tiles ago released this dY1 buffer
      tc::tc_fence_after();
      // pool1 backward on chip: dY1[y][x][o] = dp1m[y/2][x/2][o] where the window argmax is
      // (y % 2, x % 2), else 0; column k = (y_local, j), x = 4j + s
      const float* dp = reinterpret_cast<const float*>(smem + st * D_STAGE + BT);
      const uint8_t* am = smem + st * D_STAGE + BT + D_DP;
#pragma unroll
      for (int ci = 0; ci < 4; ++ci) {
        const int pyl = 4 * hf + ci;  // pooled row (local): image rows 2·pyl, 2·pyl + 1
        float v[16];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int idx = (pyl * 16 + 2 * j + (s4 >> 1)) * C1 + o;
          const float g = dp[idx];
          const uint32_t code = am[idx];
          v[j] = code == (uint32_t)(s4 & 1) ? g : 0.f;
          v[8 + j] = code == (uint32_t)(2 | (s4 & 1)) ? g : 0.f;
          gsum += v[j] + v[8 + j];
        }
        tc::tmem_st16(tbase + lrow + D_TA + ab * 128 + hf * 64 + ci * 16, v);
      }
      tc::tmem_wait_st();
      tc::tc_fence_before();
      tc::mbar_arrive(abuilt + ab);
      if (!seg1) continue;
      // ---- segment end: dW[o][dy][dx][c] = Σ_s G[(o,s)][(dy, dx+s, c)] -> partial z = a + c
      tc::mbar_wait(gfull, gph);
      gph ^= 1;
      tc::tc_fence_after();
      float* out = p.part + (int64_t)(a + c) * C1 * NPART;
      for (int dy = 0; dy < 5; ++dy) {
        float v[16];
        tc::tmem_ld16(tbase + lrow + D_TG + dy * 32 + hf * 16, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) scr[m * 33 + hf * 16 + e] = v[e];
        asm volatile("bar.sync 1, 256;" ::: "memory");
        for (int e = tid; e < C1 * 20; e += 256) {
          const int oo = e / 20, r = e % 20, dx = r >> 2, cc = r & 3;
          float g = 0.f;
#pragma unroll
          for (int s = 0; s < 4; ++s) g += scr[(32 * s + oo) * 33 + (dx + s) * 4 + cc];
          out[oo * NPART + (dy * 5 + dx) * 4 + cc] = g;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
      tc::tc_fence_before();
      tc::mbar_arrive(gempty);
      bscr[(4 * hf + s4) * 32 + o] = gsum;
      gsum = 0.f;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tid < C1) {
        float g = 0.f;
        for (int i = 0; i < 8; ++i) g += bscr[i * 32 + tid];
        out[tid * NPART + 100] = g;
      }
      asm volatile("bar.sync 1, 256;" ::: "memory");
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

// Window layout of the packed input: xg[r][y'][j][u][c] = xpack[r][y' - 2][4j + u - 2][c]
// (zero outside the image; xpack holds 16-byte pixels with channel 3 zero).
__global__ void k_pack_xg(const float4* __restrict__ xpack, int64_t rows, float4* __restrict__ xg) {
  constexpr int per = XG_Y * XG_J * 8;  // float4 per row
  const int64_t tot = rows * per;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / per;
    const int rem = (int)(e - r * per), yp = rem >> 6, j = (rem >> 3) & 7, uu = rem & 7;
    const int y = yp - 2, x = 4 * j + uu - 2;
    xg[e] = (y >= 0 && y < H && x >= 0 && x < W) ? xpack[(r * H + y) * W + x] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

bool encode_xg(CUtensorMap* m, const float* xg, int64_t xrows, int swz) {
  uint64_t d[4] = {32, XG_J, XG_Y, (uint64_t)xrows};
  uint64_t s[3] = {128, 128 * XG_J, 4ull * XG_FLOATS};
  uint32_t b[4] = {32, XG_J, 20, 1};
  return tmap_encode(m, xg, 4, d, s, b, swz);
}

}  // namespace

int64_t conv1_xg_floats() { return XG_FLOATS; }

int pack_xg(const float* xpack, int64_t rows, float* xg, cudaStream_t st) {
  if (rows <= 0) return 0;
  const int64_t n = rows * XG_Y * XG_J * 8;
  k_pack_xg<<<(int)std::min<int64_t>((n + 255) / 256, 1 << 20), 256, 0, st>>>(reinterpret_cast<const float4*>(xpack), rows,
                                                                            reinterpret_cast<float4*>(xg));
  return 1;
}

// conv1 forward + bias + ReLU + 2x2 pool (+ argmax) on tensor cores: xg -> p1, am1.
int conv1_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wstride, const float* xg,
                 int64_t xrows, int64_t slots, float* p1, uint8_t* am1, cudaStream_t st) {
  CUtensorMap mx;
  if (!encode_xg(&mx, xg, xrows, 1)) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv1_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
    attr = true;
  }
  const int64_t U = 2 * wa.sum_bs;
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(wa.sms, U));
  C1Args p{wa.sidx, wa.bpre, wa.A, wa.B, G, U, wbase + L.o_c1w, wbase + L.o_c1b, wstride, p1, am1};
  launch_pdl(wa.pdl, k_conv1_fwd_tc, dim3(G), F_THREADS, F_SMEM, st, mx, p);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

// conv1 weight gradient on tensor cores: partials [A + G][32][101] for the dW reduction
// (balanced split over U = 2·Σ|b| half-sample tiles, kbps = 2).
int conv1_dw_tc(const Layout& L, const WaveArgs& wa, const float* xg, int64_t xrows, const float* dp1m,
                const uint8_t* am1, int64_t slots, float* part, int64_t part_cap, int* g_out, cudaStream_t st) {
  CUtensorMap mx, md, ma;
  // pooled rows of dp1m [S][16][16][32] fp32 and of am1 (u8, viewed as 8 x 4-byte words per pixel)
  uint64_t dd[4] = {32, W / 2, H / 2, (uint64_t)slots};
  uint64_t sd[3] = {128, 128 * (W / 2), 128 * (W / 2) * (H / 2)};
  uint32_t bd[4] = {32, W / 2, 8, 1};
  uint64_t da[4] = {8, W / 2, H / 2, (uint64_t)slots};
  uint64_t sa[3] = {32, 32 * (W / 2), 32 * (W / 2) * (H / 2)};
  uint32_t ba[4] = {8, W / 2, 8, 1};
  if (!encode_xg(&mx, xg, xrows, 2) || !tmap_encode(&md, dp1m, 4, dd, sd, bd, 0) || !tmap_encode(&ma, am1, 4, da, sa, ba, 0))
    return -1;
  const int64_t U = 2 * wa.sum_bs;
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(wa.sms, U));
  if ((int64_t)wa.A + G > part_cap) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_conv1_dw_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, D_SMEM);
    attr = true;
  }
  C1DwArgs p{wa.sidx, wa.bpre, wa.A, wa.B, G, U, part};
  launch_pdl(wa.pdl, k_conv1_dw_tc, dim3(G), D_THREADS, D_SMEM, st, mx, md, ma, p);
  *g_out = G;
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

bool conv1_tc_supported(const Layout& L) {
  return L.model == 1 && L.d.H0 == H && L.d.W0 == W && L.d.cpad == 4 && L.d.C1 == C1;
}

}  // namespace flb
