// k_lstm_tc.cu — the char-LSTM's batched per-client GEMMs on tcgen05 (kind::tf32, fp32
// accumulators in TMEM, operands staged by TMA), SURVEY §8 a6 / PAPER.md P:457.
//
// Off the recurrence, one SGD step of a client is five dense contractions (M = B·T = 320 rows
// (batch row r, time t), H = 256, G = 4H = 1024):
//   P1  layer-1 input projection  xp[r,t,n]   = Σ_k H0[r,t+1,k] W_ih1[n,k] + b_ih1[n] + b_hh1[n]
//   P2  layer-1 dX                dX[r,t,k]   = Σ_n dpre1[r,t,n] W_ih1[n,k]
//   W3  W_hh1 -= η Σ_{r,t} dpre1[r,t,n] H1[r,t,k]      (H1[t] = h_{t-1}, H[0] = 0)
//   W4  W_ih1 -= η Σ_{r,t} dpre1[r,t,n] H0[r,t+1,k]
//   W6  W_hh0 -= η Σ_{r,t} dpre0[r,t,n] H0[r,t,k]
// One CTA computes one 128 x 256 output tile of one client (grid = tiles x clients), K in
// blocks of 32 fp32 (one 128-byte row) through a 4-stage TMA ring; the 128 x 256 accumulator
// lives in 256 TMEM columns.
//   P-type (P1, P2): M = (r, t) rows, an M tile = 4 batch rows x 32 time steps (TMA box over
//     [slot][t][k], t past T zero-filled); A K-major; B = W_ih1 K-major (P1) or MN-major (P2).
//   W-type (W3, W4, W6): M = gate rows n (8 tiles of 128), N = k = 256, K = (r, t) in 12
//     blocks (4 r x 3 t-blocks); A = dpreᵀ and B = H both MN-major (SWIZZLE_128B_BASE32B);
//     the epilogue applies W <- W − η·D (θ_g read on the first wave: slot init fused).
// Warp roles (192 threads): warp 0 TMA producer + TMEM owner, warp 1 MMA issuer, warps 2-5
// epilogue (TMEM lane quarter = warp % 4, thread = accumulator row).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_util.cuh"
#include "fl_internal.h"
#include "tc_common.cuh"

namespace flb {
namespace {

constexpr int LT = 80, LH = 256, LG = 1024;
constexpr int NT = 256;                          // N tile
constexpr int A_BYTES = 128 * 128, B_BYTES = NT * 128, STAGE = A_BYTES + B_BYTES;  // 16 + 32 KB
constexpr int NST = 4;
constexpr int BAR_OFF = NST * STAGE;
constexpr int SMEM = BAR_OFF + 128 + 1024;

struct LgArgs {
  int B, wmul;          // slots per client; 0: weights from θ_g (first wave), 1: the client's slot
  int kblocks;          // K blocks of 32
  int mtiles, ntiles;   // tiles per client
  int toffA, toffB;     // time offset of the A / B activation operand (H0[t+1]: 1)
  float* out;           // P: [S][T][N] activations; W: slots (weights, + o_w)
  int64_t out_sa;       // P: per-client stride of out (B·T·N); W: P_pad
  int ldo;              // P: N of the output rows
  const float* bias0;   // P1: b_ih1 of client 0 (+ a·bias_sa)
  const float* bias1;   // P1: b_hh1
  int64_t bias_sa;
  const float* src;     // W: weights read (θ_g or slot) (+ a·src_sa)
  int64_t src_sa;
  float lr;
};

template <int PTYPE, int BMN>  // PTYPE 1: rows (r, t), A K-major; 0: W-type (A, B MN-major)
__global__ void __launch_bounds__(192, 1)
    k_lstm_gemm_tc(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, LgArgs p) {
  constexpr int AMN = PTYPE ? 0 : 1;
  constexpr uint32_t IDESC = tc::idesc_tf32(128, NT, AMN, BMN);
  const int a = blockIdx.y, mt = blockIdx.x / p.ntiles, nt = blockIdx.x % p.ntiles;
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
  uint64_t* empty = full + NST;
  uint64_t* accf = empty + NST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(accf + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapA);
      tc::prefetch_tmap(&mapB);
      for (int i = 0; i < NST; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
      }
      tc::mbar_init(accf, 1);
      tc::fence_mbar_init();
    }
    __syncwarp();
    tc::tmem_alloc<NT>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;
  const int slot0 = a * p.B;
  if (warp == 0) {
    if (tc::elect_one()) {
      for (int kb = 0; kb < p.kblocks; ++kb) {
        const int st = kb % NST, ph = (kb / NST) & 1;
        tc::mbar_wait(empty + st, ph ^ 1);
        uint8_t* sa = smem + st * STAGE;
        uint8_t* sb = sa + A_BYTES;
        tc::mbar_expect_tx(full + st, STAGE);
        if (PTYPE) {
          // A: rows (r, t) of [slot][t][K], box {32 k, 32 t, 4 r} at (k0, t0 + toff, slot0)
          tc::tma_load_3d(sa, &mapA, full + st, 32 * kb, 32 * mt + p.toffA, slot0);
          if (BMN)  // W_ih1 as (K = n, N = k): box {32 k, 32 n, 8 k-chunks}
            tc::tma_load_4d(sb, &mapB, full + st, 0, 32 * kb, 0, a * p.wmul);
          else      // W_ih1 rows n (K-major): box {32 k, 256 n}
            tc::tma_load_3d(sb, &mapB, full + st, 32 * kb, NT * nt, a * p.wmul);
        } else {
          const int r = kb / 3, t0 = 32 * (kb % 3);
          // A = dpreᵀ: box {32 n, 32 t, 4 n-chunks} at (0, t0, 4·mt, slot0 + r)
          tc::tma_load_4d(sa, &mapA, full + st, 0, t0, 4 * mt, slot0 + r);
          // B = H: box {32 k, 32 t, 8 k-chunks} at (0, t0 + toff, 0, slot0 + r)
          tc::tma_load_4d(sb, &mapB, full + st, 0, t0 + p.toffB, 0, slot0 + r);
        }
      }
    }
  } else if (warp == 1) {
    if (tc::elect_one()) {
      for (int kb = 0; kb < p.kblocks; ++kb) {
        const int st = kb % NST, ph = (kb / NST) & 1;
        tc::mbar_wait(full + st, ph);
        tc::tc_fence_after();
        const uint32_t sa = tc::smem_u32(smem + st * STAGE), sb = sa + A_BYTES;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = AMN ? tc::sdesc(sa + k * 1024, 4096, 512, tc::kSW128_32B)
                                  : tc::sdesc(sa + k * 32, 0, 1024, tc::kSW128);
          const uint64_t bd = BMN ? tc::sdesc(sb + k * 1024, 4096, 512, tc::kSW128_32B)
                                  : tc::sdesc(sb + k * 32, 0, 1024, tc::kSW128);
          tc::mma_tf32(tbase, ad, bd, IDESC, (kb | k) != 0);
        }
        tc::mma_commit(empty + st);
      }
      tc::mma_commit(accf);
    }
  } else {
    const int qd = warp & 3, i = qd * 32 + lane;  // accumulator row
    tc::mbar_wait(accf, 0);
    tc::tc_fence_after();
    if (PTYPE) {
      const int r = i >> 5, t = 32 * mt + (i & 31);
      const bool ok = t < LT;
      float* orow = p.out + (int64_t)a * p.out_sa + ((int64_t)r * LT + t) * p.ldo + NT * nt;
      const float* b0 = p.bias0 ? p.bias0 + (int64_t)a * p.bias_sa + NT * nt : nullptr;
      const float* b1 = p.bias1 ? p.bias1 + (int64_t)a * p.bias_sa + NT * nt : nullptr;
#pragma unroll 1
      for (int n0 = 0; n0 < NT; n0 += 16) {
        float v[16];
        tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + n0, v);  // warp-collective
        if (ok) {
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            if (b0) {
              o.x += b0[n0 + j], o.y += b0[n0 + j + 1], o.z += b0[n0 + j + 2], o.w += b0[n0 + j + 3];
              o.x += b1[n0 + j], o.y += b1[n0 + j + 1], o.z += b1[n0 + j + 2], o.w += b1[n0 + j + 3];
            }
            *reinterpret_cast<float4*>(orow + n0 + j) = o;
          }
        }
      }
    } else {
      const int n = 128 * mt + i;
      const float* srow = p.src + (int64_t)a * p.src_sa + (int64_t)n * LH;
      float* orow = p.out + (int64_t)a * p.out_sa + (int64_t)n * LH;
#pragma unroll 1
      for (int k0 = 0; k0 < NT; k0 += 16) {
        float v[16];
        tc::tmem_ld16(tbase + ((uint32_t)(qd * 32) << 16) + k0, v);
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const float4 w = *reinterpret_cast<const float4*>(srow + k0 + j);
          *reinterpret_cast<float4*>(orow + k0 + j) =
              make_float4(w.x - p.lr * v[j], w.y - p.lr * v[j + 1], w.z - p.lr * v[j + 2], w.w - p.lr * v[j + 3]);
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();
  if (warp == 0) tc::tmem_dealloc<NT>(tbase);
}

template <int PTYPE, int BMN>
int launch(const CUtensorMap& ma, const CUtensorMap& mb, const LgArgs& p, int A, bool pdl, cudaStream_t st) {
  auto k = k_lstm_gemm_tc<PTYPE, BMN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr = true;
  }
  launch_pdl(pdl, k, dim3(p.mtiles * p.ntiles, A), 192, SMEM, st, ma, mb, p);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

// [slot][T'][K] activations (K-major rows (r, t)): box {32 k, 32 t, B slots}
bool map_rows(CUtensorMap* m, const float* base, int K, int Tp, int64_t slots, int B) {
  uint64_t d[3] = {(uint64_t)K, (uint64_t)Tp, (uint64_t)slots};
  uint64_t s[2] = {(uint64_t)K * 4, (uint64_t)K * 4 * Tp};
  uint32_t b[3] = {32, 32, (uint32_t)B};
  return tmap_encode(m, base, 3, d, s, b, 1);
}
// [slot][T'][K] activations as MN-major (K = t rows, 32-wide chunks of the feature dim):
// box {32, 32 t, nch chunks, 1 slot}
bool map_mn(CUtensorMap* m, const float* base, int K, int Tp, int64_t slots, int nch) {
  uint64_t d[4] = {32, (uint64_t)Tp, (uint64_t)K / 32, (uint64_t)slots};
  uint64_t s[3] = {(uint64_t)K * 4, 128, (uint64_t)K * 4 * Tp};
  uint32_t b[4] = {32, 32, (uint32_t)nch, 1};
  return tmap_encode(m, base, 4, d, s, b, 2);
}

}  // namespace

bool lstm_tc_supported(int B) { return B == 4; }

int lstm_gemm_tc(int which, const LstmTcIn& in, cudaStream_t st) {
  CUtensorMap ma, mb;
  LgArgs p{};
  p.B = in.B;
  p.wmul = in.wmul;
  p.lr = in.lr;
  const int64_t S = in.slots;
  if (which == 1 || which == 2) {  // P1 / P2
    const bool p1 = which == 1;
    if (!map_rows(&ma, p1 ? in.H0 : in.dpre, p1 ? LH : LG, p1 ? LT + 1 : LT, S, in.B)) return -1;
    if (p1) {  // W_ih1 [n][k] K-major, box {32 k, 256 n, 1}
      uint64_t d[3] = {(uint64_t)LH, (uint64_t)LG, (uint64_t)in.wclients};
      uint64_t s[2] = {(uint64_t)LH * 4, (uint64_t)in.P_pad * 4};
      uint32_t b[3] = {32, NT, 1};
      if (!tmap_encode(&mb, in.wsrc + in.o_wih1, 3, d, s, b, 1)) return -1;
    } else {   // W_ih1 as (K = n, N = k) MN-major: {32 k_in, n, 8 k-chunks, client}
      uint64_t d[4] = {32, (uint64_t)LG, (uint64_t)LH / 32, (uint64_t)in.wclients};
      uint64_t s[3] = {(uint64_t)LH * 4, 128, (uint64_t)in.P_pad * 4};
      uint32_t b[4] = {32, 32, 8, 1};
      if (!tmap_encode(&mb, in.wsrc + in.o_wih1, 4, d, s, b, 2)) return -1;
    }
    p.kblocks = p1 ? LH / 32 : LG / 32;
    p.mtiles = (LT + 31) / 32;
    p.ntiles = p1 ? LG / NT : LH / NT;
    p.toffA = p1 ? 1 : 0;
    p.out = p1 ? in.xp : in.dX;
    p.ldo = p1 ? LG : LH;
    p.out_sa = (int64_t)in.B * LT * p.ldo;
    if (p1) {
      p.bias0 = in.wsrc + in.o_bih1;
      p.bias1 = in.wsrc + in.o_bhh1;
      p.bias_sa = in.wstride;
    }
    return p1 ? launch<1, 0>(ma, mb, p, in.A, in.pdl, st) : launch<1, 1>(ma, mb, p, in.A, in.pdl, st);
  }
  // W-type: 3 = W_hh1 (H1[t]), 4 = W_ih1 (H0[t+1]), 6 = W_hh0 (H0[t])
  const float* dpre = in.dpre;
  const float* H = which == 3 ? in.H1 : in.H0;
  if (!map_mn(&ma, dpre, LG, LT, S, 4) || !map_mn(&mb, H, LH, LT + 1, S, 8)) return -1;
  p.kblocks = in.B * ((LT + 31) / 32);
  p.mtiles = LG / 128;
  p.ntiles = 1;
  p.toffB = which == 4 ? 1 : 0;
  const int64_t ow = which == 3 ? in.o_whh1 : (which == 4 ? in.o_wih1 : in.o_whh0);
  p.out = in.slots_w + ow;
  p.out_sa = in.P_pad;
  p.src = in.wsrc + ow;
  p.src_sa = in.wstride;
  return launch<0, 1>(ma, mb, p, in.A, in.pdl, st);
}

}  // namespace flb
