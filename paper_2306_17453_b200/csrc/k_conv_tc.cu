// k_conv_tc.cu — 5x5 'same' convolutions of the CIFAR CNN's second layer on the 5th-gen
// tensor cores (tcgen05.mma kind::tf32, fp32 accumulators in TMEM, operands staged by TMA).
//
// Implicit GEMM without an im2col buffer.  One CTA tile is one 16-pixel-wide patch of PH_
// rows (16 or 8) of one sample's output plane (M = 16·PH_ pixels = one or two M=128
// accumulators) for all output channels N.  CIFAR's 16x16 plane is one 16x16 patch; the
// speech model's 20x49 plane is 3 x 4 patches of 8x16 (TMA zero-fills the copy outside the
// image, the epilogue stores only pixels inside it).  For each
// horizontal tap kw (and 32-channel input chunk q) TMA loads ONE shifted copy of the input
// plane, copy[h'][x][c] = X[h'-2][x+kw-2][32q+c] for h' in [0,20), x in [0,16), with the
// zero padding produced by TMA's out-of-bounds fill.  A pixel is a 128-byte SW128 row, so
// the A operand of tap (kh, kw) for M-half mh is that copy shifted by (8·mh + kh)·16 rows:
// a descriptor offset, no data movement.  Each input byte is fetched 5 times instead of 25.
//
//   conv2 forward: X = p1 (C = 32), B = W2[o][tap][c] K-major, N = 64; epilogue fuses
//                  bias + ReLU + 2x2 max-pool + argmax (reading A13) -> p2, am2.
//   conv2 dX:      X = dY2 (C = 64, 2 chunks), B[n=c][k=o] = W2[o][flip tap][c] MN-major,
//                  N = 32; epilogue stores dp1 (pre-unpool).
//
// Warp roles (192 threads): warp 0 TMA producer + TMEM owner, warp 1 MMA issuer, warps
// 2-5 epilogue (TMEM lane quarter = warp % 4).  PAPER.md P:176 (client SGD) — this is
// the dominant dense contraction of a client step.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <unordered_map>

#include "fl_internal.h"
#include "tc_common.cuh"

namespace flb {

// ------------------------------------------------------------------ host: tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

// swz: 0 none, 1 128B (16-B granules, K-major operands), 2 128B with 32-B atoms (32-bit
// MN-major operands: matches the SWIZZLE_128B_BASE32B descriptor layout, Swizzle<2,5,2>).
// Encoding a tensor map costs microseconds of host time and a round issues thousands of
// launches whose maps repeat (same buffers, extents and boxes every wave and every round), so
// encoded maps are memoised per host thread, keyed by every encode input.
namespace {
struct TmapKey {
  const void* base;
  int rank, swz;
  uint64_t dims[5], strides[4];
  uint32_t box[5];
  bool operator==(const TmapKey& o) const { return memcmp(this, &o, sizeof *this) == 0; }
};
struct TmapKeyHash {
  size_t operator()(const TmapKey& k) const {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(&k);
    uint64_t h = 1469598103934665603ull;
    for (size_t i = 0; i < sizeof k / 8; ++i) h = (h ^ w[i]) * 1099511628211ull;
    return (size_t)h;
  }
};
}  // namespace

static bool tmap_encode_uncached(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                                 const uint64_t* strides_b, const uint32_t* box, int swz);

bool tmap_encode(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_b,
                 const uint32_t* box, int swz) {
  static thread_local std::unordered_map<TmapKey, CUtensorMap, TmapKeyHash> cache;
  TmapKey k;
  memset(&k, 0, sizeof k);
  k.base = base;
  k.rank = rank;
  k.swz = swz;
  for (int i = 0; i < rank; ++i) k.dims[i] = dims[i], k.box[i] = box[i];
  for (int i = 0; i + 1 < rank; ++i) k.strides[i] = strides_b[i];
  auto it = cache.find(k);
  if (it != cache.end()) {
    *m = it->second;
    return true;
  }
  if (!tmap_encode_uncached(m, base, rank, dims, strides_b, box, swz)) return false;
  if (cache.size() > 4096) cache.clear();  // bounded: buffers are grow-only, so maps rarely churn
  cache.emplace(k, *m);
  return true;
}

static bool tmap_encode_uncached(CUtensorMap* m, const void* base, int rank, const uint64_t* dims,
                                 const uint64_t* strides_b, const uint32_t* box, int swz) {
  if (!g_encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
      return false;
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  }
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<void*>(base),
                        (const cuuint64_t*)dims, (const cuuint64_t*)strides_b, (const cuuint32_t*)box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swz == 1 ? CU_TENSOR_MAP_SWIZZLE_128B
                                 : (swz == 2 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_NONE),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    fprintf(stderr, "cuTensorMapEncodeTiled failed (%d)\n", (int)r);
    return false;
  }
  return true;
}

namespace {

constexpr int WW = 16;                   // patch width (pixels): one 128-B row per pixel, 16 per image row
constexpr int NSTAGE = 2;

template <int N, int NB, int PH_>  // N output channels; NB = rows of one tap's B tile (N, or 32 for
struct ConvSmem {                  // MN-major); PH_ = patch rows (16: two M-halves, 8: one)
  static constexpr int A_BYTES = (PH_ + 4) * WW * 128;  // one shifted copy: PH_ + 4 rows x 16 pixels
  static constexpr int B_TAP = NB * 128;
  static constexpr int B_BYTES = 5 * B_TAP;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = NSTAGE * STAGE;
  static constexpr int TOTAL = BAR_OFF + 128 + 1024;  // barriers + tmem slot + alignment slack
};

struct ConvTcArgs {
  const int32_t* bs;
  int A;                  // active clients (tiles = A·B (client, sample) pairs)
  int B;
  int wmul;               // 0: every client reads θ_g (first wave), 1: client slot
  int msplit;             // tiles per sample: 1 (both M-halves) or 2 (one M-half each, small waves)
  const float* bias;      // bias of client 0; client a at bias + a*bias_stride
  int64_t bias_stride;
  float* out;             // fwd: p2 [S][H/2][W/2][N]; dx: dp1m [S][H][W][N] (ReLU'-masked pooled gradient)
  uint8_t* am;            // fwd: argmax [S][H/2][W/2][N]
  const float* p1;        // dx: pooled conv1 output [S][H][W][N] (ReLU' of the window max)
  const uint8_t* am1;     // dx: pool1 argmax [S][H][W][N]
  int H, W;               // image plane of this layer (CIFAR 16x16, speech 20x49)
  int ph, pw;             // patches per sample along h (PH_ rows each) and w (16 columns each)
};

// N: output channels; CH: 32-channel chunks of the input; BMN: B operand MN-major;
// FLIP: transposed conv (dX); POOL: fused bias + ReLU + max-pool epilogue; PH_: patch rows.
template <int N, int CH, int BMN, int FLIP, int POOL, int PH_>
__global__ void __launch_bounds__(192, 1)
    k_conv5_tc(const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapW, ConvTcArgs p) {
  constexpr int NB = BMN ? 32 : N;
  using S = ConvSmem<N, NB, PH_>;
  constexpr int A_BYTES = S::A_BYTES;
  constexpr int NMH = PH_ / 8;  // M-halves (128-pixel accumulators) per patch
  const int NP = p.ph * p.pw;   // patches per sample
  // two accumulator buffers x two M-halves x N columns
  constexpr uint32_t TMEM_COLS = (4 * N <= 32) ? 32 : (4 * N <= 64 ? 64 : (4 * N <= 128 ? 128 : 256));
  constexpr uint32_t IDESC = tc::idesc_tf32(128, N, 0, BMN);
  constexpr int NKB = 5 * CH;

  // Persistent: CTA b handles tiles t = b, b + grid, ... of the A·B (client, sample) tiles
  // (samples past a client's |b| are skipped identically by every role).  The smem stage
  // ring runs across tiles and the TMEM accumulators are double-buffered, so the loads of
  // tile i+1 and the epilogue of tile i-1 overlap the MMAs of tile i.
  // With msplit = 2 (16-row patches only) a tile is one M-half (t & 1): small waves spread a
  // sample's MMAs and epilogue over two SMs (the loads are the same either way).
  // tile t -> (slot sl, patch pt, M-half split): t = ((sl · NP) + pt) · msplit + half
  const int T = p.A * p.B * NP * p.msplit;
  auto valid = [&](int t) {
    const int sl = t / (p.msplit * NP);
    return (sl % p.B) < p.bs[sl / p.B];
  };

  // PDL: wait for the previous kernel before taking TMEM (a parked CTA holding columns
  // would stall other streams' kernels) or touching anything it writes.
  pdl_wait();
  extern __shared__ uint8_t smem_raw[];
  // align by pointer arithmetic on the shared array (an integer round trip would turn every
  // epilogue access into a generic LD/ST instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + NSTAGE;
  uint64_t* afull = empty + NSTAGE;   // [2] accumulator buffer ready for the epilogue
  uint64_t* aempty = afull + 2;       // [2] accumulator buffer drained by the epilogue
  uint32_t* tslot = reinterpret_cast<uint32_t*>(aempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      tc::prefetch_tmap(&mapX);
      tc::prefetch_tmap(&mapW);
      for (int i = 0; i < NSTAGE; ++i) {
        tc::mbar_init(full + i, 1);
        tc::mbar_init(empty + i, 1);
      }
      for (int i = 0; i < 2; ++i) {
        tc::mbar_init(afull + i, 1);
        tc::mbar_init(aempty + i, 128);
      }
      tc::fence_mbar_init();
    }
    __syncwarp();
    tc::tmem_alloc<TMEM_COLS>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (tc::elect_one()) {
      int it = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        if (!valid(t)) continue;
        const int s = t / (p.msplit * NP), a = s / p.B;  // slot index s = a*B + r
        const int pt = (t / p.msplit) % NP, y0 = (pt / p.pw) * PH_, x0 = (pt % p.pw) * WW;
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int st = it % NSTAGE, ph = (it / NSTAGE) & 1;
          const int kw = kb / CH, q = kb % CH;
          tc::mbar_wait(empty + st, ph ^ 1);
          uint8_t* sa = smem + st * S::STAGE;
          uint8_t* sb = sa + A_BYTES;
          tc::mbar_expect_tx(full + st, S::STAGE);
          tc::tma_load_4d(sa, &mapX, full + st, 32 * q, x0 + kw - 2, y0 - 2, s);
          for (int kh = 0; kh < 5; ++kh) {
            const int tap = FLIP ? (4 - kh) * 5 + (4 - kw) : kh * 5 + kw;
            tc::tma_load_4d(sb + kh * S::B_TAP, &mapW, full + st, 0, tap, BMN ? 32 * q : 0, a * p.wmul);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (tc::elect_one()) {
      int it = 0, tc_ = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        if (!valid(t)) continue;
        const int mh0 = p.msplit == 2 ? (t & 1) : 0, mh1 = p.msplit == 2 ? mh0 + 1 : NMH;
        const int buf = tc_ & 1, aph = (tc_ >> 1) & 1;
        tc::mbar_wait(aempty + buf, aph ^ 1);  // epilogue finished reading this buffer
        tc::tc_fence_after();
        const uint32_t acc0 = tbase + buf * 2 * N;
        for (int kb = 0; kb < NKB; ++kb, ++it) {
          const int st = it % NSTAGE, ph = (it / NSTAGE) & 1;
          tc::mbar_wait(full + st, ph);
          tc::tc_fence_after();
          const uint32_t sa = tc::smem_u32(smem + st * S::STAGE);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int kh = 0; kh < 5; ++kh)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint64_t bd = BMN ? tc::sdesc(sb + kh * S::B_TAP + k * 1024, NB * 128, 512, tc::kSW128_32B)
                                      : tc::sdesc(sb + kh * S::B_TAP + k * 32, 0, 1024, tc::kSW128);
#pragma unroll
              for (int mh = 0; mh < NMH; ++mh) {
                if (mh < mh0 || mh >= mh1) continue;
                const uint64_t ad = tc::sdesc(sa + (mh * 8 + kh) * WW * 128 + k * 32, 0, 1024, tc::kSW128);
                tc::mma_tf32(acc0 + mh * N, ad, bd, IDESC, (kb | kh | k) != 0);
              }
            }
          tc::mma_commit(empty + st);  // stage free once these MMAs have read it
        }
        tc::mma_commit(afull + buf);   // accumulators of this tile complete
        ++tc_;
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> global
    const int qd = warp & 3;                 // TMEM lane quarter of this warp
    const int i = qd * 32 + lane;            // accumulator row = pixel within the M-half
    int tc_ = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
    if (!valid(t)) continue;
    const int s = t / (p.msplit * NP), a = s / p.B;
    const int pt = (t / p.msplit) % NP, y0 = (pt / p.pw) * PH_, x0 = (pt % p.pw) * WW;
    const int mh0 = p.msplit == 2 ? (t & 1) : 0, mh1 = p.msplit == 2 ? mh0 + 1 : NMH;
    const int buf = tc_ & 1, aph = (tc_ >> 1) & 1;
    ++tc_;
    tc::mbar_wait(afull + buf, aph);
    tc::tc_fence_after();
    const uint32_t tacc = tbase + buf * 2 * N;
    const float* bias = p.bias + (int64_t)a * p.bias_stride * p.wmul;
#pragma unroll
    for (int mh = 0; mh < NMH; ++mh) {
      if (mh < mh0 || mh >= mh1) continue;
      const int h = y0 + mh * 8 + (i >> 4), w = x0 + (i & 15);  // image pixel of this accumulator row
#pragma unroll
      for (int n0 = 0; n0 < N; n0 += 16) {
        float v[16];
        tc::tmem_ld16(tacc + ((uint32_t)(qd * 32) << 16) + mh * N + n0, v);
        if (POOL) {
          // window (2i..2i+1, 2j..2j+1) = lanes l, l^1, l^16, l^17 of this warp
          float pv[16];
          uint8_t pa[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const float x00 = v[j] + bias[n0 + j];
            const float x01 = __shfl_xor_sync(0xffffffffu, x00, 1);
            const float x10 = __shfl_xor_sync(0xffffffffu, x00, 16);
            const float x11 = __shfl_xor_sync(0xffffffffu, x00, 17);
            float bv = x00;
            int bi = 0;
            if (x01 > bv) { bv = x01; bi = 1; }
            if (x10 > bv) { bv = x10; bi = 2; }
            if (x11 > bv) { bv = x11; bi = 3; }
            pv[j] = bv > 0.f ? bv : 0.f;
            pa[j] = (uint8_t)bi;
          }
          // floor pooling: only windows inside the image (the patch may overhang it)
          const int H2 = p.H >> 1, W2 = p.W >> 1;
          if ((lane & 17) == 0 && (h >> 1) < H2 && (w >> 1) < W2) {
            const int64_t o = (((int64_t)s * H2 + (h >> 1)) * W2 + (w >> 1)) * N + n0;
            float4* dst = reinterpret_cast<float4*>(p.out + o);
#pragma unroll
            for (int j = 0; j < 4; ++j) dst[j] = make_float4(pv[4 * j], pv[4 * j + 1], pv[4 * j + 2], pv[4 * j + 3]);
            uint32_t packed[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
              packed[j] = pa[4 * j] | (pa[4 * j + 1] << 8) | (pa[4 * j + 2] << 16) | ((uint32_t)pa[4 * j + 3] << 24);
            *reinterpret_cast<uint4*>(p.am + o) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
          }
        } else {
          // ReLU' of pool1 fused: dp1m = dp1 where the pooled value is > 0, else 0.  The
          // routing to the window's argmax (pool1 backward) happens where dY1 is consumed
          // (conv1's dW expands it into its B operand), so dY1 is never written to HBM.
          const int64_t o = (((int64_t)s * p.H + h) * p.W + w) * N + n0;
          if (h < p.H && w < p.W) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float4 pv = *reinterpret_cast<const float4*>(p.p1 + o + 4 * j);
              *reinterpret_cast<float4*>(p.out + o + 4 * j) =
                  make_float4(pv.x > 0.f ? v[4 * j] : 0.f, pv.y > 0.f ? v[4 * j + 1] : 0.f,
                              pv.z > 0.f ? v[4 * j + 2] : 0.f, pv.w > 0.f ? v[4 * j + 3] : 0.f);
            }
          }
        }
      }
    }
    tc::tc_fence_before();
    tc::mbar_arrive(aempty + buf);  // this thread's TMEM reads of the buffer are done
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  pdl_trigger();  // late trigger: a dependent kernel's CTAs park on SM resources until it runs
  if (warp == 0) tc::tmem_dealloc<TMEM_COLS>(tbase);
}

// One M-half per tile when the doubled tile count still fits on the wave's SMs.  Opt-in
// (FL_MSPLIT=1): it shortens a lone client's step (2000 samples: 7.2 -> 6.7 ms) but costs
// throughput when the critical-path streams share the GPU with the bulk (C2 16.6 -> 17.1 ms).
int msplit_for(const WaveArgs& wa) {
  static const bool on = [] {
    const char* e = getenv("FL_MSPLIT");
    return e && e[0] == '1';
  }();
  return (on && 2 * wa.sum_bs <= wa.sms) ? 2 : 1;
}

template <int N, int CH, int BMN, int FLIP, int POOL, int PH_>
cudaError_t launch_conv5(const CUtensorMap& mx, const CUtensorMap& mw, const ConvTcArgs& p, int A, bool pdl, int sms,
                         cudaStream_t st) {
  constexpr int NB = BMN ? 32 : N;
  const int smem = ConvSmem<N, NB, PH_>::TOTAL;
  auto kfn = k_conv5_tc<N, CH, BMN, FLIP, POOL, PH_>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int tiles = A * p.B * p.ph * p.pw * p.msplit;
  launch_pdl(pdl, kfn, dim3(tiles < sms ? tiles : sms), 192, smem, st, mx, mw, p);
  return cudaGetLastError();
}

// conv2 weights c2w[o][tap][c] of every client slot (or θ_g) as a 4-D tensor
// (c, tap, o, client) with a box of {32 c, 1 tap, nb o-rows, 1 client}.
bool make_w2_map(CUtensorMap* m, const Layout& L, const float* base, int64_t nclients, int nb, int swz) {
  const CnnDims& d = L.d;
  uint64_t dims[4] = {(uint64_t)d.C1, 25, (uint64_t)d.C2, (uint64_t)nclients};
  uint64_t str[3] = {(uint64_t)d.C1 * 4, (uint64_t)25 * d.C1 * 4, (uint64_t)L.P_pad * 4};
  uint32_t box[4] = {32, 1, (uint32_t)nb, 1};
  return tmap_encode(m, base + L.o_c2w, 4, dims, str, box, swz);
}

// NHWC activations [S][H][W][C] with a box of one (ph + 4)-row x 16-pixel x 32-channel copy.
bool make_plane_map(CUtensorMap* m, const float* base, int C, int H, int W, int ph, int64_t slots) {
  uint64_t dims[4] = {(uint64_t)C, (uint64_t)W, (uint64_t)H, (uint64_t)slots};
  uint64_t str[3] = {(uint64_t)C * 4, (uint64_t)C * 4 * W, (uint64_t)C * 4 * W * H};
  uint32_t box[4] = {32, WW, (uint32_t)ph + 4, 1};
  return tmap_encode(m, base, 4, dims, str, box, 1);
}

// patch rows: a single 16x16 patch covers CIFAR's plane; other planes use 8-row patches
// (less overhang: speech's 20 rows = 3 x 8 instead of 2 x 16)
int patch_rows(const CnnDims& d) { return (d.H1 == 16 && d.W1 == 16) ? 16 : 8; }

}  // namespace

bool conv_tc_supported(const Layout& L) {
  // conv2 of either CNN: 5x5 'same', 32 -> 64 channels, any plane at least 8 x 16
  return (L.model == FL_MODEL_CNN_CIFAR || L.model == FL_MODEL_CNN_SPEECH) && L.d.C1 == 32 && L.d.C2 == 64 &&
         L.d.H1 >= 8 && L.d.W1 >= 16;
}

// conv2 forward + bias + ReLU + pool on tensor cores: p1 -> p2, am2.
int conv2_fwd_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wclients, const float* p1,
                 int64_t slots, float* p2, uint8_t* am2, cudaStream_t st) {
  const CnnDims& d = L.d;
  const int ph = patch_rows(d);
  CUtensorMap mx, mw;
  if (!make_plane_map(&mx, p1, 32, d.H1, d.W1, ph, slots) || !make_w2_map(&mw, L, wbase, wclients, 64, 1)) return -1;
  ConvTcArgs p{wa.bs, wa.A, wa.B, wa.first ? 0 : 1, ph == 16 ? msplit_for(wa) : 1, wbase + L.o_c2b, L.P_pad, p2, am2,
               nullptr, nullptr, d.H1, d.W1, (d.H1 + ph - 1) / ph, (d.W1 + WW - 1) / WW};
  const cudaError_t e = ph == 16 ? launch_conv5<64, 1, 0, 0, 1, 16>(mx, mw, p, wa.A, wa.pdl, wa.sms, st)
                                 : launch_conv5<64, 1, 0, 0, 1, 8>(mx, mw, p, wa.A, wa.pdl, wa.sms, st);
  return e == cudaSuccess ? 1 : -1;
}

// conv2 dX (transposed conv) on tensor cores: dY2 -> dp1.
int conv2_dx_tc(const Layout& L, const WaveArgs& wa, const float* wbase, int64_t wclients, const float* dY2,
                int64_t slots, const float* p1, float* dp1m, cudaStream_t st) {
  const CnnDims& d = L.d;
  const int ph = patch_rows(d);
  CUtensorMap mx, mw;
  if (!make_plane_map(&mx, dY2, 64, d.H1, d.W1, ph, slots) || !make_w2_map(&mw, L, wbase, wclients, 32, 2)) return -1;
  ConvTcArgs p{wa.bs, wa.A, wa.B, wa.first ? 0 : 1, ph == 16 ? msplit_for(wa) : 1, nullptr, 0, dp1m, nullptr, p1,
               nullptr, d.H1, d.W1, (d.H1 + ph - 1) / ph, (d.W1 + WW - 1) / WW};
  const cudaError_t e = ph == 16 ? launch_conv5<32, 2, 1, 1, 0, 16>(mx, mw, p, wa.A, wa.pdl, wa.sms, st)
                                 : launch_conv5<32, 2, 1, 1, 0, 8>(mx, mw, p, wa.A, wa.pdl, wa.sms, st);
  return e == cudaSuccess ? 1 : -1;
}

}  // namespace flb
