// k_lstm.cu — local SGD of the LEAF char-LSTM (reading A10):
// embed 80 -> 8, LSTM 8 -> 256, LSTM 256 -> 256 over T = 80 characters, fc 256 -> 80 on h_T,
// softmax-CE (mean over |b|), BPTT, SGD (a7) — one wave = one step of every active client.
//
// The recurrences are the critical path (T dependent phases per layer, forward and
// backward), so they run as thread-block CLUSTERS of 16 CTAs per client (a non-portable
// cluster size; 87 KB of shared memory per CTA so two CTAs share an SM): each CTA keeps its
// 64-row slice of W_hh (the i, f, g, o rows of 16 hidden units, padded k-major so the
// forward and the transposed backward products are both bank-conflict free) resident in
// shared memory for all T steps, owns those 16 units' cell state, and exchanges h_t (forward)
// or the partial W_hhᵀ·dpre sums (backward, reduce-scatter) through distributed shared memory
// with st.async stores that complete on the receivers' mbarriers (no per-step cluster barrier).  Everything that is not on the recurrence — the
// input projections, dX of layer 2, every weight gradient (K = |b|·T) with the SGD step in its
// epilogue, the embedding and the fc head — is batched per client outside the time loop.
// Deterministic: every sum has a fixed order.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dev_util.cuh"
#include "fl_internal.h"
#include "tc_common.cuh"

namespace cg = cooperative_groups;

namespace flb {
namespace {

constexpr int LT = 80, LH = 256, LG = 1024, LE = 8, LV = 80;
constexpr int CL = 16;             // CTAs per client cluster (non-portable size: 2 CTAs fit per SM)
constexpr int UPC = LH / CL;       // 16 hidden units per CTA
constexpr int RPC = 4 * UPC;       // 64 gate rows per CTA
constexpr int WPF = LH + 4;       // fwd: row-major [RPC][LH] slice, pitch 260 (float4 rows, conflict-free)
constexpr int WPB = RPC + 4;      // bwd: k-major [LH][RPC] slice, pitch 68 (float4 over rows)
constexpr int REC_SMEM = (LH * WPB + 2 * 4 * LH + 4 * RPC + 2 * CL * 4 * UPC) * 4 + 64;  // + 2 mbarriers
constexpr uint32_t XCH_BYTES = CL * 4 * UPC * 4;  // bytes one CTA receives per step (8 sources x 4 rows x 32)

// Remote (DSMEM) store of one float into cluster CTA `rank`'s shared memory, completing
// on that CTA's mbarrier: the consumer waits on its own barrier instead of a cluster-wide
// barrier (whose release fence is a GPU-scope membar per step).
__device__ __forceinline__ uint32_t mapa_u32(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_f32(uint32_t raddr, float v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(__float_as_uint(v)), "r"(rbar)
               : "memory");
}
static_assert(RPC * WPF <= LH * WPB, "both slice layouts fit the same smem carve-out");

__device__ __forceinline__ float sigm(float v) { return 1.f / (1.f + __expf(-v)); }

// global gate row of local row rl of cluster rank c: gate rl/32 (i, f, g, o), unit 32c + rl%32
__device__ __forceinline__ int grow_of(int rl, int c) { return (rl / UPC) * LH + UPC * c + (rl % UPC); }

struct RecArgs {
  const float* wsrc;   // client a's parameters at wsrc + a*wstride (θ_g on the first wave: stride 0)
  int64_t wstride;
  int64_t o_whh;       // W_hh [LG][LH]
  int B;               // slots per client (batch)
  const float* xp;     // fwd: [S][T][LG] input projection + both biases
  float* G;            // [S][T][LG] post-activation gates (fwd writes, bwd reads)
  float* C;            // [S][T+1][LH] cell states, C[., 0] = 0
  float* H;            // [S][T+1][LH] hidden states, H[., 0] = 0
  const float* ext;    // bwd: external dL/dh — ext_mode 0: [S][LH] at t = T-1 only; 1: [S][T][LH]
  int ext_mode;
  float* dpre;         // bwd: [S][T][LG] gradient of the gate pre-activations
};

// Forward recurrence of one layer for one client: a cluster of CL = 16 CTAs, FT threads each.
constexpr int FT = 4 * RPC;  // thread (row, k-quarter)
constexpr int NOWN = 4 * UPC;  // cell-owner threads: (batch row, unit)
// Forward recurrence, register-resident variant: W_hh is constant over the T steps, so each
// thread keeps its 4-row x 16-column segment of the CTA's slice in registers for the whole
// sequence.  Thread (rg, ks) = (tid / 16, tid % 16) owns rows 4·rg .. 4·rg+3 and columns
// {4·ks + 64·j + u}; per step it reads 16 float4 of h_{t-1} (each feeds 4 rows, 16 FMAs) and
// the 16 partial (row, batch) sums of a row group are reduce-scattered over its 16 lanes
// with 15 shuffles (fixed butterfly order); lane ks then owns (row, batch) j = bitrev4(ks).
// Shared-memory traffic per step is a quarter of a shared-memory-resident W_hh's (which re-reads h for
// every row; round 1, removed).
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(FT, 2) k_lstm_fwd_reg(RecArgs p) {
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), a = blockIdx.x / CL, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* hb = sm + LH * WPB;       // [2][4][LH] h_{t-1} of the 4 batch rows (ping-pong)
  float* gs = hb + 2 * 4 * LH;     // [4][RPC] activated gates of this CTA's rows
  uint64_t* hbar = reinterpret_cast<uint64_t*>(sm + LH * WPB + 2 * 4 * LH + 4 * RPC + 2 * CL * 4 * UPC);  // [2]
  const int rg = tid >> 4, ks = tid & 15;
  float4 w[4][4];  // [row r][column block j]: W_hh[row 4rg+r][4ks + 64j .. +3]
  {
    const float* W = p.wsrc + (int64_t)a * p.wstride + p.o_whh;
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        w[r][j] = __ldg(reinterpret_cast<const float4*>(W + (int64_t)grow_of(4 * rg + r, c) * LH + 4 * ks + 64 * j));
  }
  for (int e = tid; e < 2 * 4 * LH; e += FT) hb[e] = 0.f;
  const int cb = tid / UPC, cu = tid % UPC, unit = UPC * c + cu;  // cell owned by threads < NOWN
  const int64_t cs = (int64_t)a * p.B + cb;
  float cst = 0.f;
  if (tid < NOWN) {
    p.C[cs * (LT + 1) * LH + unit] = 0.f;
    p.H[cs * (LT + 1) * LH + unit] = 0.f;
  }
  // the (row, batch) this lane owns after the reduce-scatter
  const int jo = ((ks & 1) << 3) | ((ks & 2) << 1) | ((ks & 4) >> 1) | ((ks & 8) >> 3);
  const int orow = 4 * rg + (jo >> 2), ob = jo & 3, gr = grow_of(orow, c);
  const int64_t s0 = (int64_t)a * p.B;
  const float* xr = p.xp + (s0 + ob) * LT * LG + gr;  // step t at xr + t*LG
  float xn = xr[0];
  if (tid == 0) {
    tc::mbar_init(hbar, 1);
    tc::mbar_init(hbar + 1, 1);
    tc::fence_mbar_init();
  }
  const uint32_t lh = tc::smem_u32(hb + cb * LH + unit), lb = tc::smem_u32(hbar);
  cl.sync();
  const bool tg = orow / UPC == 2;  // the cell-candidate gate uses tanh
  float sv[6];
  for (int t = 0; t < LT; ++t) {
    const int cur = t & 1, nxt = cur ^ 1;
    if (tid == 0 && t + 1 < LT) tc::mbar_expect_tx(hbar + nxt, XCH_BYTES);
    if (t > 0) tc::mbar_wait(hbar + cur, ((t - 1) >> 1) & 1);
    const float xcur = xn;
    if (t + 1 < LT) xn = xr[(int64_t)(t + 1) * LG];
    float v[16];  // v[r*4 + b]
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.f;
    const float* h = hb + cur * 4 * LH + 4 * ks;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float4 hv = *reinterpret_cast<const float4*>(h + b * LH + 64 * j);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          float q = v[r * 4 + b];
          q = fmaf(w[r][j].x, hv.x, q);
          q = fmaf(w[r][j].y, hv.y, q);
          q = fmaf(w[r][j].z, hv.z, q);
          q = fmaf(w[r][j].w, hv.w, q);
          v[r * 4 + b] = q;
        }
      }
    // reduce-scatter over the 16 lanes of the row group: level L keeps the half selected by
    // lane bit L and adds the partner's other half
#pragma unroll
    for (int L = 0; L < 4; ++L) {
      const int n = 16 >> L, hlf = n >> 1;
      const bool up = (ks >> L) & 1;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < hlf) {
          const float send = up ? v[i] : v[i + hlf];
          const float keep = up ? v[i + hlf] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1 << L);
        }
      }
    }
    const float pre = v[0] + xcur;
    gs[ob * RPC + orow] = tg ? tanhf(pre) : sigm(pre);
    __syncthreads();
    if (tid < NOWN) {
      const float ig = gs[cb * RPC + cu], fg = gs[cb * RPC + UPC + cu], gg = gs[cb * RPC + 2 * UPC + cu],
                  og = gs[cb * RPC + 3 * UPC + cu];
      cst = fg * cst + ig * gg;                 // c_t = f c_{t-1} + i g
      const float hv = og * tanhf(cst);         // h_t = o tanh(c_t)
      if (t + 1 < LT)
#pragma unroll
        for (int r = 0; r < CL; ++r) st_async_f32(mapa_u32(lh + nxt * 4 * LH * 4, r), hv, mapa_u32(lb + nxt * 8, r));
      sv[0] = cst, sv[1] = hv, sv[2] = ig, sv[3] = fg, sv[4] = gg, sv[5] = og;
    }
    __syncthreads();  // gs is rewritten by the next step
    if (tid < NOWN) {
      p.C[(cs * (LT + 1) + t + 1) * LH + unit] = sv[0];
      p.H[(cs * (LT + 1) + t + 1) * LH + unit] = sv[1];
      float* g = p.G + (cs * LT + t) * LG + unit;
      g[0] = sv[2];
      g[LH] = sv[3];
      g[2 * LH] = sv[4];
      g[3 * LH] = sv[5];
    }
  }
  cl.sync();  // no CTA exits while a peer may still address its shared memory
}

// Backward (BPTT) recurrence of one layer for one client.  The cell owners prefetch the next
// (earlier) step's gates, cell states and external gradient while the current step's
// W_hhᵀ·dpre partials (thread k, float4 over rows) are formed and reduce-scattered.
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(256, 2) k_lstm_bwd(RecArgs p) {
  pdl_wait();
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank(), a = blockIdx.x / CL, tid = threadIdx.x;
  extern __shared__ float sm[];
  float* Wt = sm;                           // [LH][WPB] k-major
  float* ds = sm + LH * WPB + 2 * 4 * LH;   // [RPC][4] dpre of this CTA's rows (4 batch rows contiguous)
  float* part = ds + 4 * RPC;               // [2][CL src][4][UPC] partial W_hhᵀ·dpre for this CTA's units
  uint64_t* pbar = reinterpret_cast<uint64_t*>(part + 2 * CL * 4 * UPC);  // [2] partials of a step landed
  {
    const float* W = p.wsrc + (int64_t)a * p.wstride + p.o_whh;
    for (int e = tid; e < RPC * LH; e += 256) {
      const int rl = e / LH, k = e - rl * LH;
      Wt[k * WPB + rl] = __ldg(W + (int64_t)grow_of(rl, c) * LH + k);
    }
  }
  const int cb = tid / UPC, cu = tid % UPC, unit = UPC * c + cu;
  const int64_t cs = (int64_t)a * p.B + cb;
  float dcs = 0.f, dhr = 0.f;  // carried dL/dc_t and the recurrent dL/dh_t of this cell
  // per-step inputs of the cell owners, prefetched one step ahead
  float nig = 0.f, nfg = 0.f, ngg = 0.f, nog = 0.f, nct = 0.f, ncp = 0.f, nex = 0.f;
  auto fetch = [&](int t) {
    const float* g = p.G + (cs * LT + t) * LG + unit;
    nig = g[0], nfg = g[LH], ngg = g[2 * LH], nog = g[3 * LH];
    nct = p.C[(cs * (LT + 1) + t + 1) * LH + unit];
    ncp = p.C[(cs * (LT + 1) + t) * LH + unit];
    nex = p.ext_mode == 0 ? ((t == LT - 1) ? p.ext[cs * LH + unit] : 0.f) : p.ext[(cs * LT + t) * LH + unit];
  };
  if (tid < NOWN) fetch(LT - 1);
  float sd[4];
  if (tid == 0) {
    tc::mbar_init(pbar, 1);
    tc::mbar_init(pbar + 1, 1);
    tc::fence_mbar_init();
  }
  // this thread's partial (column k = tid) goes to unit owner k / UPC: remote slot + barrier
  const uint32_t rpart = mapa_u32(tc::smem_u32(part + c * 4 * UPC + (tid % UPC)), tid / UPC);
  const uint32_t rpbar = mapa_u32(tc::smem_u32(pbar), tid / UPC);
  cl.sync();
  for (int t = LT - 1; t >= 0; --t) {
    const int pb = t & 1;
    if (tid == 0 && t > 0) tc::mbar_expect_tx(pbar + pb, XCH_BYTES);
    if (tid < NOWN) {
      const float dh = dhr + nex;
      const float ig = nig, fg = nfg, gg = ngg, og = nog, ct = nct, cp = ncp;
      if (t > 0) fetch(t - 1);
      const float tc = tanhf(ct);
      const float dct = dcs + dh * og * (1.f - tc * tc);
      const float di = dct * gg * ig * (1.f - ig), df = dct * cp * fg * (1.f - fg),
                  dg = dct * ig * (1.f - gg * gg), dob = dh * tc * og * (1.f - og);
      dcs = dct * fg;
      ds[cu * 4 + cb] = di;
      ds[(UPC + cu) * 4 + cb] = df;
      ds[(2 * UPC + cu) * 4 + cb] = dg;
      ds[(3 * UPC + cu) * 4 + cb] = dob;
      sd[0] = di, sd[1] = df, sd[2] = dg, sd[3] = dob;
    }
    __syncthreads();
    {  // partial dL/dh_{t-1}[b][k] over this CTA's 128 rows, scattered to the unit's owner CTA
      const int k = tid;
      float acc[4];
      const float* w = Wt + k * WPB;
      float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0, q2 = q0, q3 = q0;  // 16 independent chains
#pragma unroll 4
      for (int r = 0; r < RPC; r += 4) {
        const float4 wv = *reinterpret_cast<const float4*>(w + r);
        const float4 d0 = *reinterpret_cast<const float4*>(ds + (r + 0) * 4);
        const float4 d1 = *reinterpret_cast<const float4*>(ds + (r + 1) * 4);
        const float4 d2 = *reinterpret_cast<const float4*>(ds + (r + 2) * 4);
        const float4 d3 = *reinterpret_cast<const float4*>(ds + (r + 3) * 4);
        q0.x = fmaf(wv.x, d0.x, q0.x), q0.y = fmaf(wv.x, d0.y, q0.y), q0.z = fmaf(wv.x, d0.z, q0.z), q0.w = fmaf(wv.x, d0.w, q0.w);
        q1.x = fmaf(wv.y, d1.x, q1.x), q1.y = fmaf(wv.y, d1.y, q1.y), q1.z = fmaf(wv.y, d1.z, q1.z), q1.w = fmaf(wv.y, d1.w, q1.w);
        q2.x = fmaf(wv.z, d2.x, q2.x), q2.y = fmaf(wv.z, d2.y, q2.y), q2.z = fmaf(wv.z, d2.z, q2.z), q2.w = fmaf(wv.z, d2.w, q2.w);
        q3.x = fmaf(wv.w, d3.x, q3.x), q3.y = fmaf(wv.w, d3.y, q3.y), q3.z = fmaf(wv.w, d3.z, q3.z), q3.w = fmaf(wv.w, d3.w, q3.w);
      }
      acc[0] = (q0.x + q1.x) + (q2.x + q3.x);
      acc[1] = (q0.y + q1.y) + (q2.y + q3.y);
      acc[2] = (q0.z + q1.z) + (q2.z + q3.z);
      acc[3] = (q0.w + q1.w) + (q2.w + q3.w);
      if (t > 0)
#pragma unroll
        for (int b = 0; b < 4; ++b) st_async_f32(rpart + (pb * CL * 4 + b) * UPC * 4, acc[b], rpbar + pb * 8);
    }
    if (t > 0) tc::mbar_wait(pbar + pb, ((LT - 1 - t) >> 1) & 1);  // all CL CTAs' partials for my units
    if (tid < NOWN) {  // fixed source order
      float s = 0.f;
#pragma unroll
      for (int src = 0; src < CL; ++src) s += part[((pb * CL + src) * 4 + cb) * UPC + cu];
      dhr = s;
      float* d = p.dpre + (cs * LT + t) * LG + unit;  // stored after the barrier (see k_lstm_fwd_reg)
      d[0] = sd[0];
      d[LH] = sd[1];
      d[2 * LH] = sd[2];
      d[3 * LH] = sd[3];
    }
    __syncthreads();  // ds is rewritten by the next step
  }
  cl.sync();  // no CTA exits while a peer may still address its shared memory
}

// ---------------------------------------------------------------- batched per-client GEMM
// C(a, i, j) = Σ_kk A(a, i, kk) · Bm(a, j, kk); an operand element (a, x, y) lives at
// base + a·sa + (x / Tx)·sxr + (x % Tx)·sxt + (y / Ty)·syr + (y % Ty)·syt (Tx / Ty decompose
// a (batch row, time) index; INT32_MAX = plain affine).  Epilogue: store (+ up to two bias
// vectors over j) or SGD (dst = src − η·C).  64 x 64 tiles, 256 threads, fp32 FFMA.
struct Opnd {
  const float* base;
  int64_t sa, sxr, sxt, syr, syt;
  int Tx, Ty;
  __device__ __forceinline__ int64_t xoff(int a, int x) const {
    return a * sa + (Tx == 0x7fffffff ? (int64_t)x * sxt : (int64_t)(x / Tx) * sxr + (int64_t)(x % Tx) * sxt);
  }
  __device__ __forceinline__ int64_t yoff(int y) const {
    return Ty == 0x7fffffff ? (int64_t)y * syt : (int64_t)(y / Ty) * syr + (int64_t)(y % Ty) * syt;
  }
};
struct GemmArgs {
  Opnd A, Bm;
  int M, N, K;
  int mode;                // 0: out = C + bias0 + bias1; 1: SGD
  float* out;              // element (a, i, j) at out + a*o_sa + (i/To)*o_r + (i%To)*o_t + j*o_j
  int64_t o_sa, o_r, o_t, o_j;
  int To;
  const float* bias0;      // mode 0: bias vectors over j of client a at bias + a*b_sa (may be null)
  const float* bias1;
  int64_t b_sa;
  const float* src;        // mode 1: client a's current W at src + a*src_sa (same indexing as out)
  int64_t src_sa;
  float lr;
};

__global__ void __launch_bounds__(256) k_lstm_gemm(GemmArgs p) {
  pdl_wait();
  __shared__ float As[16][65], Bs[16][65];
  const int a = blockIdx.z, i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[4][4] = {};
  // a thread loads tile row x = tid % 64 (fixed for the whole K loop) at k = tid / 64 + 4q
  const int lx = threadIdx.x & 63, lk = threadIdx.x >> 6;
  const bool va = i0 + lx < p.M, vb = j0 + lx < p.N;
  const float* pa = p.A.base + (va ? p.A.xoff(a, i0 + lx) : 0);
  const float* pb = p.Bm.base + (vb ? p.Bm.xoff(a, j0 + lx) : 0);
  for (int k0 = 0; k0 < p.K; k0 += 16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int kk = lk + 4 * q, k = k0 + kk;
      As[kk][lx] = (va && k < p.K) ? pa[p.A.yoff(k)] : 0.f;
      Bs[kk][lx] = (vb && k < p.K) ? pb[p.Bm.yoff(k)] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = As[kk][ty + 16 * u], bv[u] = Bs[kk][tx + 16 * u];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i >= p.M || j >= p.N) continue;
      const int64_t o = (int64_t)(i / p.To) * p.o_r + (int64_t)(i % p.To) * p.o_t + (int64_t)j * p.o_j;
      if (p.mode == 0) {
        float r = acc[u][v];
        if (p.bias0) r += p.bias0[a * p.b_sa + j];
        if (p.bias1) r += p.bias1[a * p.b_sa + j];
        p.out[a * p.o_sa + o] = r;
      } else {
        p.out[a * p.o_sa + o] = p.src[a * p.src_sa + o] - p.lr * acc[u][v];
      }
    }
}

// 128x128 tiles, 8x8 outputs per thread (two 4-row x two 4-column quads, 64 apart, read as
// float4 from shared memory), BK = 8 with register prefetch of the next k-tile.  Every output
// accumulates its K products in ascending k with one fmaf each, the same order as the 64x64
// k_lstm_gemm, so results are bit-identical; the 8x8 register block halves shared-memory
// traffic per FMA.
constexpr int G2_T = 128, G2_K = 8, G2_P = G2_T + 4;
__global__ void __launch_bounds__(256) k_lstm_gemm128(GemmArgs p) {
  pdl_wait();
  __shared__ __align__(16) float As[2][G2_K][G2_P];
  __shared__ __align__(16) float Bs[2][G2_K][G2_P];
  const int a = blockIdx.z, i0 = blockIdx.y * G2_T, j0 = blockIdx.x * G2_T;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  // Loads of a 128 x 8 operand tile: 4 elements per thread.  Row-contiguous operands (the
  // row index is the unit-stride one): thread = row lx, k = lk + 2q (a warp reads 32
  // consecutive rows).  k-contiguous operands: thread = row tid/2, k = 4·(tid&1) + q (two
  // threads read one row's 8 consecutive k).
  const bool ka = p.A.Ty == 0x7fffffff && p.A.syt == 1, kb = p.Bm.Ty == 0x7fffffff && p.Bm.syt == 1;
  const int rA = ka ? threadIdx.x >> 1 : threadIdx.x & 127, kA = ka ? 4 * (threadIdx.x & 1) : threadIdx.x >> 7;
  const int rB = kb ? threadIdx.x >> 1 : threadIdx.x & 127, kB = kb ? 4 * (threadIdx.x & 1) : threadIdx.x >> 7;
  const int dA = ka ? 1 : 2, dB = kb ? 1 : 2;  // k step between a thread's 4 elements
  const bool va = i0 + rA < p.M, vb = j0 + rB < p.N;
  const float* pa = p.A.base + (va ? p.A.xoff(a, i0 + rA) : 0);
  const float* pb = p.Bm.base + (vb ? p.Bm.xoff(a, j0 + rB) : 0);
  float ra[4], rb[4];
  auto gload = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = k0 + kA + dA * q, kq = k0 + kB + dB * q;
      ra[q] = (va && k < p.K) ? pa[p.A.yoff(k)] : 0.f;
      rb[q] = (vb && kq < p.K) ? pb[p.Bm.yoff(kq)] : 0.f;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 4; ++q) As[buf][kA + dA * q][rA] = ra[q], Bs[buf][kB + dB * q][rB] = rb[q];
  };
  float acc[8][8] = {};
  gload(0);
  sstore(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < p.K; k0 += G2_K) {
    const bool more = k0 + G2_K < p.K;
    if (more) gload(k0 + G2_K);
#pragma unroll
    for (int kk = 0; kk < G2_K; ++kk) {
      float av[8], bv[8];
      *reinterpret_cast<float4*>(av) = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      *reinterpret_cast<float4*>(av + 4) = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      *reinterpret_cast<float4*>(bv) = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      *reinterpret_cast<float4*>(bv + 4) = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(av[u], bv[v], acc[u][v]);
    }
    if (more) {
      sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int u = 0; u < 8; ++u)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int i = i0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + u - 4);
      const int j = j0 + (v < 4 ? tx * 4 + v : 64 + tx * 4 + v - 4);
      if (i >= p.M || j >= p.N) continue;
      const int64_t o = (int64_t)(i / p.To) * p.o_r + (int64_t)(i % p.To) * p.o_t + (int64_t)j * p.o_j;
      if (p.mode == 0) {
        float r = acc[u][v];
        if (p.bias0) r += p.bias0[a * p.b_sa + j];
        if (p.bias1) r += p.bias1[a * p.b_sa + j];
        p.out[a * p.o_sa + o] = r;
      } else {
        p.out[a * p.o_sa + o] = p.src[a * p.src_sa + o] - p.lr * acc[u][v];
      }
    }
}

// ---------------------------------------------------------------- embedding, layer-0 input
// E[s][t][j] = emb[x_t][j]; Xp0[s][t][n] = W_ih0[n]·E[s][t] + b_ih0[n] + b_hh0[n].  One CTA per slot.
struct EmbArgs {
  const uint8_t* xpack;   // [R][LT] characters
  const int32_t* sidx;    // slot -> packed row or -1
  const float* wsrc;
  int64_t wstride;
  int64_t o_emb, o_wih0, o_bih0, o_bhh0;
  int B;
  float* E;               // [S][LT][LE]
  float* xp;              // [S][LT][LG]
};
__global__ void __launch_bounds__(256) k_lstm_embed(EmbArgs p) {
  pdl_wait();
  __shared__ float Ws[LG * LE], bsum[LG], es[LT * LE];
  const int s = blockIdx.x, a = s / p.B;
  const float* w = p.wsrc + (int64_t)a * p.wstride;
  for (int e = threadIdx.x; e < LG * LE; e += 256) Ws[e] = w[p.o_wih0 + e];
  for (int e = threadIdx.x; e < LG; e += 256) bsum[e] = w[p.o_bih0 + e] + w[p.o_bhh0 + e];
  const int row = p.sidx[s];
  for (int e = threadIdx.x; e < LT * LE; e += 256) {
    const int t = e / LE, j = e - t * LE;
    // padding rows (row < 0): char 0 (dz = 0 there).  The load always reads row max(row, 0): the
    // compiler turned the conditional load into an unconditional one (compute-sanitizer flagged
    // the row -1 read before the buffer).
    const int chl = p.xpack[(int64_t)(row >= 0 ? row : 0) * LT + t];
    const int ch = row >= 0 ? chl : 0;
    es[e] = w[p.o_emb + ch * LE + j];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < LT * LE; e += 256) p.E[(int64_t)s * LT * LE + e] = es[e];
  for (int e = threadIdx.x; e < LT * LG; e += 256) {
    const int t = e / LG, n = e - t * LG;
    float acc = bsum[n];
#pragma unroll
    for (int j = 0; j < LE; ++j) acc = fmaf(Ws[n * LE + j], es[t * LE + j], acc);
    p.xp[(int64_t)s * LT * LG + e] = acc;
  }
}

// ---------------------------------------------------------------- fc head + CE + fc SGD
// One CTA per client: z = W_fc h2_T + b_fc, dz = (softmax − onehot)/|b| (0 past |b|),
// dh2_T = W_fcᵀ dz, W_fc -= η Σ_r dz ⊗ h2_T, b_fc -= η Σ_r dz.
struct HeadArgs {
  const float* H1;        // [S][T+1][LH] layer-2 hidden states
  const int32_t* ypack;
  const int32_t* sidx;
  const int32_t* bs;
  const float* wsrc;
  int64_t wstride;
  float* dst;
  int64_t P_pad, o_wfc, o_bfc;
  int B;
  float lr;
  float* dhT;             // [S][LH]
};
__global__ void __launch_bounds__(256) k_lstm_head(HeadArgs p) {
  pdl_wait();
  __shared__ float hT[4][LH], dz[4][LV];
  extern __shared__ float Wf[];  // [LV][LH] (80 KB, dynamic)
  const int a = blockIdx.x, b = p.bs[a], tid = threadIdx.x;
  const float* w = p.wsrc + (int64_t)a * p.wstride;
  for (int e = tid; e < LV * LH; e += 256) Wf[e] = w[p.o_wfc + e];
  for (int e = tid; e < 4 * LH; e += 256) {
    const int r = e / LH, k = e - r * LH;
    const float hv = p.H1[(((int64_t)a * p.B + (r < p.B ? r : 0)) * (LT + 1) + LT) * LH + k];  // in-bounds load
    hT[r][k] = r < p.B ? hv : 0.f;
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  for (int idx = warp; idx < 4 * LV; idx += 8) {
    const int r = idx / LV, q = idx - r * LV;
    float s = 0.f;
    for (int k = lane; k < LH; k += 32) s = fmaf(Wf[q * LH + k], hT[r][k], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) dz[r][q] = s + w[p.o_bfc + q];
  }
  __syncthreads();
  if (tid < 4) {
    const int r = tid;
    if (r < b) {
      const int y = p.ypack[p.sidx[a * p.B + r]];
      float mx = dz[r][0];
      for (int q = 1; q < LV; ++q) mx = fmaxf(mx, dz[r][q]);
      float s = 0.f;
      for (int q = 0; q < LV; ++q) s += expf(dz[r][q] - mx);
      const float inv = 1.f / (float)b;
      for (int q = 0; q < LV; ++q) dz[r][q] = (expf(dz[r][q] - mx) / s - (q == y ? 1.f : 0.f)) * inv;
    } else {
      for (int q = 0; q < LV; ++q) dz[r][q] = 0.f;
    }
  }
  __syncthreads();
  for (int e = tid; e < p.B * LH; e += 256) {
    const int r = e / LH, k = e - r * LH;
    float s = 0.f;
    if (r < 4)
      for (int q = 0; q < LV; ++q) s = fmaf(Wf[q * LH + k], dz[r][q], s);
    p.dhT[((int64_t)a * p.B + r) * LH + k] = s;
  }
  float* d = p.dst + (int64_t)a * p.P_pad;
  for (int e = tid; e < LV * LH; e += 256) {
    const int q = e / LH, k = e - q * LH;
    float g = 0.f;
    for (int r = 0; r < 4; ++r) g = fmaf(dz[r][q], hT[r][k], g);
    d[p.o_wfc + e] = Wf[e] - p.lr * g;
  }
  if (tid < LV) {
    float g = 0.f;
    for (int r = 0; r < 4; ++r) g += dz[r][tid];
    d[p.o_bfc + tid] = w[p.o_bfc + tid] - p.lr * g;
  }
}

// ---------------------------------------------------------------- biases and embedding SGD
// b_ih, b_hh -= η Σ_{r,t} dpre (both receive the same gradient).  grid (LG/256, A).
__global__ void k_lstm_bias_sgd(const float* __restrict__ dpre, int B, const float* wsrc, int64_t wstride,
                                float* dst, int64_t P_pad, int64_t o_bih, int64_t o_bhh, float lr) {
  pdl_wait();
  const int a = blockIdx.y, n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= LG) return;
  float g = 0.f;
  for (int r = 0; r < B; ++r) {
    const float* d = dpre + (((int64_t)a * B + r) * LT) * LG + n;
    for (int t = 0; t < LT; ++t) g += d[(int64_t)t * LG];
  }
  const float* w = wsrc + (int64_t)a * wstride;
  float* o = dst + (int64_t)a * P_pad;
  o[o_bih + n] = w[o_bih + n] - lr * g;
  o[o_bhh + n] = w[o_bhh + n] - lr * g;
}

// emb[c][j] -= η Σ_{(r,t): x_{r,t} = c} dE[r][t][j], dE = dpre0 · W_ih0 (old).  One CTA per client.
__global__ void k_lstm_emb_sgd(const float* __restrict__ dE, const uint8_t* __restrict__ xpack,
                               const int32_t* __restrict__ sidx, int B, const float* wsrc, int64_t wstride,
                               float* dst, int64_t P_pad, int64_t o_emb, float lr) {
  pdl_wait();
  const int a = blockIdx.x;
  const float* w = wsrc + (int64_t)a * wstride;
  float* o = dst + (int64_t)a * P_pad;
  for (int e = threadIdx.x; e < LV * LE; e += blockDim.x) {
    const int ch = e / LE, j = e - ch * LE;
    float g = 0.f;
    for (int r = 0; r < B; ++r) {
      const int row = sidx[a * B + r];
      const float* de = dE + (((int64_t)a * B + r) * LT) * LE + j;
      for (int t = 0; t < LT; ++t) {
        const int cl = xpack[(int64_t)(row >= 0 ? row : 0) * LT + t];  // always an in-bounds load
        const int c = row >= 0 ? cl : 0;
        if (c == ch) g += de[t * LE];
      }
    }
    o[o_emb + e] = w[o_emb + e] - lr * g;
  }
}

Opnd affine(const float* base, int64_t sa, int64_t sx, int64_t sy) {
  return Opnd{base, sa, 0, sx, 0, sy, 0x7fffffff, 0x7fffffff};
}

}  // namespace

bool lstm_layout(Layout* L) {
  L->model = FL_MODEL_CHAR_LSTM;
  LstmOff& q = L->lo;
  auto up32 = [](int64_t x) { return (x + 31) / 32 * 32; };
  // canonical torch order: emb, wih0, whh0, bih0, bhh0, wih1, whh1, bih1, bhh1, wfc, bfc
  const int64_t sz[11] = {LV * LE, LG * LE, LG * LH, LG, LG, LG * LH, LG * LH, LG, LG, LV * LH, LV};
  int64_t* dst[11] = {&q.emb, &q.wih[0], &q.whh[0], &q.bih[0], &q.bhh[0], &q.wih[1], &q.whh[1],
                      &q.bih[1], &q.bhh[1], &q.wfc, &q.bfc};
  int64_t o = 0, c = 0;
  L->canon_of.clear();
  std::vector<int64_t> m;
  for (int i = 0; i < 11; ++i) {
    *dst[i] = o;
    m.resize((size_t)up32(o + sz[i]), -1);
    for (int64_t e = 0; e < sz[i]; ++e) m[(size_t)(o + e)] = c + e;
    c += sz[i];
    o = up32(o + sz[i]);
  }
  L->P = c;  // 819,920
  L->P_pad = o;
  L->canon_of = m;
  L->D_in = LT / 4;   // 80 one-byte characters per sample, moved as 20 four-byte words
  L->D_pack = LT / 4;
  return true;
}

// One wave of local SGD for the char-LSTM (all active clients of the wave, one step each).
int lstm_wave(const Layout& L, const WaveArgs& wa, const uint8_t* xpack, const int32_t* ypack, const float* theta_g,
              float* slots, LstmBufs& b, cudaStream_t st) {
  const LstmOff& q = L.lo;
  const int A = wa.A, B = wa.B;
  const float* wbase = wa.first ? theta_g : slots;
  const int64_t wstride = wa.first ? 0 : L.P_pad;
  const float lr = wa.lr;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_lstm_fwd_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, REC_SMEM);
    cudaFuncSetAttribute(k_lstm_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, REC_SMEM);
    if (CL > 8) {  // 16-CTA clusters are a non-portable size
      cudaFuncSetAttribute(k_lstm_fwd_reg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_lstm_bwd, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    cudaFuncSetAttribute(k_lstm_head, cudaFuncAttributeMaxDynamicSharedMemorySize, LV * LH * 4);
    attr = true;
  }
  const int64_t S_T1 = (int64_t)(LT + 1) * LH;  // per-slot stride of H / C
  int n = 0;
  auto gemm = [&](const GemmArgs& g) {
    // small waves: 128x128 tiles would leave most SMs idle; the 64x64 kernel is bit-identical
    const int64_t b128 = (int64_t)((g.N + G2_T - 1) / G2_T) * ((g.M + G2_T - 1) / G2_T) * A;
    if (b128 >= 2 * 148)
      launch_pdl(wa.pdl, k_lstm_gemm128, dim3((g.N + G2_T - 1) / G2_T, (g.M + G2_T - 1) / G2_T, A), 256, 0, st, g);
    else
      launch_pdl(wa.pdl, k_lstm_gemm, dim3((g.N + 63) / 64, (g.M + 63) / 64, A), 256, 0, st, g);
    ++n;
  };
  const int M = B * LT;  // (batch row, time) rows per client
  // ---- forward: embedding + layer-0 input projection, layer-0 recurrence
  EmbArgs ea{xpack, wa.sidx, wbase, wstride, q.emb, q.wih[0], q.bih[0], q.bhh[0], B, b.E, b.xp};
  launch_pdl(wa.pdl, k_lstm_embed, dim3(A * B), 256, 0, st, ea), ++n;
  RecArgs r0{wbase, wstride, q.whh[0], B, b.xp, b.G0, b.C0, b.H0, nullptr, 0, nullptr};
  auto fwd = k_lstm_fwd_reg;
  launch_pdl(wa.pdl, fwd, dim3(A * CL), FT, REC_SMEM, st, r0), ++n;
  // tensor-core GEMMs (TF32, k_lstm_tc.cu) unless math = 1 (FP32 SIMT everywhere)
  const bool tc = wa.use_tc && lstm_tc_supported(B);
  LstmTcIn ti{A, B, wa.first ? 0 : 1, b.slots, wbase, wstride, wa.first ? 1 : wa.wclients, L.P_pad, slots,
              q.wih[1], q.whh[1], q.whh[0], q.bih[1], q.bhh[1], b.H0, b.H1, b.dpre, b.xp, b.dX, lr, wa.pdl};
  auto tcg = [&](int which) {
    if (lstm_gemm_tc(which, ti, st) < 0) return false;
    ++n;
    return true;
  };
  // layer-1 input projection: xp[s][t] = W_ih1 · H0[s][t+1] + b_ih1 + b_hh1
  if (tc) {
    if (!tcg(1)) return -1;
  } else {
    GemmArgs g{};
    g.A = Opnd{b.H0 + LH, (int64_t)B * S_T1, S_T1, LH, 0, 1, LT, 0x7fffffff};
    g.Bm = affine(wbase + q.wih[1], wstride, LH, 1);
    g.M = M, g.N = LG, g.K = LH, g.mode = 0;
    g.out = b.xp, g.o_sa = (int64_t)M * LG, g.o_r = (int64_t)LT * LG, g.o_t = LG, g.o_j = 1, g.To = LT;
    g.bias0 = wbase + q.bih[1], g.bias1 = wbase + q.bhh[1], g.b_sa = wstride;
    gemm(g);
  }
  RecArgs r1{wbase, wstride, q.whh[1], B, b.xp, b.G1, b.C1, b.H1, nullptr, 0, nullptr};
  launch_pdl(wa.pdl, fwd, dim3(A * CL), FT, REC_SMEM, st, r1), ++n;
  // ---- head (fc SGD) and layer-1 BPTT
  HeadArgs ha{b.H1, ypack, wa.sidx, wa.bs, wbase, wstride, slots, L.P_pad, q.wfc, q.bfc, B, lr, b.dhT};
  launch_pdl(wa.pdl, k_lstm_head, dim3(A), 256, LV * LH * 4, st, ha), ++n;
  RecArgs rb1{wbase, wstride, q.whh[1], B, nullptr, b.G1, b.C1, b.H1, b.dhT, 0, b.dpre};
  launch_pdl(wa.pdl, k_lstm_bwd, dim3(A * CL), 256, REC_SMEM, st, rb1), ++n;
  // dX of layer 1 (old W_ih1): dX[s][t][k] = Σ_n dpre[s][t][n] W_ih1[n][k]
  if (tc) {
    if (!tcg(2)) return -1;
  } else {
    GemmArgs g{};
    g.A = affine(b.dpre, (int64_t)M * LG, LG, 1);
    g.Bm = affine(wbase + q.wih[1], wstride, 1, LH);
    g.M = M, g.N = LH, g.K = LG, g.mode = 0;
    g.out = b.dX, g.o_sa = (int64_t)M * LH, g.o_r = (int64_t)LT * LH, g.o_t = LH, g.o_j = 1, g.To = LT;
    gemm(g);
  }
  // layer-1 weight gradients + SGD: W_hh1 -= η Σ dpreᵀ H1[t], W_ih1 -= η Σ dpreᵀ H0[t+1]
  if (tc) {
    if (!tcg(3) || !tcg(4)) return -1;
  }
  for (int which = 0; which < 2 && !tc; ++which) {
    GemmArgs g{};
    g.A = Opnd{b.dpre, (int64_t)M * LG, 0, 1, (int64_t)LT * LG, LG, 0x7fffffff, LT};  // (n, m = (r, t))
    const float* hsrc = which == 0 ? b.H1 : b.H0 + LH;
    g.Bm = Opnd{hsrc, (int64_t)B * S_T1, 0, 1, S_T1, LH, 0x7fffffff, LT};            // (k, m)
    g.M = LG, g.N = LH, g.K = M, g.mode = 1;
    const int64_t ow = which == 0 ? q.whh[1] : q.wih[1];
    g.out = slots + ow, g.o_sa = L.P_pad, g.o_r = 0, g.o_t = LH, g.o_j = 1, g.To = 0x7fffffff;
    g.src = wbase + ow, g.src_sa = wstride, g.lr = lr;
    gemm(g);
  }
  launch_pdl(wa.pdl, k_lstm_bias_sgd, dim3(LG / 256, A), 256, 0, st, (const float*)b.dpre, B, wbase, wstride, slots,
             L.P_pad, q.bih[1], q.bhh[1], lr), ++n;
  // ---- layer-0 BPTT with the external gradient dX, then its gradients
  RecArgs rb0{wbase, wstride, q.whh[0], B, nullptr, b.G0, b.C0, b.H0, b.dX, 1, b.dpre};
  launch_pdl(wa.pdl, k_lstm_bwd, dim3(A * CL), 256, REC_SMEM, st, rb0), ++n;
  {  // dE = dpre0 · W_ih0 (old), before W_ih0 is updated
    GemmArgs g{};
    g.A = affine(b.dpre, (int64_t)M * LG, LG, 1);
    g.Bm = affine(wbase + q.wih[0], wstride, 1, LE);
    g.M = M, g.N = LE, g.K = LG, g.mode = 0;
    g.out = b.dE, g.o_sa = (int64_t)M * LE, g.o_r = (int64_t)LT * LE, g.o_t = LE, g.o_j = 1, g.To = LT;
    gemm(g);
  }
  if (tc) {  // W_hh0 -= η Σ dpre0ᵀ H0[t]
    if (!tcg(6)) return -1;
  } else {  // W_hh0 -= η Σ dpre0ᵀ H0[t]
    GemmArgs g{};
    g.A = Opnd{b.dpre, (int64_t)M * LG, 0, 1, (int64_t)LT * LG, LG, 0x7fffffff, LT};
    g.Bm = Opnd{b.H0, (int64_t)B * S_T1, 0, 1, S_T1, LH, 0x7fffffff, LT};
    g.M = LG, g.N = LH, g.K = M, g.mode = 1;
    g.out = slots + q.whh[0], g.o_sa = L.P_pad, g.o_r = 0, g.o_t = LH, g.o_j = 1, g.To = 0x7fffffff;
    g.src = wbase + q.whh[0], g.src_sa = wstride, g.lr = lr;
    gemm(g);
  }
  {  // W_ih0 -= η Σ dpre0ᵀ E
    GemmArgs g{};
    g.A = Opnd{b.dpre, (int64_t)M * LG, 0, 1, (int64_t)LT * LG, LG, 0x7fffffff, LT};
    g.Bm = Opnd{b.E, (int64_t)M * LE, 0, 1, (int64_t)LT * LE, LE, 0x7fffffff, LT};
    g.M = LG, g.N = LE, g.K = M, g.mode = 1;
    g.out = slots + q.wih[0], g.o_sa = L.P_pad, g.o_r = 0, g.o_t = LE, g.o_j = 1, g.To = 0x7fffffff;
    g.src = wbase + q.wih[0], g.src_sa = wstride, g.lr = lr;
    gemm(g);
  }
  launch_pdl(wa.pdl, k_lstm_bias_sgd, dim3(LG / 256, A), 256, 0, st, (const float*)b.dpre, B, wbase, wstride, slots,
             L.P_pad, q.bih[0], q.bhh[0], lr), ++n;
  launch_pdl(wa.pdl, k_lstm_emb_sgd, dim3(A), 256, 0, st, (const float*)b.dE, xpack, wa.sidx, B, wbase, wstride, slots,
             L.P_pad, q.emb, lr), ++n;
  return cudaGetLastError() == cudaSuccess ? n : -1;
}

int64_t lstm_act_floats(int64_t S, int which) {
  switch (which) {
    case 0: return S * LT * LG;       // xp, G0, G1, dpre
    case 1: return S * (LT + 1) * LH; // H0, H1, C0, C1
    case 2: return S * LT * LH;       // dX
    case 3: return S * LT * LE;       // E, dE
    case 4: return S * LH;            // dhT
  }
  return 0;
}

}  // namespace flb
