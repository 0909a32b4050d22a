// k_cnn_simt.cu — one SGD wave of the CNN family on FP32 CUDA cores ("math = 1" path,
// and the reference the tensor-core kernels are checked against).
//
// A wave is SGD step t of every active local client (PAPER.md P:176,
// P:362-363).  Every layer is a grouped GEMM over the active clients (grid.z = client, or
// client x split-K chunk), expressed as an "op" with element accessors and an epilogue,
// run by one tiled SIMT GEMM template.  Activations are slot-major NHWC: slot (a, r) =
// a*B + r.  Weights of client a are read from θ_g on the first wave (slot init fused, a3)
// and from the client's slot afterwards; SGD (a7) is fused into the dW epilogues.
#include <cuda_runtime.h>
#include <stdint.h>

#include "dev_util.cuh"
#include "fl_internal.h"

namespace flb {
namespace {

constexpr int TK = 16, NT = 256;

// C[m][n] = Σ_k A(z,m,k)·Bv(z,n,k) for problem z; op.store() consumes C.
// BM x BN tile (32 or 64 each), 256 threads as 16 x 16, each thread a (BM/16) x (BN/16)
// register block; narrow layers (N or M <= 32) get narrow tiles so no half-empty tile is
// loaded and multiplied.  The k loop runs in ascending order with one fmaf per product for
// every tile shape, so the shape never changes a result bit.
template <class Op, int BM, int BN>
__global__ void __launch_bounds__(NT) k_gemm(const Op op) {
  constexpr int RM = BM / 16, RN = BN / 16;
  const int z = blockIdx.z;
  int M, N, kb, ke;
  if (!op.setup(z, M, N, kb, ke)) return;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  if (m0 >= M || n0 >= N) return;
  __shared__ float As[TK][BM + 4];
  __shared__ float Bs[TK][BN + 4];
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  float acc[RM][RN];
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) acc[i][j] = 0.f;
  for (int k0 = kb; k0 < ke; k0 += TK) {
#pragma unroll
    for (int i = 0; i < (BM * TK) / NT; ++i) {
      const int e = tid + i * NT;
      int mm, kk;
      if (Op::kAK) { mm = e / TK; kk = e % TK; } else { mm = e % BM; kk = e / BM; }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < ke) ? op.A(z, m, k) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < (BN * TK) / NT; ++i) {
      const int e = tid + i * NT;
      int nn, kk;
      if (Op::kBK) { nn = e / TK; kk = e % TK; } else { nn = e % BN; kk = e / BN; }
      const int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < ke) ? op.Bv(z, n, k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[RM], b[RN];
#pragma unroll
      for (int i = 0; i < RM; ++i) a[i] = As[kk][ty * RM + i];
#pragma unroll
      for (int j = 0; j < RN; ++j) b[j] = Bs[kk][tx * RN + j];
#pragma unroll
      for (int i = 0; i < RM; ++i)
#pragma unroll
        for (int j = 0; j < RN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RM; ++i)
#pragma unroll
    for (int j = 0; j < RN; ++j) {
      const int m = m0 + ty * RM + i, n = n0 + tx * RN + j;
      if (m < M && n < N) op.store(z, m, n, acc[i][j]);
    }
}

struct WSrc {  // weights of client z: θ_g on the first wave, the client's slot afterwards
  const float* base;
  int64_t stride;
  __device__ const float* at(int z, int64_t off) const { return base + (int64_t)z * stride + off; }
};

// conv 5x5 'same' (pad 2) as implicit GEMM. rows (r,h,w), cols o, K = (kh,kw,c).
// Y = conv(X) + bias (pre-activation).  X rows come from the packed input via sidx (conv1)
// or from the slot-major activations (conv2).
struct ConvFwd {
  static constexpr bool kAK = true, kBK = true;
  const float* X;
  const int32_t* sidx;
  const int32_t* bs;
  int B, H, W, C, O;
  WSrc w;
  int64_t o_w, o_b;
  float* Y;
  __device__ bool setup(int z, int& M, int& N, int& kb, int& ke) const {
    M = bs[z] * H * W; N = O; kb = 0; ke = 25 * C;
    return M > 0;
  }
  __device__ float A(int z, int m, int k) const {
    const int HW = H * W, r = m / HW, pix = m - r * HW, h = pix / W, x = pix - h * W;
    const int tap = k / C, c = k - tap * C, kh = tap / 5, kw = tap - kh * 5;
    const int ih = h + kh - 2, iw = x + kw - 2;
    if (ih < 0 || ih >= H || iw < 0 || iw >= W) return 0.f;
    const int64_t row = sidx ? (int64_t)sidx[z * B + r] : (int64_t)z * B + r;
    return X[((row * H + ih) * W + iw) * C + c];
  }
  __device__ float Bv(int z, int n, int k) const { return *w.at(z, o_w + (int64_t)n * 25 * C + k); }
  __device__ void store(int z, int m, int n, float v) const {
    Y[((int64_t)z * B * H * W + m) * O + n] = v + *w.at(z, o_b + n);
  }
};

// dX of a 5x5 'same' conv (transposed conv): rows (r,y,x), cols c, K = (kh,kw,o).
struct ConvDx {
  static constexpr bool kAK = true, kBK = false;
  const float* dY;
  const int32_t* bs;
  int B, H, W, C, O;
  WSrc w;
  int64_t o_w;
  float* dX;
  __device__ bool setup(int z, int& M, int& N, int& kb, int& ke) const {
    M = bs[z] * H * W; N = C; kb = 0; ke = 25 * O;
    return M > 0;
  }
  __device__ float A(int z, int m, int k) const {
    const int HW = H * W, r = m / HW, pix = m - r * HW, y = pix / W, x = pix - y * W;
    const int tap = k / O, o = k - tap * O, kh = tap / 5, kw = tap - kh * 5;
    const int iy = y - kh + 2, ix = x - kw + 2;
    if (iy < 0 || iy >= H || ix < 0 || ix >= W) return 0.f;
    return dY[((((int64_t)z * B + r) * H + iy) * W + ix) * O + o];
  }
  __device__ float Bv(int z, int n, int k) const {
    const int tap = k / O, o = k - tap * O;
    return *w.at(z, o_w + ((int64_t)o * 25 + tap) * C + n);
  }
  __device__ void store(int z, int m, int n, float v) const { dX[((int64_t)z * B * H * W + m) * C + n] = v; }
};

// dW partial of a 5x5 conv over a chunk of rows: rows o, cols (kh,kw,c) plus a bias
// column (B = 1), K = pixels of the chunk's samples.
struct ConvDw {
  static constexpr bool kAK = false, kBK = false;
  const float* dY;
  const float* X;
  const int32_t* sidx;
  const int32_t* bs;
  int B, H, W, C, O, nch, rpc;
  float* part;
  __device__ bool setup(int z, int& M, int& N, int& kb, int& ke) const {
    const int a = z / nch, ch = z - a * nch, r0 = ch * rpc;
    int r1 = r0 + rpc;
    if (r1 > bs[a]) r1 = bs[a];
    M = O; N = 25 * C + 1; kb = 0; ke = (r1 - r0) * H * W;
    return r1 > r0;
  }
  __device__ float A(int z, int m, int k) const {
    const int a = z / nch, ch = z - a * nch, HW = H * W;
    const int r = ch * rpc + k / HW, pix = k % HW;
    return dY[(((int64_t)a * B + r) * HW + pix) * O + m];
  }
  __device__ float Bv(int z, int n, int k) const {
    if (n == 25 * C) return 1.f;
    const int a = z / nch, ch = z - a * nch, HW = H * W;
    const int r = ch * rpc + k / HW, pix = k % HW, h = pix / W, x = pix - h * W;
    const int tap = n / C, c = n - tap * C, kh = tap / 5, kw = tap - kh * 5;
    const int ih = h + kh - 2, iw = x + kw - 2;
    if (ih < 0 || ih >= H || iw < 0 || iw >= W) return 0.f;
    const int64_t row = sidx ? (int64_t)sidx[a * B + r] : (int64_t)a * B + r;
    return X[((row * H + ih) * W + iw) * C + c];
  }
  __device__ void store(int z, int m, int n, float v) const {
    const int N = 25 * C + 1;
    part[(int64_t)z * O * N + (int64_t)m * N + n] = v;
  }
};

// fc1 forward: h = ReLU(p2·W1ᵀ + b1). rows r, cols n, K = F.
struct FcFwd {
  static constexpr bool kAK = true, kBK = true;
  const float* X;
  const int32_t* bs;
  int B, F, HID;
  WSrc w;
  int64_t o_w, o_b;
  float* h;
  __device__ bool setup(int z, int& M, int& N, int& kb, int& ke) const {
    M = bs[z]; N = HID; kb = 0; ke = F;
    return M > 0;
  }
  __device__ float A(int z, int m, int k) const { return X[((int64_t)z * B + m) * F + k]; }
  __device__ float Bv(int z, int n, int k) const { return *w.at(z, o_w + (int64_t)n * F + k); }
  __device__ void store(int z, int m, int n, float v) const {
    v += *w.at(z, o_b + n);
    h[((int64_t)z * B + m) * HID + n] = v > 0.f ? v : 0.f;
  }
};

// fc1 forward split over K (small waves: a client's F = 15,360-long dot products would
// otherwise run on HID/64 blocks): z = client·S + chunk, partial sums to part[z][m][n].
struct FcFwdPart {
  static constexpr bool kAK = true, kBK = true;
  const float* X;
  const int32_t* bs;
  int B, F, HID, S;
  WSrc w;
  int64_t o_w;
  float* part;  // [A·S][B][HID]
  __device__ bool setup(int z, int& M, int& N, int& kb, int& ke) const {
    const int a = z / S, c = z - a * S, kc = (F + S - 1) / S;
    M = bs[a]; N = HID; kb = c * kc; ke = min(F, kb + kc);
    return M > 0 && kb < ke;
  }
  __device__ float A(int z, int m, int k) const { return X[((int64_t)(z / S) * B + m) * F + k]; }
  __device__ float Bv(int z, int n, int k) const { return *w.at(z / S, o_w + (int64_t)n * F + k); }
  __device__ void store(int z, int m, int n, float v) const { part[((int64_t)z * B + m) * HID + n] = v; }
};
// h = ReLU(Σ_chunks part + b1), chunks in fixed order.
__global__ void k_fc_fwd_reduce(const float* __restrict__ part, const int32_t* __restrict__ bs, int B, int HID, int S,
                                WSrc w, int64_t o_b, float* __restrict__ h) {
  const int a = blockIdx.y, r = blockIdx.x;
  if (r >= bs[a]) return;
  for (int n = threadIdx.x; n < HID; n += blockDim.x) {
    float v = 0.f;
    for (int c = 0; c < S; ++c) v += part[(((int64_t)a * S + c) * B + r) * HID + n];
    v += *w.at(a, o_b + n);
    h[((int64_t)a * B + r) * HID + n] = v > 0.f ? v : 0.f;
  }
}

// fc1 dX: dp2 = dh·W1. rows r, cols k (F), K = HID.
struct FcDx {
  static constexpr bool kAK = true, kBK = false;
  const float* dh;
  const int32_t* bs;
  int B, F, HID;
  WSrc w;
  int64_t o_w;
  float* dX;
  __device__ bool setup(int z, int& M, int& N, int& kb, int& ke) const {
    M = bs[z]; N = F; kb = 0; ke = HID;
    return M > 0;
  }
  __device__ float A(int z, int m, int k) const { return dh[((int64_t)z * B + m) * HID + k]; }
  __device__ float Bv(int z, int n, int k) const { return *w.at(z, o_w + (int64_t)k * F + n); }
  __device__ void store(int z, int m, int n, float v) const { dX[((int64_t)z * B + m) * F + n] = v; }
};

// fc1 dW with fused SGD: W1 <- W1 − η·dhᵀ·p2 (+ bias column). rows n, cols k, K = r.
struct FcDwSgd {
  static constexpr bool kAK = false, kBK = false;
  const float* dh;
  const float* X;
  const int32_t* bs;
  int B, F, HID;
  WSrc w;
  float* dst;
  int64_t P_pad, o_w, o_b;
  float lr;
  __device__ bool setup(int z, int& M, int& N, int& kb, int& ke) const {
    M = HID; N = F + 1; kb = 0; ke = bs[z];
    return ke > 0;
  }
  __device__ float A(int z, int m, int k) const { return dh[((int64_t)z * B + k) * HID + m]; }
  __device__ float Bv(int z, int n, int k) const { return n < F ? X[((int64_t)z * B + k) * F + n] : 1.f; }
  __device__ void store(int z, int m, int n, float v) const {
    const int64_t off = n < F ? o_w + (int64_t)m * F + n : o_b + m;
    dst[(int64_t)z * P_pad + off] = *w.at(z, off) - lr * v;
  }
};

// ReLU + 2x2 max-pool (floor), first maximum in row-major window order (reading A13).
__global__ void k_pool(const float* __restrict__ a, int H, int W, int C, int B, const int32_t* __restrict__ bs,
                       float* __restrict__ p, uint8_t* __restrict__ am) {
  const int s = blockIdx.y, z = s / B, r = s - z * B;
  if (r >= bs[z]) return;
  const int Hp = H / 2, Wp = W / 2, tot = Hp * Wp * C;
  const float* base = a + (int64_t)s * H * W * C;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const int c = e % C, pw = (e / C) % Wp, ph = e / (C * Wp);
    const float* q = base + ((2 * ph) * W + 2 * pw) * C + c;
    float bv = q[0];
    int best = 0;
    float v = q[C];
    if (v > bv) { bv = v; best = 1; }
    v = q[W * C];
    if (v > bv) { bv = v; best = 2; }
    v = q[W * C + C];
    if (v > bv) { bv = v; best = 3; }
    p[(int64_t)s * tot + e] = bv > 0.f ? bv : 0.f;
    am[(int64_t)s * tot + e] = (uint8_t)best;
  }
}

// Backward of pool + ReLU: route dp to the window's argmax if the pooled value > 0.
__global__ void k_unpool(const float* __restrict__ dp, const float* __restrict__ p, const uint8_t* __restrict__ am,
                         int H, int W, int C, int B, const int32_t* __restrict__ bs, float* __restrict__ dY) {
  const int s = blockIdx.y, z = s / B, r = s - z * B;
  if (r >= bs[z]) return;
  const int Hp = H / 2, Wp = W / 2, ptot = Hp * Wp * C, tot = H * W * C;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    const int c = e % C, x = (e / C) % W, y = e / (C * W);
    const int ph = y >> 1, pw = x >> 1;
    float g = 0.f;
    if (ph < Hp && pw < Wp) {
      const int64_t pe = (int64_t)s * ptot + (ph * Wp + pw) * C + c;
      if (am[pe] == ((y & 1) * 2 + (x & 1)) && p[pe] > 0.f) g = dp[pe];
    }
    dY[(int64_t)s * tot + e] = g;
  }
}

// conv1 forward of a 1-channel input (the speech model) fused with bias + ReLU + 2x2 max-pool
// (+ argmax, first maximum in row-major window order, reading A13): one block per active
// sample, the zero-padded plane and the client's 32x25 filter in shared memory, thread =
// (channel c = tid % 32, pooled cells q = tid / 32 + 8j); the pre-pool map is never stored.
__global__ void __launch_bounds__(256) k_c1fwd_pool_1ch(const float* __restrict__ xpack,
                                                        const int32_t* __restrict__ sidx,
                                                        const int32_t* __restrict__ bs, int B, int H0, int W0, WSrc w,
                                                        int64_t o_w, int64_t o_b, float* __restrict__ p1,
                                                        uint8_t* __restrict__ am1) {
  pdl_wait();
  extern __shared__ float xs[];  // [(H0 + 4)][(W0 + 4)] then ws [32][25], wb [32]
  const int s = blockIdx.x, z = s / B, r = s - z * B;
  if (r >= bs[z]) return;
  const int H1 = H0 / 2, W1 = W0 / 2, PW = W0 + 4, NP = (H0 + 4) * PW;
  float* ws = xs + NP;
  float* wb = ws + 32 * 25;
  const float* xr = xpack + (int64_t)sidx[s] * H0 * W0;
  for (int e = threadIdx.x; e < NP; e += blockDim.x) {
    const int yy = e / PW - 2, xx = e % PW - 2;
    xs[e] = (yy >= 0 && yy < H0 && xx >= 0 && xx < W0) ? xr[yy * W0 + xx] : 0.f;
  }
  for (int e = threadIdx.x; e < 32 * 25; e += blockDim.x) ws[e] = *w.at(z, o_w + e);
  if (threadIdx.x < 32) wb[threadIdx.x] = *w.at(z, o_b + threadIdx.x);
  __syncthreads();
  const int c = threadIdx.x & 31;
  float wr[25];
#pragma unroll
  for (int t = 0; t < 25; ++t) wr[t] = ws[c * 25 + t];
  const float bias = wb[c];
  for (int q = threadIdx.x >> 5; q < H1 * W1; q += 8) {
    const int y0 = 2 * (q / W1), x0 = 2 * (q % W1);
    float v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float* xp = xs + (y0 + (u >> 1)) * PW + x0 + (u & 1);
      float a = bias;
#pragma unroll
      for (int kh = 0; kh < 5; ++kh)
#pragma unroll
        for (int kw = 0; kw < 5; ++kw) a = fmaf(wr[kh * 5 + kw], xp[kh * PW + kw], a);
      v[u] = a;
    }
    float bv = v[0];
    int bi = 0;
#pragma unroll
    for (int u = 1; u < 4; ++u)
      if (v[u] > bv) { bv = v[u]; bi = u; }
    const int64_t o = ((int64_t)s * H1 * W1 + q) * 32 + c;
    p1[o] = bv > 0.f ? bv : 0.f;
    am1[o] = (uint8_t)bi;
  }
}

// conv1 dW of a 1-channel input (the speech model) straight from the pooled gradient: pool1's
// backward routes each pooled cell's (ReLU'-masked) gradient g = dp1m[s][ph][pw][c] to ONE pixel
// (y, x) of its window (the argmax am1), so dW1[c][kh][kw] = Σ g · x[y+kh-2][x+kw-2] and
// db1[c] = Σ g over the pooled cells: a quarter of the dense dY1 work and dY1 never exists.
// Block (chunk ch, client a) = samples [ch·rpc, ch·rpc + rpc) of a's batch; thread = (channel
// c = tid % 32, cell group tid / 32); the 16 groups are summed in fixed order.  Writes the
// chunk's partial [32 c][26] (25 taps + bias) in k_dw_reduce_sgd's [A·nch] chunk layout.
__global__ void __launch_bounds__(512) k_c1dw_pooled(const float* __restrict__ dp1m, const uint8_t* __restrict__ am1,
                                                     const float* __restrict__ xpack, const int32_t* __restrict__ sidx,
                                                     const int32_t* __restrict__ bs, int B, int H0, int W0, int nch,
                                                     int rpc, float* __restrict__ part) {
  constexpr int NG = 16, U = 8;  // cell groups (512 threads / 32 channels); cells whose loads are in flight together
  pdl_wait();
  extern __shared__ float xs[];  // [(H0 + 4)][(W0 + 4)] zero-padded input plane; later [NG][32][26] partials
  const int a = blockIdx.y, ch = blockIdx.x, c = threadIdx.x & 31, gq = threadIdx.x >> 5;
  const int r0 = ch * rpc, r1 = min(r0 + rpc, bs[a]);
  const int H1 = H0 / 2, W1 = W0 / 2, NQ = H1 * W1, PW = W0 + 4, NP = (H0 + 4) * PW;
  float acc[26];
#pragma unroll
  for (int j = 0; j < 26; ++j) acc[j] = 0.f;
  for (int r = r0; r < r1; ++r) {
    const int64_t s = (int64_t)a * B + r;
    const float* xr = xpack + (int64_t)sidx[s] * H0 * W0;
    __syncthreads();  // the previous sample's plane is no longer read
    for (int e = threadIdx.x; e < NP; e += blockDim.x) {
      const int yy = e / PW - 2, xx = e % PW - 2;
      xs[e] = (yy >= 0 && yy < H0 && xx >= 0 && xx < W0) ? xr[yy * W0 + xx] : 0.f;
    }
    __syncthreads();
    const float* dg = dp1m + s * NQ * 32;
    const uint8_t* ag = am1 + s * NQ * 32;
    for (int q0 = gq; q0 < NQ; q0 += NG * U) {
      // issue the U cells' gradient / argmax loads before any use: the loop is latency-bound
      float g[U];
      int am[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = q0 + NG * u;
        g[u] = q < NQ ? __ldg(dg + q * 32 + c) : 0.f;
        am[u] = q < NQ ? __ldg(ag + q * 32 + c) : 0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (g[u] == 0.f) continue;
        const int q = q0 + NG * u;
        const int y = 2 * (q / W1) + (am[u] >> 1), x = 2 * (q % W1) + (am[u] & 1);
        const float* xp = xs + y * PW + x;  // padded (y + kh, x + kw) = pixel (y + kh - 2, x + kw - 2)
#pragma unroll
        for (int kh = 0; kh < 5; ++kh)
#pragma unroll
          for (int kw = 0; kw < 5; ++kw) acc[kh * 5 + kw] = fmaf(g[u], xp[kh * PW + kw], acc[kh * 5 + kw]);
        acc[25] += g[u];
      }
    }
  }
  __syncthreads();
  float* red = xs;  // [NG groups][32 c][26]
#pragma unroll
  for (int j = 0; j < 26; ++j) red[(gq * 32 + c) * 26 + j] = acc[j];
  __syncthreads();
  float* out = part + ((int64_t)a * nch + ch) * 32 * 26;
  for (int e = threadIdx.x; e < 32 * 26; e += blockDim.x) {
    float v = 0.f;
    for (int gg = 0; gg < NG; ++gg) v += red[gg * 32 * 26 + e];  // fixed order
    out[e] = v;
  }
}

// Σ of the split-K partials, then fused SGD on the conv weights and bias.
// Partials: [A*nch] chunks of rpc samples (bpre == nullptr), or the balanced split-K layout
// (bpre != nullptr): client a's partials are z = a + c for the CTAs c0..c1 covering its k-blocks
// [kbps·bpre[a], kbps·bpre[a+1]) of U, split evenly over G CTAs.
__global__ void k_dw_reduce_sgd(const float* __restrict__ part, int nch, int rpc, const int32_t* __restrict__ bs,
                                int O, int N, WSrc w, int64_t o_w, int64_t o_b, float* dst, int64_t P_pad, float lr,
                                const int32_t* __restrict__ bpre, int G, int64_t U, int kbps) {
  pdl_wait();  // (PDL) previous kernel's writes visible; the implicit trigger is at exit
  const int a = blockIdx.y;
  const int tot = O * N;
  const float* pa;
  int nvalid;
  if (bpre) {
    const int64_t v0 = (int64_t)kbps * bpre[a], v1 = (int64_t)kbps * bpre[a + 1] - 1;
    const int c0 = (int)(((v0 + 1) * G + U - 1) / U) - 1, c1 = (int)(((v1 + 1) * G + U - 1) / U) - 1;
    pa = part + (int64_t)(a + c0) * tot;
    nvalid = c1 - c0 + 1;
  } else {
    pa = part + (int64_t)a * nch * tot;
    nvalid = (bs[a] + rpc - 1) / rpc;
  }
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += gridDim.x * blockDim.x) {
    float g = 0.f;
    g = ordered_sum(pa + e, nvalid, tot);
    const int m = e / N, n = e - m * N;
    const int64_t off = n < N - 1 ? o_w + (int64_t)m * (N - 1) + n : o_b + m;
    const float nv = *w.at(a, off) - lr * g;
    dst[(int64_t)a * P_pad + off] = nv;
  }
}

// Both tensor-core dW reductions of a wave in one launch (conv1: blocks [0, r1.nblk), conv2:
// the rest): the same ordered sum + SGD as k_dw_reduce_sgd's balanced split-K branch, one
// launch fewer per wave.  conv1 also writes the forward's tap-major copy (r1.wt).
struct DwRed {
  const float* part;
  int O, N;
  int64_t o_w, o_b;
  int G;
  int64_t U;
  int kbps, nblk;
};
// fc2 (classifier) SGD folded into the wave's final reduction launch: W2[q][n] -= η Σ_r dz[r][q] h[r][n],
// b2[q] -= η Σ_r dz[r][q] (the same fmaf chain in r as k_head_sgd).  Nothing reads W2 between the
// head's forward and the end of the wave, so the update can wait until here.
struct HeadSgd {
  const float* h;       // [slots][HID] fc1 activations of the wave
  const float* dz;      // [slots][NCLS] softmax-CE gradient of the logits
  const int32_t* bs;
  int B, HID, NCLS;
  int64_t o_w, o_b;
  int nblk;
};
__global__ void __launch_bounds__(256) k_dw_reduce2_sgd(DwRed r1, DwRed r2, HeadSgd hd, const int32_t* __restrict__ bpre,
                                                        WSrc w, float* dst, int64_t P_pad, float lr) {
  pdl_wait();
  if ((int)blockIdx.x >= r1.nblk + r2.nblk) {  // fc2 SGD
    const int a = blockIdx.y, b = hd.bs[a];
    const int e = ((int)blockIdx.x - r1.nblk - r2.nblk) * blockDim.x + threadIdx.x;
    const float* dzz = hd.dz + (int64_t)a * hd.B * hd.NCLS;
    const float* hz = hd.h + (int64_t)a * hd.B * hd.HID;
    if (e < hd.NCLS * hd.HID) {
      const int q = e / hd.HID, n = e - q * hd.HID;
      float g = 0.f;
      for (int r = 0; r < b; ++r) g = fmaf(__ldg(dzz + r * hd.NCLS + q), __ldg(hz + (int64_t)r * hd.HID + n), g);
      dst[(int64_t)a * P_pad + hd.o_w + e] = *w.at(a, hd.o_w + e) - lr * g;
    } else if (e < hd.NCLS * hd.HID + hd.NCLS) {
      const int q = e - hd.NCLS * hd.HID;
      float g = 0.f;
      for (int r = 0; r < b; ++r) g += __ldg(dzz + r * hd.NCLS + q);
      dst[(int64_t)a * P_pad + hd.o_b + q] = *w.at(a, hd.o_b + q) - lr * g;
    }
    return;
  }
  const bool second = (int)blockIdx.x >= r1.nblk;
  const DwRed& r = second ? r2 : r1;
  const int bx = second ? (int)blockIdx.x - r1.nblk : (int)blockIdx.x;
  const int a = blockIdx.y, tot = r.O * r.N;
  const int64_t v0 = (int64_t)r.kbps * bpre[a], v1 = (int64_t)r.kbps * bpre[a + 1] - 1;
  const int c0 = (int)(((v0 + 1) * r.G + r.U - 1) / r.U) - 1, c1 = (int)(((v1 + 1) * r.G + r.U - 1) / r.U) - 1;
  const float* pa = r.part + (int64_t)(a + c0) * tot;
  for (int e = bx * blockDim.x + threadIdx.x; e < tot; e += r.nblk * blockDim.x) {
    const float g = ordered_sum(pa + e, c1 - c0 + 1, tot);
    const int m = e / r.N, n = e - m * r.N;
    const int64_t off = n < r.N - 1 ? r.o_w + (int64_t)m * (r.N - 1) + n : r.o_b + m;
    const float nv = *w.at(a, off) - lr * g;
    dst[(int64_t)a * P_pad + off] = nv;
  }
}

// Classifier head, forward half, parallel over (client, chunk of HR batch rows): logits =
// h·W2ᵀ + b2, softmax-CE (mean over |b|, reading A9), dz = (p − onehot)/|b| -> dzbuf,
// dh = (dz·W2) ⊙ [h > 0]; rows past |b| get dz = dh = 0.  Reads W2 before the update.
constexpr int HR = 4;
__global__ void __launch_bounds__(256) k_head_fwd(const float* __restrict__ h, const int32_t* __restrict__ ypack,
                                                  const int32_t* __restrict__ sidx, const int32_t* __restrict__ bs,
                                                  int B, int HID, int NCLS, WSrc w, int64_t o_w, int64_t o_b,
                                                  float* __restrict__ dzbuf, float* __restrict__ dh) {
  pdl_wait();  // (PDL) previous kernel's writes visible; the implicit trigger is at exit
  extern __shared__ float sm[];
  const int z = blockIdx.x, r0 = blockIdx.y * HR, b = bs[z];
  if (r0 >= B) return;
  float* Ws = sm;                  // [NCLS][HID]
  float* zs = Ws + NCLS * HID;     // [HR][NCLS]
  float* hs = zs + HR * NCLS;      // [HR][HID] staged activations
  const int nr = max(0, min(HR, b - r0));
  if (nr > 0) {
    // every global load issued before any store (one round trip), then compute from smem
    const float4* W4 = reinterpret_cast<const float4*>(w.at(z, o_w));
    const float4* h4 = reinterpret_cast<const float4*>(h + ((int64_t)z * B + r0) * HID);
    const int nw4 = NCLS * HID / 4, nh4 = nr * HID / 4;
    for (int base = 0; base < nw4 + nh4; base += 12 * 256) {
      float4 v[12];
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const int e = base + threadIdx.x + i * 256;
        if (e < nw4) v[i] = __ldg(W4 + e);
        else if (e < nw4 + nh4) v[i] = __ldg(h4 + (e - nw4));
      }
#pragma unroll
      for (int i = 0; i < 12; ++i) {
        const int e = base + threadIdx.x + i * 256;
        if (e < nw4) reinterpret_cast<float4*>(Ws)[e] = v[i];
        else if (e < nw4 + nh4) reinterpret_cast<float4*>(hs)[e - nw4] = v[i];
      }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int idx = warp; idx < nr * NCLS; idx += nw) {
      const int rr = idx / NCLS, q = idx - rr * NCLS;
      const float* hr = hs + rr * HID;
      float s = 0.f;
      for (int n = lane; n < HID; n += 32) s = fmaf(Ws[q * HID + n], hr[n], s);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) zs[rr * NCLS + q] = s + *w.at(z, o_b + q);
    }
    __syncthreads();
    if (threadIdx.x < nr) {
      float* zr = zs + threadIdx.x * NCLS;
      const int y = ypack[sidx[z * B + r0 + threadIdx.x]];
      float mx = zr[0];
      for (int q = 1; q < NCLS; ++q) mx = fmaxf(mx, zr[q]);
      float s = 0.f;
      for (int q = 0; q < NCLS; ++q) s += expf(zr[q] - mx);
      const float inv = 1.f / (float)b;
      for (int q = 0; q < NCLS; ++q) zr[q] = (expf(zr[q] - mx) / s - (q == y ? 1.f : 0.f)) * inv;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < HR * NCLS; e += blockDim.x) {
    const int rr = e / NCLS;
    if (r0 + rr < B) dzbuf[((int64_t)z * B + r0) * NCLS + e] = rr < nr ? zs[e] : 0.f;
  }
  for (int e = threadIdx.x; e < HR * HID; e += blockDim.x) {
    const int rr = e / HID, n = e - rr * HID;
    if (r0 + rr >= B) continue;
    const int64_t hi = ((int64_t)z * B + r0 + rr) * HID + n;
    float s = 0.f;
    if (rr < nr) {
      for (int q = 0; q < NCLS; ++q) s = fmaf(Ws[q * HID + n], zs[rr * NCLS + q], s);
      s = hs[rr * HID + n] > 0.f ? s : 0.f;
    }
    dh[hi] = s;
  }
}

// Classifier head, update half, parallel over (client, 64-column chunk): W2 <- W2 − η·dzᵀh,
// b2 <- b2 − η·Σ_r dz (chunk 0).
__global__ void __launch_bounds__(256) k_head_sgd(const float* __restrict__ h, const float* __restrict__ dzbuf,
                                                  const int32_t* __restrict__ bs, int B, int HID, int NCLS, WSrc w,
                                                  int64_t o_w, int64_t o_b, float* dst, int64_t P_pad, float lr) {
  pdl_wait();  // (PDL) previous kernel's writes visible; the implicit trigger is at exit
  extern __shared__ float sm[];
  const int z = blockIdx.x, n0 = blockIdx.y * 64, b = bs[z];
  if (b == 0) return;
  float* dzs = sm;                 // [b][NCLS]
  float* hs = dzs + B * NCLS;      // [b][64] columns n0.. of h
  float* Wd = dst + (int64_t)z * P_pad;
  const float* dzz = dzbuf + (int64_t)z * B * NCLS;
  const float* hz = h + (int64_t)z * B * HID;
  {  // all loads in flight before any store: dz (<= B*NCLS) and the h column chunk (<= B*64)
    constexpr int LZ = 2, LH = 8;
    float zv[LZ], hv[LH];
#pragma unroll
    for (int i = 0; i < LZ; ++i) {
      const int e = threadIdx.x + i * 256;
      zv[i] = e < b * NCLS ? __ldg(dzz + e) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < LH; ++i) {
      const int e = threadIdx.x + i * 256, r = e >> 6, n = n0 + (e & 63);
      hv[i] = (e < b * 64 && n < HID) ? __ldg(hz + (int64_t)r * HID + n) : 0.f;
    }
#pragma unroll
    for (int i = 0; i < LZ; ++i)
      if (threadIdx.x + i * 256 < b * NCLS) dzs[threadIdx.x + i * 256] = zv[i];
#pragma unroll
    for (int i = 0; i < LH; ++i)
      if (threadIdx.x + i * 256 < b * 64) hs[threadIdx.x + i * 256] = hv[i];
    for (int e = threadIdx.x + LZ * 256; e < b * NCLS; e += blockDim.x) dzs[e] = dzz[e];  // B*NCLS > 512
    for (int e = threadIdx.x + LH * 256; e < b * 64; e += blockDim.x) {                   // B > 32
      const int r = e >> 6, n = n0 + (e & 63);
      hs[e] = n < HID ? hz[(int64_t)r * HID + n] : 0.f;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NCLS * 64; e += blockDim.x) {
    const int q = e / 64, nl = e & 63, n = n0 + nl;
    if (n >= HID) continue;
    float g = 0.f;
    for (int r = 0; r < b; ++r) g = fmaf(dzs[r * NCLS + q], hs[r * 64 + nl], g);
    Wd[o_w + q * HID + n] = *w.at(z, o_w + q * HID + n) - lr * g;
  }
  if (blockIdx.y == 0 && threadIdx.x < NCLS) {
    const int q = threadIdx.x;
    float g = 0.f;
    for (int r = 0; r < b; ++r) g += dzs[r * NCLS + q];
    Wd[o_b + q] = *w.at(z, o_b + q) - lr * g;
  }
}

template <class Op>
void launch(const Op& op, int Mmax, int Nmax, int Z, cudaStream_t st) {
  const bool nm = Mmax <= 32, nn = Nmax <= 32;
  dim3 grid((Mmax + (nm ? 31 : 63)) / (nm ? 32 : 64), (Nmax + (nn ? 31 : 63)) / (nn ? 32 : 64), Z);
  if (nm && nn) k_gemm<Op, 32, 32><<<grid, NT, 0, st>>>(op);
  else if (nm) k_gemm<Op, 32, 64><<<grid, NT, 0, st>>>(op);
  else if (nn) k_gemm<Op, 64, 32><<<grid, NT, 0, st>>>(op);
  else k_gemm<Op, 64, 64><<<grid, NT, 0, st>>>(op);
}

}  // namespace

int cnn_wave_simt(const Layout& L, const WaveArgs& wa, const float* xpack, const int32_t* ypack,
                  const float* theta_g, float* slots, CnnBufs& b, cudaStream_t st) {
  const CnnDims& d = L.d;
  const int A = wa.A, B = wa.B;
  const WSrc w{wa.first ? theta_g : slots, wa.first ? 0 : L.P_pad};
  KProf& pf = *wa.prof;
  const double S = (double)wa.sum_bs, hw0 = (double)d.H0 * d.W0, hw1 = (double)d.H1 * d.W1;
  // algorithmic FLOPs of each GEMM (conv1 K = 25*cin, not the padded 25*cpad)
  const double f_c1 = 2.0 * S * hw0 * d.C1 * 25 * d.cin, f_c2 = 2.0 * S * hw1 * d.C2 * 25 * d.C1,
               f_f1 = 2.0 * S * d.HID * d.F, f_f2 = 2.0 * S * d.NCLS * d.HID;
  const double wbytes = 4.0 * (double)A * (double)d.HID * d.F;  // one pass over the fc1 weights
  int n = 0;
  // ---- forward
  const bool tc1 = wa.use_tc && conv1_tc_supported(L);
  pf.begin(st);
  if (tc1) {  // bias + ReLU + pool fused into the epilogue
    if (conv1_fwd_tc(L, wa, w.base, w.stride, b.xg, b.xrows, b.slots, b.p1, b.am1, st) < 0) return -1;
    ++n;
    pf.end(K_CONV1_FWD, f_c1, 4.0 * S * hw0 * d.cin + 5.0 * S * hw1 * d.C1, st);
  } else if (wa.use_tc && d.cin == 1 && d.C1 == 32) {  // speech: conv1 + bias + ReLU + pool in one pass
    const size_t sm = sizeof(float) * ((d.H0 + 4) * (d.W0 + 4) + 32 * 25 + 32);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_c1fwd_pool_1ch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr = true;
    }
    launch_pdl(wa.pdl, k_c1fwd_pool_1ch, dim3(A * B), 256, sm, st, xpack, wa.sidx, wa.bs, B, d.H0, d.W0, w, L.o_c1w,
               L.o_c1b, b.p1, b.am1), ++n;
    pf.end(K_CONV1_FWD, f_c1, 4.0 * S * hw0 * d.cin + 5.0 * S * hw1 * d.C1, st);
  } else {
    launch(ConvFwd{xpack, wa.sidx, wa.bs, B, d.H0, d.W0, d.cpad, d.C1, w, L.o_c1w, L.o_c1b, b.a1},
           B * d.H0 * d.W0, d.C1, A, st), ++n;
    pf.end(K_CONV1_FWD, f_c1, 4.0 * S * hw0 * (d.cin + d.C1), st);
    pf.begin(st);
    k_pool<<<dim3(8, A * B), 256, 0, st>>>(b.a1, d.H0, d.W0, d.C1, B, wa.bs, b.p1, b.am1), ++n;
    pf.end(K_POOL1, 0, S * hw0 * d.C1 * (4.0 + 5.0 / 4.0), st);
  }
  const bool tc = wa.use_tc && conv_tc_supported(L);
  const int64_t wcl = wa.first ? 1 : wa.wclients;
  if (tc) {  // tcgen05 implicit GEMM with fused bias + ReLU + pool epilogue
    pf.begin(st);
    if (conv2_fwd_tc(L, wa, w.base, wcl, b.p1, b.slots, b.p2, b.am2, st) < 0) return -1;
    ++n;
    pf.end(K_CONV2_FWD, f_c2, 4.0 * S * hw1 * d.C1 + 5.0 * S * hw1 * d.C2 / 4.0, st);
  } else {
    pf.begin(st);
    launch(ConvFwd{b.p1, nullptr, wa.bs, B, d.H1, d.W1, d.C1, d.C2, w, L.o_c2w, L.o_c2b, b.a2},
           B * d.H1 * d.W1, d.C2, A, st), ++n;
    pf.end(K_CONV2_FWD, f_c2, 4.0 * S * hw1 * (d.C1 + d.C2), st);
    pf.begin(st);
    k_pool<<<dim3(4, A * B), 256, 0, st>>>(b.a2, d.H1, d.W1, d.C2, B, wa.bs, b.p2, b.am2), ++n;
    pf.end(K_POOL2, 0, S * hw1 * d.C2 * (4.0 + 5.0 / 4.0), st);
  }
  const bool tcf = wa.use_tc && fc1_tc_supported(L, B);
  pf.begin(st);
  if (tcf) {
    int nl = 0;
    if (fc1_fwd_tc(L, wa, w.base, wa.first ? 1 : wa.wclients, b.p2, b.slots, b.h, b.fc1_part, b.fc1_part_floats, st,
                   &nl) < 0)
      return -1;
    n += nl;
  } else {
    // split K when the wave is small: about 4 waves of 64-wide blocks over the GPU
    const int nb = (d.HID + 63) / 64;
    int S = (int)std::min<int64_t>(16, std::max<int64_t>(1, (4 * 148 + (int64_t)A * nb - 1) / ((int64_t)A * nb)));
    while (S > 1 && (int64_t)A * S * B * d.HID > b.fc1_part_floats) --S;
    if (S > 1) {
      launch(FcFwdPart{b.p2, wa.bs, B, d.F, d.HID, S, w, L.o_f1w, b.fc1_part}, B, d.HID, A * S, st), ++n;
      k_fc_fwd_reduce<<<dim3(B, A), 256, 0, st>>>(b.fc1_part, wa.bs, B, d.HID, S, w, L.o_f1b, b.h), ++n;
    } else {
      launch(FcFwd{b.p2, wa.bs, B, d.F, d.HID, w, L.o_f1w, L.o_f1b, b.h}, B, d.HID, A, st), ++n;
    }
  }
  pf.end(K_FC1_FWD, f_f1, wbytes + 4.0 * S * (d.F + d.HID), st);
  const size_t hsm = sizeof(float) * (size_t)(d.NCLS * d.HID + HR * d.NCLS + HR * d.HID);
  static size_t hsm_set = 0;
  if (hsm > hsm_set) {
    cudaFuncSetAttribute(k_head_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    hsm_set = hsm;
  }
  pf.begin(st);
  launch_pdl(wa.pdl, k_head_fwd, dim3(A, (B + HR - 1) / HR), 256, hsm, st, b.h, ypack, wa.sidx, wa.bs, B, d.HID, d.NCLS, w, L.o_f2w,
                                                          L.o_f2b, b.dz, b.dh), ++n;
  // the CIFAR tensor-core path does the fc2 SGD in the wave's final reduction (k_dw_reduce2_sgd)
  const bool fold_head_sgd = wa.use_tc && conv_tc_supported(L) && conv1_tc_supported(L);
  if (!fold_head_sgd)
    launch_pdl(wa.pdl, k_head_sgd, dim3(A, (d.HID + 63) / 64), 256, sizeof(float) * B * (d.NCLS + 64), st, b.h, b.dz,
               wa.bs, B, d.HID, d.NCLS, w, L.o_f2w, L.o_f2b, slots, L.P_pad, wa.lr), ++n;
  pf.end(K_HEAD, 3.0 * f_f2, 8.0 * A * d.NCLS * d.HID + 8.0 * S * d.HID, st);
  // ---- backward (each layer's dX reads W before its dW epilogue overwrites it)
  pf.begin(st);
  if (tcf) {  // one W1 pass: dX (+ pool2/ReLU backward -> dY2), dW, SGD
    if (fc1_bwd_tc(L, wa, w.base, wa.first ? 1 : wa.wclients, slots, wa.wclients, b.dh, b.p2, b.am2, b.slots, b.dY2,
                   st) < 0)
      return -1;
    ++n;
    pf.end(K_FC1_DW, 2.0 * f_f1, 2.0 * wbytes + 4.0 * S * (d.F + d.HID) + S * hw1 * d.C2 * (9.0 / 4.0), st);
  } else {
    launch(FcDx{b.dh, wa.bs, B, d.F, d.HID, w, L.o_f1w, b.dp2}, B, d.F, A, st), ++n;
    pf.end(K_FC1_DX, f_f1, wbytes + 4.0 * S * (d.F + d.HID), st);
    pf.begin(st);
    k_unpool<<<dim3(4, A * B), 256, 0, st>>>(b.dp2, b.p2, b.am2, d.H1, d.W1, d.C2, B, wa.bs, b.dY2), ++n;
    pf.end(K_UNPOOL2, 0, S * hw1 * d.C2 * (4.0 + 9.0 / 4.0), st);
    pf.begin(st);
    launch(FcDwSgd{b.dh, b.p2, wa.bs, B, d.F, d.HID, w, slots, L.P_pad, L.o_f1w, L.o_f1b, wa.lr}, d.HID, d.F + 1, A,
           st), ++n;
    pf.end(K_FC1_DW, f_f1, 2.0 * wbytes + 4.0 * S * (d.F + d.HID), st);
  }
  pf.begin(st);
  if (tc) {  // pool1/ReLU backward fused into the epilogue: writes dY1 directly
    if (conv2_dx_tc(L, wa, w.base, wcl, b.dY2, b.slots, b.p1, b.dp1, st) < 0) return -1;
    ++n;
    pf.end(K_CONV2_DX, f_c2, 4.0 * S * hw1 * (d.C2 + 2.0 * d.C1), st);  // dY2, p1 in; dp1m out
  } else {
    launch(ConvDx{b.dY2, wa.bs, B, d.H1, d.W1, d.C1, d.C2, w, L.o_c2w, b.dp1}, B * d.H1 * d.W1, d.C1, A, st), ++n;
    pf.end(K_CONV2_DX, f_c2, 4.0 * S * hw1 * (d.C1 + d.C2), st);
    pf.begin(st);
    k_unpool<<<dim3(8, A * B), 256, 0, st>>>(b.dp1, b.p1, b.am1, d.H0, d.W0, d.C1, B, wa.bs, b.dY1), ++n;
    pf.end(K_UNPOOL1, 0, S * hw0 * d.C1 * (4.0 + 9.0 / 4.0), st);
  }
  const int rpc = (B + b.nch - 1) / b.nch;
  if (tc && tc1) {  // both dW GEMMs on tcgen05, then one launch reduces both (ordered sums + SGD)
    int g2 = 0, g1 = 0;
    pf.begin(st);
    if (conv2_dw_tc(L, wa, b.p1, b.dY2, b.slots, b.part2, b.part2_tc_cap, &g2, st) < 0) return -1;
    ++n;
    pf.end(K_CONV2_DW, f_c2, 4.0 * S * hw1 * (d.C1 + d.C2), st);
    pf.begin(st);
    if (conv1_dw_tc(L, wa, b.xg, b.xrows, b.dp1, b.am1, b.slots, b.part1, b.part1_tc_cap, &g1, st) < 0)
      return -1;
    ++n;
    pf.end(K_CONV1_DW, f_c1, 4.0 * S * hw0 * d.cin + 5.0 * S * hw1 * d.C1, st);
    const int N2 = 25 * d.C1 + 1, N1 = 25 * d.cpad + 1;
    DwRed r1{b.part1, d.C1, N1, L.o_c1w, L.o_c1b, g1, 2 * wa.sum_bs, 2, (d.C1 * N1 + 255) / 256};  // half-sample tiles
    const int kps2 = conv2_dw_kps(L);
    DwRed r2{b.part2, d.C2, N2, L.o_c2w, L.o_c2b, g2, (int64_t)kps2 * wa.sum_bs, kps2, (d.C2 * N2 + 255) / 256};
    HeadSgd hd{b.h, b.dz, wa.bs, B, d.HID, d.NCLS, L.o_f2w, L.o_f2b, (d.NCLS * d.HID + d.NCLS + 255) / 256};
    pf.begin(st);
    launch_pdl(wa.pdl, k_dw_reduce2_sgd, dim3(r1.nblk + r2.nblk + hd.nblk, A), 256, 0, st, r1, r2, hd, wa.bpre, w, slots,
               L.P_pad, wa.lr), ++n;
    pf.end(K_CONV2_DWR, 0, 8.0 * A * (d.C2 * 25 * d.C1 + d.C1 * 25 * d.cin), st);
    return n;
  }
  if (tc) {  // tcgen05 dW with all 800 (tap, c) rows resident in TMEM; SGD in the reduction
    int g2 = 0;
    pf.begin(st);
    if (conv2_dw_tc(L, wa, b.p1, b.dY2, b.slots, b.part2, b.part2_tc_cap, &g2, st) < 0) return -1;
    ++n;
    pf.end(K_CONV2_DW, f_c2, 4.0 * S * hw1 * (d.C1 + d.C2), st);
    pf.begin(st);
    if (conv2_dw_reduce_tc(L, wa, w.base, w.stride, slots, b.part2, g2, st) < 0) return -1;
    ++n;
    pf.end(K_CONV2_DWR, 0, 8.0 * A * d.C2 * 25 * d.C1, st);
  } else {
    pf.begin(st);
    launch(ConvDw{b.dY2, b.p1, nullptr, wa.bs, B, d.H1, d.W1, d.C1, d.C2, b.nch, rpc, b.part2}, d.C2,
           25 * d.C1 + 1, A * b.nch, st), ++n;
    pf.end(K_CONV2_DW, f_c2, 4.0 * S * hw1 * (d.C1 + d.C2), st);
    pf.begin(st);
    launch_pdl(wa.pdl, k_dw_reduce_sgd, dim3(16, A), 256, 0, st, b.part2, b.nch, rpc, wa.bs, d.C2, 25 * d.C1 + 1, w, L.o_c2w,
                                                 L.o_c2b, slots, L.P_pad, wa.lr, nullptr, 0, 0, 0), ++n;
    pf.end(K_CONV2_DWR, 0, 8.0 * A * d.C2 * 25 * d.C1, st);
  }
  int nch1 = b.nch, rpc1 = rpc, g1 = 0;
  const bool pooled_c1dw = tc && !tc1 && d.cin == 1 && d.C1 == 32;  // speech: dW from dp1m + am1 directly
  if (tc && !tc1 && !pooled_c1dw) {  // route the tensor-core dX's dp1m through pool1's argmax -> dY1
    pf.begin(st);
    k_unpool<<<dim3(8, A * B), 256, 0, st>>>(b.dp1, b.p1, b.am1, d.H0, d.W0, d.C1, B, wa.bs, b.dY1), ++n;
    pf.end(K_UNPOOL1, 0, S * hw0 * d.C1 * (4.0 + 9.0 / 4.0), st);
  }
  pf.begin(st);
  if (pooled_c1dw) {
    const size_t sm = sizeof(float) * std::max((d.H0 + 4) * (d.W0 + 4), 16 * 32 * 26);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_c1dw_pooled, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      attr = true;
    }
    launch_pdl(wa.pdl, k_c1dw_pooled, dim3(b.nch, A), 512, sm, st, b.dp1, b.am1, xpack, wa.sidx, wa.bs, B, d.H0,
               d.W0, b.nch, rpc, b.part1), ++n;
  } else if (tc1) {
    if (conv1_dw_tc(L, wa, b.xg, b.xrows, b.dp1, b.am1, b.slots, b.part1, b.part1_tc_cap, &g1, st) < 0)
      return -1;
    ++n;
  } else {
    launch(ConvDw{b.dY1, xpack, wa.sidx, wa.bs, B, d.H0, d.W0, d.cpad, d.C1, b.nch, rpc, b.part1}, d.C1,
           25 * d.cpad + 1, A * b.nch, st), ++n;
  }
  pf.end(K_CONV1_DW, f_c1,
         (tc1 || pooled_c1dw) ? 4.0 * S * hw0 * d.cin + 5.0 * S * hw1 * d.C1 : 4.0 * S * hw0 * (d.cin + d.C1), st);
  pf.begin(st);
  launch_pdl(wa.pdl, k_dw_reduce_sgd, dim3((d.C1 * (25 * d.cpad + 1) + 127) / 128, A), 128, 0, st, 
      b.part1, nch1, rpc1, wa.bs, d.C1, 25 * d.cpad + 1, w, L.o_c1w,
                                              L.o_c1b, slots, L.P_pad, wa.lr,
      tc1 ? wa.bpre : nullptr, g1, 2 * wa.sum_bs, 2), ++n;  // conv1 tensor-core dW: half-sample tiles
  pf.end(K_CONV1_DWR, 0, 8.0 * A * d.C1 * 25 * d.cin, st);
  return n;
}

}  // namespace flb
