// tc_probe.cu — standalone check of tcgen05 kind::tf32 descriptor conventions.
// D[128 x N] = A[128 x 32] · B, A K-major (SW128), B either K-major ([N][32]) or MN-major
// ([32 k][N]) staged by plain stores into the SW128 pattern (no TMA).  Prints max error
// vs a host reference for several LBO/SBO/mode variants.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include "../paper_2306_17453_b200/csrc/tc_common.cuh"
using namespace flb;

// byte offset of (row, 16B chunk) inside a SW128 tile of 128-byte rows
__device__ int sw128(int row, int chunk) { return row * 128 + ((chunk ^ (row & 7)) * 16); }
// Swizzle<2,5,2>: 32-byte granules XOR (row & 3); byte offset of (row, byte-in-row)
__device__ int sw128_32b(int row, int byte) { return row * 128 + ((((byte >> 5) ^ (row & 3)) << 5) | (byte & 31)); }

template <int N, int BMN>
__global__ void probe(const float* A, const float* Bm, float* D, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;                 // 128 rows x 128 B
  uint8_t* sb = smem + 128 * 128;     // K-major: N rows x 128B ; MN-major: 32 k-rows x (N/32 chunks of 128B) with LBO between chunks
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  int t = threadIdx.x;
  // A: row m, k in [0,32): element (m,k) at chunk k/4, offset k%4
  for (int e = t; e < 128 * 32; e += blockDim.x) {
    int m = e / 32, k = e % 32;
    *(float*)(sa + sw128(m, k / 4) + (k % 4) * 4) = A[m * 32 + k];
  }
  for (int e = t; e < N * 32; e += blockDim.x) {
    int n = e / 32, k = e % 32;   // B(n,k)
    float v = Bm[n * 32 + k];
    if (BMN == 0) *(float*)(sb + sw128(n, k / 4) + (k % 4) * 4) = v;
    else if (BMN == 2) *(float*)(sb + sw128_32b(n, k * 4)) = v;  // K-major rows in the BASE32B pattern
    else {
      int chunk = n / 32, nn = n % 32;  // MN chunk of 32 elements
      *(float*)(sb + chunk * lbo + sw128_32b(k, nn * 4)) = v;
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (t < 32) {
    if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
    __syncwarp();
    tc::tmem_alloc<256>(&tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  uint32_t tb = tslot;
  if (t == 0) {
    constexpr uint32_t ID = tc::idesc_tf32(128, N, 0, BMN == 1 ? 1 : 0);
    for (int k = 0; k < 4; ++k) {
      uint64_t ad = tc::sdesc(tc::smem_u32(sa) + k * 32, 0, 1024, tc::kSW128);
      uint64_t bd = BMN == 1 ? tc::sdesc(tc::smem_u32(sb) + k * 1024, lbo, sbo, 1)
                  : BMN == 2 ? tc::sdesc(tc::smem_u32(sb) + k * 32, lbo, sbo, 1)
                             : tc::sdesc(tc::smem_u32(sb) + k * 32, 0, 1024, tc::kSW128);
      tc::mma_tf32(tb, ad, bd, ID, k > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  int w = t / 32;
  for (int n0 = 0; n0 < N; n0 += 16) {
    float v[16];
    tc::tmem_ld16(tb + ((uint32_t)(w * 32) << 16) + n0, v);
    for (int j = 0; j < 16; ++j) D[(w * 32 + (t & 31)) * N + n0 + j] = v[j];
  }
  tc::tc_fence_before();
  __syncthreads();
  if (t < 32) tc::tmem_dealloc<256>(tb);
}

template <int N, int BMN>
void run(uint32_t lbo, uint32_t sbo) {
  float *A, *Bm, *D;
  if (cudaMallocManaged(&A, 128 * 32 * 4) != cudaSuccess) { printf("context dead\n"); exit(1); }
  cudaMallocManaged(&Bm, N * 32 * 4);
  cudaMallocManaged(&D, 128 * N * 4);
  for (int i = 0; i < 128 * 32; ++i) A[i] = (float)((i * 37 % 17) - 8) / 8.f;
  for (int i = 0; i < N * 32; ++i) Bm[i] = (float)((i * 11 % 13) - 6) / 4.f;
  cudaMemset(D, 0, 128 * N * 4);
  probe<N, BMN><<<1, 128, 64 * 1024>>>(A, Bm, D, lbo, sbo);
  cudaError_t e = cudaDeviceSynchronize();
  double err = 0, mx = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < 32; ++k) r += (double)A[m * 32 + k] * Bm[n * 32 + k];
      err = fmax(err, fabs(r - D[m * N + n]));
      mx = fmax(mx, fabs(r));
    }
  printf("N=%d BMN=%d lbo=%u sbo=%u: %s max_err=%.3g (max |ref| %.3g) D[0]=%g D[1]=%g\n", N, BMN, lbo, sbo,
         cudaGetErrorString(e), err, mx, D[0], D[1]);
  cudaFree(A); cudaFree(Bm); cudaFree(D);
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  if (argc > 1) {  // one K-major BASE32B variant per process (a bad descriptor faults the context)
    cudaFuncSetAttribute(probe<32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    run<32, 2>((uint32_t)atoi(argv[1]), (uint32_t)atoi(argv[2]));
    return 0;
  }
  cudaFuncSetAttribute(probe<64, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(probe<32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaFuncSetAttribute(probe<64, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  run<64, 0>(0, 1024);
  run<32, 1>(4096, 512);
  run<32, 1>(4096, 1024);
  run<64, 1>(4096, 512);
  run<64, 1>(8192, 512);
  return 0;
}
