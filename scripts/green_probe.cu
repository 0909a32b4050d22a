// Probe: do runtime-API launches into a green-context stream run on the partition's SMs only,
// and can they use cudaMalloc'd (primary-context) memory?  nvcc -arch=sm_100a green_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include <set>
#include <vector>

__global__ void k_smid(int* out, int iters) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  float x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = x * 1.0000001f + 1e-7f;
  if (threadIdx.x == 0) out[blockIdx.x] = (int)s + (x < -1.f ? 1 : 0);
}

template <class F>
F get(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
    printf("no entry point %s\n", name);
    return nullptr;
  }
  return (F)fn;
}

int main(int argc, char** argv) {
  int want = argc > 1 ? atoi(argv[1]) : 48;
  cudaFree(0);
  auto getRes = get<CUresult (*)(CUdevice, CUdevResource*, CUdevResourceType)>("cuDeviceGetDevResource");
  auto split = get<CUresult (*)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned, unsigned)>(
      "cuDevSmResourceSplitByCount");
  auto gen = get<CUresult (*)(CUdevResourceDesc*, CUdevResource*, unsigned)>("cuDevResourceGenerateDesc");
  auto gcreate = get<CUresult (*)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned)>("cuGreenCtxCreate");
  auto gstream = get<CUresult (*)(CUstream*, CUgreenCtx, unsigned, int)>("cuGreenCtxStreamCreate");
  CUdevResource all, part, rem;
  printf("getRes %d\n", (int)getRes(0, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SMs %u\n", all.sm.smCount);
  unsigned nb = 1;
  CUresult r = split(&part, &nb, &all, &rem, 0, (unsigned)want);
  printf("split %d groups %u part SMs %u remainder %u\n", (int)r, nb, part.sm.smCount, rem.sm.smCount);
  CUdevResourceDesc desc;
  printf("gen %d\n", (int)gen(&desc, &part, 1));
  CUgreenCtx g;
  printf("gcreate %d\n", (int)gcreate(&g, desc, 0, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s;
  printf("gstream %d\n", (int)gstream(&s, g, CU_STREAM_NON_BLOCKING, 0));
  int* d;
  cudaMalloc(&d, 4096 * 4);
  const int nblk = 2048;
  for (int rep = 0; rep < 2; ++rep) {
    cudaStream_t st = rep == 0 ? (cudaStream_t)s : nullptr;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    k_smid<<<nblk, 256, 0, st>>>(d, 20000);
    cudaEventRecord(b, st);
    cudaError_t e = cudaStreamSynchronize(st);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    std::vector<int> h(nblk);
    cudaMemcpy(h.data(), d, nblk * 4, cudaMemcpyDeviceToHost);
    std::set<int> sms(h.begin(), h.end());
    printf("%s: err=%s distinct SMs=%zu time %.3f ms\n", rep == 0 ? "green stream" : "default stream",
           cudaGetErrorString(e), sms.size(), ms);
  }
  return 0;
}
