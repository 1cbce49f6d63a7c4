// Where does the block scheduler put a 48-CTA kernel (one CTA per SM, 216 KB
// smem) on an idle B200, and where does a second one go while the first is
// still resident?  Also times a streaming HBM copy by each placement.  Used
// to study why an early PDL trigger slows the bulk-copy all-reduce.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/smid_probe tools/smid_probe.cu
//   tools/_build/smid_probe [ctas=48] [peer=0]   (peer=1: read a buffer on GPU 1 over NVLink)
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__global__ void hold(unsigned* ids, volatile int* release, int* started) {
  extern __shared__ char s[];
  if (threadIdx.x == 0) {
    ids[blockIdx.x] = smid();
    s[0] = 0;
    __threadfence_system();
    atomicAdd_system(started, 1);
    while (*release == 0) __nanosleep(1000);
  }
}

__global__ void copy(unsigned* ids, const float4* src, float4* dst, size_t n) {
  extern __shared__ char s[];
  if (threadIdx.x == 0) ids[blockIdx.x] = smid(), s[0] = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int main(int argc, char** argv) {
  const int ctas = argc > 1 ? atoi(argv[1]) : 48;
  const size_t smem = 216 * 1024;
  cudaFuncSetAttribute(hold, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(copy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  unsigned *ida, *idb, *idc;
  int* rel;
  cudaMalloc(&ida, 4096);
  cudaMalloc(&idb, 4096);
  cudaMalloc(&idc, 4096);
  cudaMallocManaged(&rel, 4);
  const size_t n = (size_t)256 << 20 >> 4;  // 256 MiB of float4
  float4 *src, *dst;
  cudaMalloc(&src, n * 16);
  cudaMalloc(&dst, n * 16);
  cudaMemset(src, 1, n * 16);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed_copy = [&](unsigned* ids) {
    float best = 1e9f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0, s2);
      copy<<<ctas, 512, smem, s2>>>(ids, src, dst, n);
      cudaEventRecord(e1, s2);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return 2.0 * n * 16 / (best * 1e-3) / 1e9;
  };
  // optional: the copy reads a PEER GPU's buffer (NVLink) instead of local HBM
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  const bool peer = argc > 2 && atoi(argv[2]) != 0 && ndev > 1;
  if (peer) {
    cudaSetDevice(1);
    float4* rsrc;
    cudaMalloc(&rsrc, n * 16);
    cudaMemset(rsrc, 1, n * 16);
    cudaDeviceSynchronize();
    cudaSetDevice(0);
    cudaDeviceEnablePeerAccess(1, 0);
    src = rsrc;
  }
  // 1. alone
  const double alone = timed_copy(idc);
  // 2. while `hold` occupies `ctas` SMs
  int* started;
  cudaHostAlloc(&started, 4, cudaHostAllocMapped);
  *started = 0;
  *rel = 0;
  hold<<<ctas, 32, smem, s1>>>(ida, rel, started);
  for (int spin = 0; *(volatile int*)started < ctas && spin < 2000000; ++spin) {
  }
  const double beside = timed_copy(idb);
  *(volatile int*)rel = 1;
  cudaDeviceSynchronize();
  std::vector<unsigned> a(ctas), b(ctas), c(ctas);
  cudaMemcpy(a.data(), ida, ctas * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(b.data(), idb, ctas * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(c.data(), idc, ctas * 4, cudaMemcpyDeviceToHost);
  auto dump = [&](const char* name, const std::vector<unsigned>& v) {
    printf("\"%s\": [", name);
    for (int i = 0; i < ctas; ++i) printf("%s%u", i ? "," : "", v[i]);
    printf("]");
  };
  printf("{\"ctas\": %d, \"peer_src\": %d, \"copy_alone_gbs\": %.1f, \"copy_beside_hold_gbs\": %.1f, ", ctas, (int)peer,
         alone, beside);
  dump("smid_alone", c);
  printf(", ");
  dump("smid_hold", a);
  printf(", ");
  dump("smid_beside", b);
  printf(", \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
