// NVLink SHARP multicast probe (one process, every visible GPU): does an
// all-gather by multicast stores (each GPU sends its slice ONCE; the switch
// replicates it) beat the unicast push FTAR uses now (each GPU writes its
// slice to every peer), alone and while an RS-like peer-pull load runs?
// Not part of the library.  Build/run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/nvls tools/nvls_probe.cu -lcuda && /tmp/nvls
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CU(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); printf("{\"error\":\"%s:%d %s\"}\n", __FILE__, __LINE__, s_); return 1; } } while (0)
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\":\"%s:%d %s\"}\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kMax = 8;
struct Ptrs { float* p[kMax]; };

// multicast all-gather: my slice -> every member's buffer through the switch
__global__ void mc_push(float* mc_dst, const float* src, uint64_t nvec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const float4 x = reinterpret_cast<const float4*>(src)[v];
    float* a = mc_dst + v * 4;
    asm volatile("multimem.st.weak.global.v4.f32 [%0], {%1,%2,%3,%4};" :: "l"(a), "f"(x.x), "f"(x.y), "f"(x.z), "f"(x.w) : "memory");
  }
}

// unicast push (what FTAR's push mode does): my slice -> each peer's buffer
__global__ void uc_push(Ptrs dst, int n, int me, uint64_t off, const float* src, uint64_t nvec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    const float4 x = reinterpret_cast<const float4*>(src)[v];
    for (int j = 0; j < n; ++j) reinterpret_cast<float4*>(dst.p[j] + off)[v] = x;
  }
}

// RS-like load: pull my slice from every peer's input and sum (reads only)
__global__ void rs_pull(Ptrs in, int n, int me, uint64_t off, float* out, uint64_t nvec) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
    float4 acc = make_float4(0, 0, 0, 0);
    for (int j = 0; j < n; ++j) {
      const float4 x = reinterpret_cast<const float4*>(in.p[j] + off)[v];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    reinterpret_cast<float4*>(out)[v] = acc;
  }
}

__global__ void fill(float* p, uint64_t n, float base) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    p[i] = base + (float)(i % 1024);
}

int main(int argc, char** argv) {
  int G = 0;
  CK(cudaGetDeviceCount(&G));
  if (G > kMax) G = kMax;
  if (G < 2) { printf("{\"error\":\"need >= 2 GPUs\"}\n"); return 0; }
  CU(cuInit(0));
  const uint64_t S = 256ull << 20;  // bytes of the full (fp32) bucket per GPU
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    for (int e = 0; e < G; ++e) if (e != d) { cudaDeviceEnablePeerAccess(e, 0); cudaGetLastError(); }
  }
  CUmulticastObjectProp mp{};
  mp.numDevices = G;
  mp.size = S;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t gran = 0;
  CU(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const uint64_t SZ = (S + gran - 1) / gran * gran;
  mp.size = SZ;
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &mp));
  std::vector<CUdevice> dev(G);
  for (int d = 0; d < G; ++d) { CU(cuDeviceGet(&dev[d], d)); CU(cuMulticastAddDevice(mc, dev[d])); }
  std::vector<CUmemGenericAllocationHandle> mem(G);
  std::vector<CUdeviceptr> uc(G);
  std::vector<CUmemAccessDesc> all(G);
  for (int d = 0; d < G; ++d) {
    all[d].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    all[d].location.id = d;
    all[d].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    CU(cuMemCreate(&mem[d], SZ, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, mem[d], 0, SZ, 0));
    CU(cuMemAddressReserve(&uc[d], SZ, gran, 0, 0));
    CU(cuMemMap(uc[d], SZ, 0, mem[d], 0));
    CU(cuMemSetAccess(uc[d], SZ, all.data(), G));  // every GPU may read/write it (unicast push baseline)
  }
  CUdeviceptr mcva;
  CU(cuMemAddressReserve(&mcva, SZ, gran, 0, 0));
  CU(cuMemMap(mcva, SZ, 0, mc, 0));
  CU(cuMemSetAccess(mcva, SZ, all.data(), G));
  // inputs (RS load) and local slices
  const uint64_t E = S / 4, slice = E / G, nvec = slice / 4;
  std::vector<float*> in(G), src(G), red(G);
  std::vector<cudaStream_t> st(G), st2(G);
  for (int d = 0; d < G; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&in[d], S));
    CK(cudaMalloc(&src[d], slice * 4));
    CK(cudaMalloc(&red[d], slice * 4));
    fill<<<264, 512>>>(in[d], E, 0.f);
    fill<<<264, 512>>>(src[d], slice, (float)(d * 100000));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&st2[d], cudaStreamNonBlocking));
  }
  for (int d = 0; d < G; ++d) { CK(cudaSetDevice(d)); CK(cudaDeviceSynchronize()); }
  Ptrs ucp{}, inp{};
  for (int d = 0; d < G; ++d) { ucp.p[d] = reinterpret_cast<float*>(uc[d]); inp.p[d] = in[d]; }
  const int ctas = argc > 1 ? atoi(argv[1]) : 64;

  // mode: 0 = multicast AG, 1 = unicast AG, 2 = RS pull only, 3 = RS + mc AG, 4 = RS + uc AG
  auto run = [&](int mode, int iters) -> double {
    std::vector<cudaEvent_t> a(G), b(G);
    for (int d = 0; d < G; ++d) { cudaSetDevice(d); cudaEventCreate(&a[d]); cudaEventCreate(&b[d]); }
    for (int d = 0; d < G; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); }
    for (int d = 0; d < G; ++d) { cudaSetDevice(d); cudaEventRecord(a[d], st[d]); }
    for (int it = 0; it < iters; ++it)
      for (int d = 0; d < G; ++d) {
        cudaSetDevice(d);
        const uint64_t off = (uint64_t)d * slice;
        if (mode == 0 || mode == 3) mc_push<<<ctas, 512, 0, st[d]>>>(reinterpret_cast<float*>(mcva) + off, src[d], nvec);
        if (mode == 1 || mode == 4) uc_push<<<ctas, 512, 0, st[d]>>>(ucp, G, d, off, src[d], nvec);
        if (mode >= 2) rs_pull<<<ctas, 512, 0, st2[d]>>>(inp, G, d, off, red[d], nvec);
      }
    for (int d = 0; d < G; ++d) {
      cudaSetDevice(d);
      cudaEvent_t j; cudaEventCreate(&j); cudaEventRecord(j, st2[d]); cudaStreamWaitEvent(st[d], j, 0);
      cudaEventRecord(b[d], st[d]);
    }
    double worst = 0;
    for (int d = 0; d < G; ++d) {
      cudaSetDevice(d); cudaEventSynchronize(b[d]);
      float ms; cudaEventElapsedTime(&ms, a[d], b[d]);
      if (ms > worst) worst = ms;
    }
    return worst / iters;
  };
  const char* names[] = {"mc_allgather", "unicast_allgather", "rs_pull_only", "rs_pull+mc_allgather", "rs_pull+unicast_allgather"};
  for (int mode = 0; mode < 5; ++mode) {
    run(mode, 2);
    const double ms = run(mode, 10);
    // per-GPU ingress of the AG: (G-1)/G of the bucket; of the RS: (G-1)/G too
    const double ag_bytes = (double)S * (G - 1) / G;
    printf("{\"G\":%d,\"ctas\":%d,\"mode\":\"%s\",\"ms\":%.4f,\"ag_ingress_GBps\":%.1f}\n", G, ctas, names[mode], ms,
           (mode == 2 ? 0.0 : ag_bytes / (ms * 1e-3) / 1e9));
  }
  // correctness: after a multicast AG every GPU holds every slice
  run(0, 1);
  int bad = 0;
  std::vector<float> h(4);
  for (int d = 0; d < G && !bad; ++d)
    for (int s = 0; s < G; ++s) {
      CK(cudaMemcpy(h.data(), reinterpret_cast<float*>(uc[d]) + (uint64_t)s * slice + 5, 16, cudaMemcpyDeviceToHost));
      if (h[0] != (float)(s * 100000 + 5)) { bad = 1; break; }
    }
  printf("{\"mc_allgather_correct\":%s}\n", bad ? "false" : "true");
  return 0;
}
