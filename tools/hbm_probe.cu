// HBM ceiling probe for the N=1 bench kernel (local_oneshot_kernel): what a
// plain copy and the 4-input / 4-output fold reach on this GPU, by unroll and
// CTAs per SM.  Not part of the library; build and run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_probe tools/hbm_probe.cu && /tmp/hbm_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint4 ld_nc(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
template <int ST>
__device__ __forceinline__ void st_v(void* p, uint4 v) {
  if (ST == 0) *reinterpret_cast<uint4*>(p) = v;
  else if (ST == 1) asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  else asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

template <int U>
__global__ void copy_k(uint4* __restrict__ d, const uint4* __restrict__ s, uint64_t nv) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride * U) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t i = v + u * stride; r[u] = i < nv ? ld_nc(s + i) : make_uint4(0, 0, 0, 0); }
#pragma unroll
    for (int u = 0; u < U; ++u) { uint64_t i = v + u * stride; if (i < nv) d[i] = r[u]; }
  }
}

struct P4 { const float* in[4]; float* out[4]; };

// 4 inputs folded in order, the sum written to 4 outputs (grid-stride vectors)
template <int U, int ST>
__global__ void fold4_k(P4 p, uint64_t nv) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride * U) {
    uint4 r[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = v + u * stride;
      uint64_t ii = i < nv ? i : 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) r[u][k] = ld_nc(p.in[k] + ii * 4);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = v + u * stride;
      float a[4];
      a[0] = __uint_as_float(r[u][0].x); a[1] = __uint_as_float(r[u][0].y); a[2] = __uint_as_float(r[u][0].z); a[3] = __uint_as_float(r[u][0].w);
#pragma unroll
      for (int k = 1; k < 4; ++k) {
        a[0] = __fadd_rn(a[0], __uint_as_float(r[u][k].x)); a[1] = __fadd_rn(a[1], __uint_as_float(r[u][k].y));
        a[2] = __fadd_rn(a[2], __uint_as_float(r[u][k].z)); a[3] = __fadd_rn(a[3], __uint_as_float(r[u][k].w));
      }
      uint4 o = make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]), __float_as_uint(a[3]));
      if (i < nv)
#pragma unroll
        for (int k = 0; k < 4; ++k) st_v<ST>(p.out[k] + i * 4, o);
    }
  }
}

// tiled: each CTA owns contiguous chunks of `TILE` vectors (better DRAM page locality per stream)
template <int U, int ST>
__global__ void fold4_tiled_k(P4 p, uint64_t nv, uint64_t tile) {
  for (uint64_t t0 = (uint64_t)blockIdx.x * tile; t0 < nv; t0 += (uint64_t)gridDim.x * tile) {
    const uint64_t t1 = t0 + tile < nv ? t0 + tile : nv;
    for (uint64_t v = t0 + threadIdx.x; v < t1; v += (uint64_t)blockDim.x * U) {
      uint4 r[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint64_t i = v + u * blockDim.x;
        uint64_t ii = i < t1 ? i : t0;
#pragma unroll
        for (int k = 0; k < 4; ++k) r[u][k] = ld_nc(p.in[k] + ii * 4);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        uint64_t i = v + u * blockDim.x;
        float a[4];
        a[0] = __uint_as_float(r[u][0].x); a[1] = __uint_as_float(r[u][0].y); a[2] = __uint_as_float(r[u][0].z); a[3] = __uint_as_float(r[u][0].w);
#pragma unroll
        for (int k = 1; k < 4; ++k) {
          a[0] = __fadd_rn(a[0], __uint_as_float(r[u][k].x)); a[1] = __fadd_rn(a[1], __uint_as_float(r[u][k].y));
          a[2] = __fadd_rn(a[2], __uint_as_float(r[u][k].z)); a[3] = __fadd_rn(a[3], __uint_as_float(r[u][k].w));
        }
        uint4 o = make_uint4(__float_as_uint(a[0]), __float_as_uint(a[1]), __float_as_uint(a[2]), __float_as_uint(a[3]));
        if (i < t1)
#pragma unroll
          for (int k = 0; k < 4; ++k) st_v<ST>(p.out[k] + i * 4, o);
      }
    }
  }
}

template <class F>
float time_ms(F f, int iters) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int i = 0; i < iters; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  const uint64_t E = 64ull << 20;  // elements per stream (256 MiB fp32), the bench's bucket
  const uint64_t bytes = E * 4, nv = E / 4;
  float *in[4], *out[4];
  for (int k = 0; k < 4; ++k) { CK(cudaMalloc(&in[k], bytes)); CK(cudaMalloc(&out[k], bytes)); cudaMemset(in[k], 0, bytes); }
  char *ca, *cb; CK(cudaMalloc(&ca, 4 * bytes)); CK(cudaMalloc(&cb, 4 * bytes));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double moved = 8.0 * bytes;  // 4 in + 4 out
  float ms = time_ms([&] { cudaMemcpyAsync(cb, ca, 4 * bytes, cudaMemcpyDeviceToDevice); }, 10);
  printf("{\"kind\":\"cudaMemcpy D2D 1 GiB\",\"GBps\":%.1f}\n", 2.0 * 4 * bytes / ms / 1e6);
  for (int bps : {1, 2, 4}) {
    ms = time_ms([&] { copy_k<4><<<sms * bps, 512>>>((uint4*)cb, (const uint4*)ca, 4 * nv); }, 10);
    printf("{\"kind\":\"copy U4\",\"blocks_per_sm\":%d,\"GBps\":%.1f}\n", bps, 2.0 * 4 * bytes / ms / 1e6);
  }
  P4 p;
  for (int k = 0; k < 4; ++k) { p.in[k] = in[k]; p.out[k] = out[k]; }
#define RUN(U, ST, BPS, TPB)                                                                                  \
  ms = time_ms([&] { fold4_k<U, ST><<<sms * BPS, TPB>>>(p, nv); }, 10);                                        \
  printf("{\"kind\":\"fold4 grid-stride\",\"U\":%d,\"st\":%d,\"blocks_per_sm\":%d,\"tpb\":%d,\"GBps\":%.1f}\n", U, ST, BPS, TPB, moved / ms / 1e6);
  RUN(4, 1, 1, 512) RUN(4, 1, 2, 512) RUN(2, 1, 2, 512) RUN(2, 1, 4, 512) RUN(1, 1, 4, 512) RUN(1, 1, 8, 256)
  RUN(4, 0, 1, 512) RUN(2, 0, 2, 512) RUN(4, 2, 1, 512) RUN(2, 2, 2, 512) RUN(2, 2, 4, 512) RUN(1, 2, 4, 512)
#define RUNT(U, ST, BPS, TILE)                                                                                \
  ms = time_ms([&] { fold4_tiled_k<U, ST><<<sms * BPS, 512>>>(p, nv, TILE); }, 10);                            \
  printf("{\"kind\":\"fold4 tiled\",\"U\":%d,\"st\":%d,\"blocks_per_sm\":%d,\"tile_vec\":%d,\"GBps\":%.1f}\n", U, ST, BPS, (int)TILE, moved / ms / 1e6);
  RUNT(4, 1, 1, 4096) RUNT(4, 1, 1, 16384) RUNT(2, 1, 2, 4096) RUNT(2, 2, 2, 4096) RUNT(4, 2, 1, 8192) RUNT(2, 2, 2, 16384)
  return 0;
}
