// Micro-timing of the small kernel's local fold (diagnostic, not product
// code): one CTA of 512 threads folds N=4 local 1 KB / 64 KB buffers with
// the same device functions the kernels use, thread 0 stamping clock64()
// around owner_of, fold_range and fold_tiles.  Built as one translation
// unit with the library source so it calls the real functions.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//        -Ipaper_2602_00277_b200/csrc -Iinclude -o tools/_build/fold_micro tools/fold_micro.cu -lcuda
//   tools/_build/fold_micro
#include "../paper_2602_00277_b200/csrc/ftar_b200.cu"

namespace {

__global__ void __launch_bounds__(kThreads, 1) fold_micro_kernel(LaunchParams p, const float* a, const float* b,
                                                                 const float* c, const float* d, float* out,
                                                                 uint64_t E, long long* t) {
  __shared__ const float* s_src[4];
  if (threadIdx.x == 0) {
    s_src[0] = a;
    s_src[1] = b;
    s_src[2] = c;
    s_src[3] = d;
  }
  __syncthreads();
  uint32_t nf = 0;
  for (int rep = 0; rep < 3; ++rep) {
    __syncthreads();
    long long t0 = clock64();
    int own;
    uint64_t send;
    owner_of(0, p, 4, own, send);
    long long t1 = clock64();
    fold_range<4, F32In, Unroll<4, F32In>::U, SinkOne, false>(s_src, SinkOne{out}, 0, E, own, 0xfu, true, true,
                                                              0.25f, nf);
    long long t2 = clock64();
    __syncthreads();
    long long t3 = clock64();
    fold_tiles<4, F32In, SinkOne, true>(p, s_src, SinkOne{out}, 0, E, true, true, nf, nullptr, 0x7fffffff, 1, 0);
    long long t4 = clock64();
    __syncthreads();
    long long t5 = clock64();
    if (threadIdx.x == 0) {
      t[rep * 5 + 0] = t1 - t0 + (own == 99 ? 1 : 0);  // owner_of
      t[rep * 5 + 1] = t2 - t1;                        // fold_range (thread 0)
      t[rep * 5 + 2] = t3 - t2;                        // barrier after it
      t[rep * 5 + 3] = t4 - t3;                        // fold_tiles (thread 0)
      t[rep * 5 + 4] = t5 - t4;                        // barrier after it
    }
  }
  if (nf == 12345) out[0] = 0.f;
}

}  // namespace

int main() {
  for (uint64_t E : {256ull, 16384ull}) {
    float* buf;
    cudaMalloc(&buf, 6 * E * 4 + 4096);
    cudaMemset(buf, 0, 6 * E * 4);
    long long* t;
    cudaMallocManaged(&t, 15 * sizeof(long long));
    LaunchParams p{};
    fill_geometry(p, E, 8 << 20, 4, 4);
    fold_micro_kernel<<<1, kThreads>>>(p, buf, buf + E, buf + 2 * E, buf + 3 * E, buf + 4 * E, E, t);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"elems\": %llu, \"err\": \"%s\", \"cycles\": {", (unsigned long long)E, cudaGetErrorString(e));
    const char* names[5] = {"owner_of", "fold_range_t0", "barrier1", "fold_tiles_t0", "barrier2"};
    for (int k = 0; k < 5; ++k)
      printf("%s\"%s\": [%lld, %lld, %lld]", k ? ", " : "", names[k], t[k], t[5 + k], t[10 + k]);
    printf("}}\n");
    cudaFree(buf);
    cudaFree(t);
  }
  return 0;
}
