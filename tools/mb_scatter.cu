// Microbenchmark: 1 KiB blocks written / read in a random permutation vs sequentially
// (the gather decode and the leaf gather access pattern).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_mb_scatter tools/mb_scatter.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
// write T blocks of 1 KiB (256 floats): block i -> position perm[i]; one warp per block, 8 floats per lane
__global__ void k_write(float* out, const uint32_t* perm, uint32_t T, int seq) {
  const int lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < T; i += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t dst = seq ? i : __ldg(perm + i);
    float4* o = reinterpret_cast<float4*>(out + (uint64_t)dst * 256 + lane * 8);
    __stcs(o, make_float4(1.f, 2.f, 3.f, (float)i));
    __stcs(o + 1, make_float4(5.f, 6.f, 7.f, 8.f));
  }
}
// read pattern: block i <- position perm[i]
__global__ void k_read(const float* in, const uint32_t* perm, uint32_t T, int seq, float* sink) {
  const int lane = threadIdx.x & 31;
  float acc = 0.f;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < T; i += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t src = seq ? i : __ldg(perm + i);
    const float4* p = reinterpret_cast<const float4*>(in + (uint64_t)src * 256 + lane * 8);
    float4 a = __ldcs(p), b = __ldcs(p + 1);
    acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
  }
  if (acc == 12345.f) *sink = acc;
}
int main() {
  const uint32_t T = 1u << 20;  // 1 GiB
  float *out, *sink; uint32_t* perm;
  cudaMalloc(&out, (size_t)T * 1024); cudaMalloc(&perm, T * 4); cudaMalloc(&sink, 4);
  std::vector<uint32_t> h(T); for (uint32_t i = 0; i < T; ++i) h[i] = i;
  std::mt19937 g(1); std::shuffle(h.begin(), h.end(), g);
  cudaMemcpy(perm, h.data(), T * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int grid_mul : {4, 8, 16}) for (int rd = 0; rd < 2; ++rd) for (int seq = 0; seq < 2; ++seq) {
    const int grid = 148 * grid_mul;
    for (int w = 0; w < 3; ++w) { if (rd) k_read<<<grid, 256>>>(out, perm, T, seq, sink); else k_write<<<grid, 256>>>(out, perm, T, seq); }
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) { if (rd) k_read<<<grid, 256>>>(out, perm, T, seq, sink); else k_write<<<grid, 256>>>(out, perm, T, seq); }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%s %s grid=%d: %.3f ms  %.2f TB/s\n", rd ? "read " : "write", seq ? "seq " : "perm", grid, ms, (double)T * 1024 / ms / 1e9);
  }
  return 0;
}
