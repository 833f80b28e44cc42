// Microbenchmark: write bandwidth of 1 KiB blocks (the decode's output pattern: block i ->
// position perm[i] or i) under different store shapes, plus reads and cudaMemset as
// references.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_mb_scatter tools/mb_scatter.cu
//   half  : lane l stores floats [8l, 8l+4) then [8l+4, 8l+8)   (each warp store covers half of every sector)
//   full  : lane l stores floats [4l, 4l+4) then [128+4l, 128+4l+4) (each warp store = 512 contiguous bytes)
//   *cs   : streaming stores (st.global.cs), else plain st.global
//   bulk  : the warp stages the block in shared memory, one lane writes it with cp.async.bulk (TMA)
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int MODE, bool CS>  // MODE 0 half, 1 full
__global__ void k_write(float* out, const uint32_t* perm, uint32_t T, int seq) {
  const int lane = threadIdx.x & 31;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < T; i += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t dst = seq ? i : __ldg(perm + i);
    float* b = out + (uint64_t)dst * 256;
    float4* o0 = reinterpret_cast<float4*>(b + (MODE == 0 ? lane * 8 : lane * 4));
    float4* o1 = reinterpret_cast<float4*>(b + (MODE == 0 ? lane * 8 + 4 : 128 + lane * 4));
    const float4 v0 = make_float4(1.f, 2.f, 3.f, (float)i), v1 = make_float4(5.f, 6.f, 7.f, 8.f);
    if (CS) { __stcs(o0, v0); __stcs(o1, v1); } else { *o0 = v0; *o1 = v1; }
  }
}

__global__ void k_write_bulk(float* out, const uint32_t* perm, uint32_t T, int seq) {
  __shared__ alignas(128) float stage[8][2][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int k = 0;
  for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < T; i += (gridDim.x * blockDim.x) >> 5, k ^= 1) {
    const uint32_t dst = seq ? i : __ldg(perm + i);
    float* s = stage[warp][k];
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // the buffer's previous store has read smem
    __syncwarp();
    reinterpret_cast<float4*>(s)[lane] = make_float4(1.f, 2.f, 3.f, (float)i);
    reinterpret_cast<float4*>(s)[32 + lane] = make_float4(5.f, 6.f, 7.f, 8.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(s));
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 1024;" ::"l"(out + (uint64_t)dst * 256), "r"(sa) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

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
  auto run = [&](const char* name, auto launch) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(a);
    for (int r = 0; r < 10; ++r) launch();
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 10;
    printf("%-28s %.3f ms  %.2f TB/s  %s\n", name, ms, (double)T * 1024 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  run("memset (driver)", [&] { cudaMemsetAsync(out, 0, (size_t)T * 1024); });
  for (int grid_mul : {4, 8}) {
    const int grid = 148 * grid_mul;
    char nm[64];
    for (int seq = 0; seq < 2; ++seq) {
      const char* p = seq ? "seq" : "perm";
      snprintf(nm, 64, "write half cs %s g%d", p, grid); run(nm, [&] { k_write<0, true><<<grid, 256>>>(out, perm, T, seq); });
      snprintf(nm, 64, "write half st %s g%d", p, grid); run(nm, [&] { k_write<0, false><<<grid, 256>>>(out, perm, T, seq); });
      snprintf(nm, 64, "write full cs %s g%d", p, grid); run(nm, [&] { k_write<1, true><<<grid, 256>>>(out, perm, T, seq); });
      snprintf(nm, 64, "write full st %s g%d", p, grid); run(nm, [&] { k_write<1, false><<<grid, 256>>>(out, perm, T, seq); });
      snprintf(nm, 64, "write bulk(TMA) %s g%d", p, grid); run(nm, [&] { k_write_bulk<<<grid, 256>>>(out, perm, T, seq); });
      snprintf(nm, 64, "read %s g%d", p, grid); run(nm, [&] { k_read<<<grid, 256>>>(out, perm, T, seq, sink); });
    }
  }
  return 0;
}
