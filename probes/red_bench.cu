// Scatter-add throughput on the B200: the down SSMM's epilogue pattern (DeepSeek-MoE-16B
// T=4096: 24576 (expert, token) rows x 2048 fp32 columns added into 4096 token rows, in
// 256-column pieces = one CTA's m-tile) as (A) SM-issued red.global.add.v4.f32 (the
// current epilogue) vs (B) TMA bulk reductions cp.reduce.async.bulk .add.f32 of a 1 KB
// shared-memory row per piece.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench probes/red_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

constexpr int T = 4096, D = 2048, ENT = 24576, PIECE = 256, NP = D / PIECE;

__global__ void red_v4(float* out, const int* tok, int items, float s) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int it = warp; it < items; it += nw) {
    const int e = it / NP, c = it % NP;
    float* row = out + (size_t)tok[e] * D + c * PIECE;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      float* p = row + 4 * (lane + 32 * j);
      const float v = s * (float)(lane + j);
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v), "f"(v), "f"(v), "f"(v) : "memory");
    }
  }
}

__global__ void red_bulk(float* out, const int* tok, int items, float s) {
  extern __shared__ __align__(128) float buf[];  // [warps][4][PIECE]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  int n = 0;
  for (int it = warp; it < items; it += nw, ++n) {
    const int e = it / NP, c = it % NP;
    float* sb = buf + ((size_t)w * 4 + (n & 3)) * PIECE;
    if (n >= 4 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const float v = s * (float)(lane + j);
      reinterpret_cast<float4*>(sb)[lane + 32 * j] = make_float4(v, v, v, v);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      float* row = out + (size_t)tok[e] * D + c * PIECE;
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(row),
                   "r"((uint32_t)__cvta_generic_to_shared(sb)), "r"(PIECE * 4)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  std::vector<int> h(ENT);
  std::mt19937 rng(1);
  for (int i = 0; i < ENT; ++i) h[i] = rng() % T;
  int* tok;
  float* out;
  cudaMalloc(&tok, ENT * 4);
  cudaMalloc(&out, (size_t)T * D * 4);
  cudaMemcpy(tok, h.data(), ENT * 4, cudaMemcpyHostToDevice);
  const int items = ENT * NP;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = (double)ENT * D * 4;
  for (int threads : {256, 512}) {
    for (int mode = 0; mode < 2; ++mode) {
      const size_t sm = mode ? (size_t)(threads / 32) * 4 * PIECE * 4 : 0;
      if (mode) cudaFuncSetAttribute(red_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      float best = 1e9f;
      for (int r = 0; r < 6; ++r) {
        cudaMemset(out, 0, (size_t)T * D * 4);
        cudaEventRecord(a);
        if (mode) red_bulk<<<148, threads, sm>>>(out, tok, items, 1.f);
        else red_v4<<<148, threads>>>(out, tok, items, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r && ms < best) best = ms;
      }
      cudaError_t e = cudaGetLastError();
      printf("%s threads=%d: %.3f ms, %.2f TB/s of fp32 reductions (%s)\n", mode ? "bulk reduce 1KB" : "red.v4", threads,
             best, bytes / best / 1e9, cudaGetErrorString(e));
    }
  }
  return 0;
}
