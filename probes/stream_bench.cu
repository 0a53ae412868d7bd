// Microbenchmark: DRAM streaming rate of cp.async.bulk into an smem ring
// (one CTA per SM, each CTA streams a private contiguous region once), as a
// function of copy size and ring depth.  Mirrors the SSMM weight stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_bench stream_bench.cu
#include <cuda_runtime.h>
#include <cstdint>

#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}

__global__ void __launch_bounds__(64, 1) stream(const uint8_t* src, size_t per_cta, int chunk, int nchunk_per_stage, int S,
                                               int evict_first, size_t wrap) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int stage_bytes = chunk * nchunk_per_stage;
  uint64_t* full = (uint64_t*)(sm + S * stage_bytes);
  uint64_t* empty = full + S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const uint8_t* base = src + ((size_t)blockIdx.x * per_cta) % wrap;
  const int iters = (int)(per_cta / stage_bytes);
  uint64_t pol;
  if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&empty[st], ((it / S) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(stage_bytes) : "memory");
      for (int c = 0; c < nchunk_per_stage; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su(sm + st * stage_bytes + c * chunk)), "l"(src + (((size_t)(base - src) + (size_t)it * stage_bytes + c * chunk) % wrap)), "r"(chunk),
                     "r"(su(&full[st])), "l"(pol) : "memory");
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&full[st], (it / S) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[st])) : "memory");
    }
  }
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const size_t per_cta = (size_t)6 << 20;  // 6 MB per CTA -> 888 MB total (>> L2)
  uint8_t* src;
  CK(cudaMalloc(&src, per_cta * 148));
  CK(cudaMemset(src, 1, per_cta * 148));
  struct Cfg { int chunk, nchunk, S; } cfgs[] = {
      {18496, 2, 5}, {18496, 2, 3}, {18496, 1, 10}, {16384, 1, 12}, {32768, 1, 6}, {65536, 1, 3},
      {8192, 1, 24}, {4096, 4, 12}, {18496, 2, 2}};
  for (size_t wrap : {per_cta * 148, (size_t)32 << 20})
  for (auto c : cfgs)
    for (int ef = 0; ef < 1; ++ef) {
      const int smem = c.chunk * c.nchunk * c.S + 2048;
      if (smem > 232448) continue;
      CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        stream<<<148, 64, smem>>>(src, per_cta, c.chunk, c.nchunk, c.S, ef, wrap);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
      }
      const size_t iters = per_cta / ((size_t)c.chunk * c.nchunk);
      const double bytes = 148.0 * iters * c.chunk * c.nchunk;
      printf("%s chunk %6d x%d  stages %2d  in-flight %4d KB  %s  %7.3f ms  %7.1f GB/s\n", wrap < per_cta * 148 ? "L2  " : "DRAM", c.chunk, c.nchunk, c.S,
             c.chunk * c.nchunk * c.S / 1024, ef ? "evict_first " : "evict_normal", best, bytes / best / 1e6);
    }
  return 0;
}
