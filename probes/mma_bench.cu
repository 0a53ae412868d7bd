// Microbenchmark: issue rate of tcgen05.mma (.sp and dense, kind::f16, cta_group::1,
// M=128) from smem operands, per N, with/without disable_output_lane masks.
// One CTA per SM; one elected thread issues R MMAs back to back; clk per MMA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench mma_bench.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t dsw128(uint32_t a) {
  return (uint64_t)((a & 0x3FFFF) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t dint(uint32_t a) {
  return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)8 << 16) | ((uint64_t)8 << 32) | (1ull << 46);
}

template <int N, int MODE>  // MODE 0 sparse, 1 sparse+mask, 2 dense
__global__ void __launch_bounds__(128, 1) bench(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  uint8_t* A = sm;                 // 16 KB
  uint8_t* B = sm + 16384;         // N * 128 * 2
  uint8_t* E = B + N * 256;        // 2 KB
  for (int i = threadIdx.x; i < (16384 + N * 256 + 2048) / 4; i += 128) ((uint32_t*)sm)[i] = (i >= (16384 + N * 256) / 4) ? 0x44444444u : 0x3c003c00u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x < 32) {
    const uint32_t idesc_sp = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t idesc_d = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint32_t ecol = 508;
    asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.cp.cta_group::1.128x128b [%0], %1;}" ::"r"(tm + ecol), "l"(dint(su(E))));
    const uint64_t ad = dsw128(su(A)), bd = dsw128(su(B));
    uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    if (MODE == 1) { m0 = 0xAAAAAAAAu; m1 = 0x55555555u; m2 = 0xF0F0F0F0u; m3 = 0x0F0F0F0Fu; }
    __syncwarp();
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t d = tm + ((r & 1) ? 256 : 0) * (N <= 128 ? 1 : 0);
      if (MODE == 2) {
        asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;}"
                     ::"r"(d), "l"(ad), "l"(bd), "r"(idesc_d));
      } else {
        asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.mma.sp.cta_group::1.kind::f16 [%0], %1, %2, [%8], %3, {%4, %5, %6, %7}, 1;}"
                     ::"r"(d), "l"(ad), "l"(bd), "r"(idesc_sp | (r & 1)), "r"(m0), "r"(m1), "r"(m2), "r"(m3), "r"(tm + ecol));
      }
    }
    asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(su(&bar)));
    uint32_t done = 0;
    do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(su(&bar))); } while (!done);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int MODE>
void run(const char* name) {
  const int reps = 4096;
  const int smem = 16384 + N * 256 + 2048 + 1024;
  cudaFuncSetAttribute(bench<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  bench<N, MODE><<<148, 128, smem>>>(reps, d);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<N, MODE><<<148, 128, smem>>>(reps, d);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double clk = 0; for (int i = 0; i < 148; ++i) clk += h[i]; clk /= 148;
  const double k = MODE == 2 ? 16 : 32;  // logical K per MMA
  const double flops = 2.0 * 128 * N * k * reps * 148;
  printf("%-22s N=%3d  %7.1f clk/MMA  %8.1f TFLOP/s (dense-equivalent of the issued MMAs)\n", name, N, clk / reps, flops / (ms * 1e-3) / 1e12);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  run<16, 0>("sparse");  run<64, 0>("sparse");  run<112, 0>("sparse");  run<128, 0>("sparse");
  run<224, 0>("sparse"); run<256, 0>("sparse");
  run<112, 1>("sparse+mask"); run<224, 1>("sparse+mask");
  run<112, 2>("dense K16"); run<256, 2>("dense K16");
  return 0;
}
