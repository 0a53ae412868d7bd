// Microbenchmark: L2 -> smem delivery rate of cp.async.bulk, unicast vs
// .multicast::cluster, for clusters of CL CTAs that all need the same bytes
// (the SSMM weight stream shared by CTAs on the same m-tile).  Each CTA keeps
// an S-stage ring; `mc` = 0: every CTA fetches every chunk itself; `mc` = 1:
// chunk c of a stage is fetched by rank c % CL and multicast to all ranks.
// Reported: bytes landed in shared memory per second (all CTAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mcast_bench mcast_bench.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t crank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void wait_cl(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}

template <int CL>
__global__ void __launch_bounds__(64, 1) kern(const uint8_t* src, size_t wrap, int chunk, int nchunk, int S, int iters, int mc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int stage_bytes = chunk * nchunk;
  uint64_t* full = (uint64_t*)(sm + S * stage_bytes);
  uint64_t* empty = full + S;
  const uint32_t rank = CL > 1 ? crank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[s])), "r"(mc ? CL : 1));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (CL > 1) cooperative_groups::this_cluster().sync(); else __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  const size_t cl_id = blockIdx.x / CL;
  if (threadIdx.x == 0) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait_cl(&empty[st], ((it / S) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(stage_bytes) : "memory");
      for (int c = 0; c < nchunk; ++c) {
        const uint8_t* g = src + ((cl_id * 7919 + (size_t)it) * stage_bytes + (size_t)c * chunk) % wrap;
        const uint32_t dst = su(sm + st * stage_bytes + c * chunk);
        if (!mc) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(dst), "l"(g), "r"(chunk), "r"(su(&full[st])), "l"(pol) : "memory");
        } else if (c % CL == (int)rank) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster.L2::cache_hint [%0], [%1], %2, [%3], %4, %5;"
                       ::"r"(dst), "l"(g), "r"(chunk), "r"(su(&full[st])), "h"((uint16_t)((1u << CL) - 1)), "l"(pol) : "memory");
        }
      }
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait_cl(&full[st], (it / S) & 1);
      if (!mc) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[st])) : "memory");
      } else {
        for (int r = 0; r < CL; ++r) {
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su(&empty[st])), "r"(r));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
      }
    }
  }
  if (CL > 1) cooperative_groups::this_cluster().sync();
}

template <int CL>
void run(const uint8_t* src, size_t wrap, int chunk, int nchunk, int S, int mc, int nsm) {
  const int stage = chunk * nchunk;
  const int smem = S * stage + 1024 + 2 * S * 8 + 64;
  auto k = kern<CL>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3(nsm / CL * CL); cfg.blockDim = dim3(64); cfg.dynamicSmemBytes = smem; cfg.attrs = at; cfg.numAttrs = 1;
  const int iters = (int)((size_t)64 << 20) / stage;  // 64 MB landed per CTA
  for (int rep = 0; rep < 2; ++rep) CK(cudaLaunchKernelEx(&cfg, k, src, wrap, chunk, nchunk, S, iters, mc));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  CK(cudaLaunchKernelEx(&cfg, k, src, wrap, chunk, nchunk, S, iters, mc));
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double landed = (double)(nsm / CL * CL) * iters * stage;
  printf("CL=%d mc=%d chunk=%6d x%d S=%d : landed %.2f TB/s (%.1f B/clk/SM @1.9GHz), L2 reads %.2f TB/s\n", CL, mc, chunk, nchunk, S,
         landed / ms / 1e9, landed / ms / 1e9 * 1e12 / (nsm / CL * CL) / 1.9e9, landed / ms / 1e9 / (mc ? CL : 1));
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const size_t wrap = (size_t)48 << 20;  // L2-resident source
  uint8_t* src; CK(cudaMalloc(&src, wrap + (1 << 20))); CK(cudaMemset(src, 1, wrap + (1 << 20)));
  for (int chunk : {18688, 37376}) {
    const int nchunk = chunk == 18688 ? 2 : 1;
    for (int S : {4}) {
      run<1>(src, wrap, chunk, nchunk, S, 0, nsm);
      run<2>(src, wrap, chunk, nchunk, S, 0, nsm);
      run<2>(src, wrap, chunk, nchunk, S, 1, nsm);
      run<4>(src, wrap, chunk, nchunk, S, 0, nsm);
      run<4>(src, wrap, chunk, nchunk, S, 1, nsm);
    }
  }
  run<4>(src, wrap, 9344, 4, 4, 1, nsm);
  run<2>(src, wrap, 4096, 8, 6, 1, nsm);
  run<1>(src, wrap, 4096, 8, 6, 0, nsm);
  return 0;
}
