// Microbenchmark: L2 -> smem rate of TMA tensor loads (cp.async.bulk.tensor,
// no swizzle, 128-B rows) vs plain cp.async.bulk for the same contiguous
// bytes, one CTA per SM with an S-stage ring.  The weight image block
// (18688 B = 146 rows of 128 B) is described as a 3D tensor {64 bf16, 146, nblk}
// so one request can move 1..n consecutive blocks.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_bench tma_bench.cu -lcuda
#include <cuda.h>
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

__global__ void __launch_bounds__(64, 1) kern(const __grid_constant__ CUtensorMap tm, const uint8_t* src, int nblk_total,
                                             int blk_per_req, int reqs_per_stage, int S, int iters, int mode) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  const int req_bytes = 18688 * blk_per_req;
  const int stage_bytes = req_bytes * reqs_per_stage;
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
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x == 0) {
    int blk = (blockIdx.x * 977) % (nblk_total - 16);
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&empty[st], ((it / S) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[st])), "r"(stage_bytes) : "memory");
      for (int r = 0; r < reqs_per_stage; ++r) {
        const uint32_t dst = su(sm + st * stage_bytes + r * req_bytes);
        if (mode == 0) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                       ::"r"(dst), "l"(src + (size_t)blk * 18688), "r"(req_bytes), "r"(su(&full[st])), "l"(pol) : "memory");
        } else {
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
                       ::"r"(dst), "l"(&tm), "r"(0), "r"(0), "r"(blk), "r"(su(&full[st])), "l"(pol) : "memory");
        }
        blk += blk_per_req;
        if (blk >= nblk_total - 16) blk -= nblk_total - 16;
      }
    }
  } else if (threadIdx.x == 32) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&full[st], (it / S) & 1);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[st])) : "memory");
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  EncodeFn enc; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  for (size_t wrap_mb : {48, 2048}) {
    const int nblk = (int)((wrap_mb << 20) / 18688);
    uint8_t* src; CK(cudaMalloc(&src, (size_t)nblk * 18688)); CK(cudaMemset(src, 1, (size_t)nblk * 18688));
    for (int bpr : {1, 2}) {
      CUtensorMap tm;
      cuuint64_t dims[3] = {64, 146, (cuuint64_t)nblk};
      cuuint64_t strides[2] = {128, 18688};
      cuuint32_t box[3] = {64, 146, (cuuint32_t)bpr};
      cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
      for (int rps : {1, 2}) {
        for (int mode : {0, 1}) {
          const int S = bpr * rps >= 4 ? 2 : bpr * rps == 2 ? 4 : 8;
          const int stage = 18688 * bpr * rps;
          const int smem = S * stage + 1024 + 2 * S * 8 + 64;
          CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
          const int iters = (int)((size_t)64 << 20) / stage;
          for (int rep = 0; rep < 2; ++rep) kern<<<nsm, 64, smem>>>(tm, src, nblk, bpr, rps, S, iters, mode);
          CK(cudaGetLastError());
          cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
          cudaEventRecord(a);
          kern<<<nsm, 64, smem>>>(tm, src, nblk, bpr, rps, S, iters, mode);
          cudaEventRecord(b); CK(cudaEventSynchronize(b));
          float ms; cudaEventElapsedTime(&ms, a, b);
          const double landed = (double)nsm * iters * stage;
          printf("src %4zu MB  %s  req %5d B x%d/stage  S=%d : %.2f TB/s (%.1f B/clk/SM @1.9GHz)\n", wrap_mb,
                 mode ? "tensor3d" : "bulk    ", 18688 * bpr, rps, S, landed / ms / 1e9, landed / ms / 1e9 * 1e12 / nsm / 1.9e9);
        }
      }
    }
    cudaFree(src);
  }
  return 0;
}
