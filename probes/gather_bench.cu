// Microbenchmark: throughput of token-row gathers into a 128B-swizzled smem tile
// on B200 (one CTA per SM, L2-resident source), for the SSMM's B operand.
//   mode 0: tile::gather4 TMA (one warp issues)
//   mode 1: 2D TMA per row (box 64 x 1)
//   mode 2: cp.async 16 B by 128 threads (wait_group 0 + proxy fence + arrive)
//   mode 3: contiguous 2D TMA tile (box 64 x 128), no gather -- reference
//   mode 4: gather4 with cluster multicast (cluster of 4 CTAs, each issues 1/4)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o gather_bench gather_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int NT = 128;            // rows per stage
constexpr int STAGE = NT * 256;    // 2 atoms x NT x 128 B
constexpr int S = 4;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void expect_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}
__device__ __forceinline__ void wait_cluster(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}

__global__ void __launch_bounds__(320, 1) bench(const __grid_constant__ CUtensorMap gmap, const __grid_constant__ CUtensorMap tmap,
                                               const uint16_t* x, int ldx, const int* sel, int nsel, int iters, int mode) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(sm + S * STAGE);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t crank = 0;
  if (mode == 4) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], (mode == 2 || mode == 8) ? (mode == 8 ? 5 : 4) : mode == 5 ? 8 : mode == 6 ? 4 : 1); mbar_init(&empty[s], mode == 4 ? 4 : 1); }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (mode == 4) { asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;"); }
  const int base = (blockIdx.x * 977) % (nsel - NT);
  if (warp == 5) {  // consumer: wait full, release
    if (lane == 0)
      for (int it = 0; it < iters; ++it) {
        const int st = it % S;
        if (mode == 4) wait_cluster(&full[st], (it / S) & 1); else wait(&full[st], (it / S) & 1);
        if (mode == 4) {  // release the slot in every CTA of the cluster (each multicast writes to all)
          for (uint32_t c = 0; c < 4; ++c) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(su(&empty[st])), "r"(c));
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
          }
        } else {
          arrive(&empty[st]);
        }
      }
  } else if ((mode == 5 && (warp < 4 || warp >= 6)) || (mode == 6 && (warp < 4 || warp >= 6))) {
    // loader warps: 0-3 and 6-9 (8 warps)
    const int lw = warp < 4 ? warp : warp - 2;         // 0..7
    const int grp = mode == 6 ? lw / 4 : 0;
    const int nthr = mode == 6 ? 128 : 256;
    const int tid = (mode == 6 ? lw % 4 : lw) * 32 + lane;
    for (int it = grp; it < iters; it += (mode == 6 ? 2 : 1)) {
      const int st = it % S;
      wait(&empty[st], ((it / S) & 1) ^ 1);
      uint8_t* b = sm + st * STAGE;
      const int col0 = (it * 128) % (ldx - 128);
      for (int idx = tid; idx < NT * 16; idx += nthr) {
        const int row = idx / 16, ch = idx % 16, atom = ch / 8, c8 = ch % 8;
        const uint16_t* src = x + (size_t)sel[base + row] * ldx + col0 + ch * 8;
        uint8_t* dst = b + atom * NT * 128 + (row / 8) * 1024 + (row % 8) * 128 + ((c8 ^ (row % 8)) << 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(dst)), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group; cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive(&full[st]);
    }
  } else if (mode == 8 && warp == 4) {
    // hybrid: rows [0, kG) of every stage by tile::gather4 from one thread
    constexpr int kG = 16;
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&empty[st], ((it / S) & 1) ^ 1);
      uint8_t* b = sm + st * STAGE;
      const int col0 = (it * 128) % (ldx - 128);
      if (lane == 0) {
        arrive_tx(&full[st], kG * 256);
        for (int g = 0; g < kG / 4; ++g)
          for (int atom = 0; atom < 2; ++atom) {
            const int* r = sel + base + 4 * g;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(b + atom * NT * 128 + g * 512)), "l"(&gmap),
                         "r"(col0 + atom * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(su(&full[st]))
                         : "memory");
          }
      }
    }
  } else if ((mode == 2 || mode == 8) && warp < 4) {
    const int tid = threadIdx.x + (mode == 8 ? 16 * 16 : 0);  // mode 8: rows from kG = 16 on
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&empty[st], ((it / S) & 1) ^ 1);
      uint8_t* b = sm + st * STAGE;
      const int col0 = (it * 128) % (ldx - 128);
      for (int idx = tid; idx < NT * 16; idx += 128) {
        const int row = idx / 16, ch = idx % 16, atom = ch / 8, c8 = ch % 8;
        const uint16_t* src = x + (size_t)sel[base + row] * ldx + col0 + ch * 8;
        uint8_t* dst = b + atom * NT * 128 + (row / 8) * 1024 + (row % 8) * 128 + ((c8 ^ (row % 8)) << 4);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(dst)), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group; cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive(&full[st]);
    }
  } else if (warp == 4 && mode != 2 && mode != 8 && (mode < 5 || mode == 7)) {
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&empty[st], ((it / S) & 1) ^ 1);
      uint8_t* b = sm + st * STAGE;
      const int col0 = (it * 128) % (ldx - 128);
      if (mode == 4) {
        if (lane == 0) arrive_tx(&full[st], STAGE);
        __syncwarp();
        // this CTA issues gathers crank, crank+4, ... and multicasts to all 4 CTAs
        for (int g = lane; g < NT / 4; g += 32) {
          if (g % 4 != (int)crank) continue;
          for (int atom = 0; atom < 2; ++atom) {
            const int* r = sel + base + 4 * g;
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.multicast::cluster"
                         " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(su(b + atom * NT * 128 + g * 512)), "l"(&gmap),
                         "r"(col0 + atom * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(su(&full[st])), "h"((uint16_t)0xF)
                         : "memory");
          }
        }
      } else {
        if (lane == 0) arrive_tx(&full[st], STAGE);
        __syncwarp();
        if (mode == 7 && lane == 0) {  // one thread issues every gather4 of the stage
          for (int g = 0; g < NT / 4; ++g)
            for (int atom = 0; atom < 2; ++atom) {
              const int* r = sel + base + 4 * g;
              asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                           " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(b + atom * NT * 128 + g * 512)), "l"(&gmap),
                           "r"(col0 + atom * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(su(&full[st]))
                           : "memory");
            }
        } else if (mode == 0) {
          for (int g = lane; g < NT / 4; g += 32)
            for (int atom = 0; atom < 2; ++atom) {
              const int* r = sel + base + 4 * g;
              asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                           " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(b + atom * NT * 128 + g * 512)), "l"(&gmap),
                           "r"(col0 + atom * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(su(&full[st]))
                           : "memory");
            }
        } else if (mode == 1) {
          for (int row = lane; row < NT; row += 32)
            for (int atom = 0; atom < 2; ++atom)
              asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                           " [%0], [%1, {%2, %3}], [%4];" ::"r"(su(b + atom * NT * 128 + row * 128)), "l"(&gmap),
                           "r"(col0 + atom * 64), "r"(sel[base + row]), "r"(su(&full[st]))
                           : "memory");
        } else if (mode == 3 && lane == 0) {
          for (int atom = 0; atom < 2; ++atom)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3}], [%4];" ::"r"(su(b + atom * NT * 128)), "l"(&tmap), "r"(col0 + atom * 64),
                         "r"(base), "r"(su(&full[st]))
                         : "memory");
        }
      }
    }
  }
  __syncthreads();
  if (mode == 4) { asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;"); }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int rows = 8192, cols = 1024;  // 16 MB: L2 resident
  uint16_t* x; int* sel;
  CK(cudaMalloc(&x, (size_t)rows * cols * 2));
  CK(cudaMemset(x, 0, (size_t)rows * cols * 2));
  std::vector<int> h(rows);
  for (int i = 0; i < rows; ++i) h[i] = (int)((i * 2654435761u) % rows);
  CK(cudaMalloc(&sel, rows * 4));
  CK(cudaMemcpy(sel, h.data(), rows * 4, cudaMemcpyHostToDevice));
  void* fp; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  EncFn enc = (EncFn)fp;
  CUtensorMap gmap, tmap;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box1[2] = {64, 1}, boxT[2] = {64, NT}, es[2] = {1, 1};
  if (enc(&gmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, box1, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc1 fail\n"); return 1; }
  if (enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, boxT, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) { printf("enc2 fail\n"); return 1; }
  const int smem = S * STAGE + 2048;
  CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 2000;
  const char* names[] = {"gather4", "tma-row", "cp.async", "tma-tile(contig)", "gather4-mcast4", "cp.async-8w", "cp.async-2x4w-alt", "gather4-1thread", "hybrid g4x16+cp.async"};
  for (int mode = 0; mode < 9; ++mode) { if (mode == 4 || mode == 1 || mode == 5 || mode == 6) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = mode == 4 ? 4 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    if (mode == 4) cfg.gridDim = dim3(144);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      CK(cudaLaunchKernelEx(&cfg, bench, gmap, tmap, (const uint16_t*)x, cols, (const int*)sel, rows, iters, mode));
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)cfg.gridDim.x * iters * STAGE;
      if (rep) printf("%-18s %8.3f ms  %8.1f GB/s smem-fill  per-SM %6.1f B/clk@1.9GHz  stage %.0f ns\n", names[mode], ms,
                      bytes / ms / 1e6, bytes / cfg.gridDim.x / (ms * 1e-3) / 1.9e9, ms * 1e6 / iters);
    }
  }
  return 0;
}
