// Microbenchmark (round 2): SEL-gather throughput into the SSMM's 128B-swizzled
// B stage with several stages IN FLIGHT (the round-1 gather_bench waited for each
// stage's cp.async group before the next, i.e. measured one stage of latency).
// Stage = H token rows x 2 K-atoms x 128 B (H = 112: the pair kernel's NT = 224
// half), S ring slots, one consumer thread that releases a slot after an optional
// busy time (emulating the MMA), 148 CTAs, source L2-resident (32 MB) or not.
//   mode 0: cp.async 16 B, 4 warps, cp.async.mbarrier.arrive.noinc (the kernel's scheme)
//   mode 1: same with 8 warps
//   mode 2: LDG.128 -> STS.128 register staging, 8 warps, then fence.proxy.async + arrive
//   mode 3: 2D TMA per row and atom (box 64 x 1), issued by the 32 lanes of one warp
//   mode 4: tile::gather4 TMA (4 rows per instruction), 32 lanes of one warp
//   mode 5: contiguous 2D TMA (box 64 x H) -- the no-gather reference
//   mode 6/7: cp.async with 12 / 16 warps; mode 8: 8 warps with the .L2::256B prefetch hint
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probes/gather2_bench probes/gather2_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int H = 112;
constexpr int STAGE = H * 256;
constexpr int SMAX = 4;
constexpr int WST = 19456;  // the pair kernel's weight tile per CTA and stage (A | E | planes)

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}
__device__ __forceinline__ uint32_t swz(int row, int ch) {  // byte offset of 16-B chunk ch (0..15) of row in a stage
  const int atom = ch >> 3, c8 = ch & 7;
  return atom * H * 128 + (row >> 3) * 1024 + (row & 7) * 128 + ((c8 ^ (row & 7)) << 4);
}

__global__ void __launch_bounds__(544, 1) bench(const __grid_constant__ CUtensorMap rmap, const __grid_constant__ CUtensorMap gmap,
                                               const __grid_constant__ CUtensorMap tmap, const uint16_t* x, int ldx, int nrows,
                                               const int* sel, int iters, int mode, int S, int busy,
                                               const uint8_t* w, size_t wsize) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* wsm = sm + SMAX * STAGE;
  uint64_t* full = (uint64_t*)(wsm + SMAX * WST);
  uint64_t* empty = full + SMAX;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nload = mode == 0 ? 4 : (mode == 1 || mode == 2 || mode == 8) ? 8 : mode == 6 ? 12 : 1;
  const bool cpa = mode <= 1 || mode >= 6;  // loader warps: 0..nload-1
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], (cpa ? nload * 32 : mode == 2 ? nload : 1) + (w ? 1 : 0));
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (warp == 16) {  // consumer
    if (lane == 0)
      for (int it = 0; it < iters; ++it) {
        const int st = it % S;
        wait(&full[st], (it / S) & 1);
        if (busy) { const long long t0 = clock64(); while (clock64() - t0 < busy) {} }
        arrive(&empty[st]);
      }
  } else if (warp == 15 && w) {  // weight stream (HBM), one bulk copy per stage
    if (lane == 0)
      for (int it = 0; it < iters; ++it) {
        const int st = it % S;
        wait(&empty[st], ((it / S) & 1) ^ 1);
        arrive_tx(&full[st], WST);
        const uint8_t* src = w + ((size_t)(blockIdx.x * (size_t)iters + it) * WST) % (wsize - WST) / 256 * 256;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su(wsm + st * WST)), "l"(src), "r"(WST), "r"(su(&full[st])) : "memory");
      }
  } else if (warp < nload) {
    const int tid = threadIdx.x, nthr = nload * 32;
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      wait(&empty[st], ((it / S) & 1) ^ 1);
      uint8_t* b = sm + st * STAGE;
      const int col0 = (it * 128) % ldx;
      const int rbase = ((blockIdx.x * 37 + it / 32) * H) % (nrows - H);  // a new token tile every 32 stages
      if (cpa) {
        for (int idx = tid; idx < H * 16; idx += nthr) {
          const int row = idx >> 4, ch = idx & 15;
          const uint16_t* src = x + (size_t)sel[rbase + row] * ldx + col0 + ch * 8;
          if (mode == 8)
            asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(su(b + swz(row, ch))), "l"(src) : "memory");
          else
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(b + swz(row, ch))), "l"(src) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(&full[st])) : "memory");
      } else if (mode == 2) {
        constexpr int PER = H * 16 / 256;  // 7 chunks per thread
        uint4 v[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int idx = tid + 256 * i, row = idx >> 4, ch = idx & 15;
          v[i] = __ldcg(reinterpret_cast<const uint4*>(x + (size_t)sel[rbase + row] * ldx + col0 + ch * 8));
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const int idx = tid + 256 * i, row = idx >> 4, ch = idx & 15;
          *reinterpret_cast<uint4*>(b + swz(row, ch)) = v[i];
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) arrive(&full[st]);
      } else {
        if (lane == 0) arrive_tx(&full[st], STAGE);
        __syncwarp();
        if (mode == 3) {
          for (int row = lane; row < H; row += 32)
            for (int atom = 0; atom < 2; ++atom)
              asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                           " [%0], [%1, {%2, %3}], [%4];" ::"r"(su(b + atom * H * 128 + row * 128)), "l"(&rmap),
                           "r"(col0 + atom * 64), "r"(sel[rbase + row]), "r"(su(&full[st]))
                           : "memory");
        } else if (mode == 4) {
          for (int g = lane; g < H / 4; g += 32)
            for (int atom = 0; atom < 2; ++atom) {
              const int* r = sel + rbase + 4 * g;
              asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                           " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(b + atom * H * 128 + g * 512)), "l"(&gmap),
                           "r"(col0 + atom * 64), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(su(&full[st]))
                           : "memory");
            }
        } else if (lane == 0) {
          for (int atom = 0; atom < 2; ++atom)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                         " [%0], [%1, {%2, %3}], [%4];" ::"r"(su(b + atom * H * 128)), "l"(&tmap), "r"(col0 + atom * 64),
                         "r"(rbase), "r"(su(&full[st]))
                         : "memory");
        }
      }
    }
  }
  __syncthreads();
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int rows = argc > 1 ? atoi(argv[1]) : 4096, cols = 4096;  // 4096 x 4096 bf16 = 32 MB (L2-resident)
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
  CUtensorMap rmap, gmap, tmap;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box1[2] = {64, 1}, boxT[2] = {64, H}, es[2] = {1, 1};
  auto E = [&](CUtensorMap* m, cuuint32_t* box) {
    if (enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("encode failed\n");
      exit(1);
    }
  };
  E(&rmap, box1);
  E(&gmap, box1);
  E(&tmap, boxT);
  const int smem = SMAX * (STAGE + WST) + 2048;
  uint8_t* wbuf;
  const size_t wsize = (size_t)1 << 30;
  CK(cudaMalloc(&wbuf, wsize));
  CK(cudaMemset(wbuf, 0, wsize));
  CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 3000;
  const char* names[] = {"cp.async 4w noinc", "cp.async 8w noinc", "ldg/sts 8w", "tma row 64x1", "tma gather4", "tma contig", "cp.async 12w", "cp.async 16w", "cp.async 8w L2::256B"};
  for (int ws : {0, 1})
    for (int S : {4})
      for (int mode = 0; mode < 7; ++mode) {
        const int busy = 0;
        if (mode == 3 || mode == 4) continue;
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
          cudaEventRecord(a);
          bench<<<148, 544, smem>>>(rmap, gmap, tmap, x, cols, rows, sel, iters, mode, S, busy, ws ? wbuf : nullptr, wsize);
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          CK(cudaGetLastError());
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (rep && ms < best) best = ms;
        }
        const double bytes = 148.0 * iters * (STAGE + (ws ? WST : 0));
        printf("weights %d S=%d %-18s %8.3f ms %8.1f GB/s  per-SM %6.1f B/clk@1.9GHz  stage %5.0f clk\n", ws, S, names[mode],
               best, bytes / best / 1e6, bytes / 148 / (best * 1e-3) / 1.9e9, best * 1e-3 * 1.9e9 / iters);
      }
  return 0;
}
