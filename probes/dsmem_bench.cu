// Microbenchmark (round 2): can two CTA pairs SHARE a SEL-gathered token stage over
// distributed shared memory instead of gathering it twice?  (The gate/up pair
// kernel is bound by the cp.async gather, probes/gather2_bench.cu: ~25 B/clk/SM.)
// Cluster of 4 CTAs; CTA c and c^2 need the same H-row token stage.  Mode 0: every
// CTA gathers all H rows itself (today's scheme).  Mode 1: each gathers H/2 rows by
// cp.async, waits for them, and pushes them to CTA c^2 with two smem->smem bulk
// copies (cp.async.bulk.shared::cluster.shared::cta, complete_tx on the peer's
// `full`).  A slot is refilled once both consumers (local + peer) released it.
// Optional HBM weight stream (19.5 KB per stage, as the pair kernel's A|E|planes).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probes/dsmem_bench probes/dsmem_bench.cu
#include <cuda_runtime.h>
#include <cstdint>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr int H = 112;
constexpr int STAGE = H * 256;
constexpr int S = 4;
constexpr int WST = 19456;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void arrive_tx(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void arrive_remote(uint32_t a) { asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory"); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}
__device__ __forceinline__ void wait_cta(uint64_t* b, uint32_t ph) {
  uint32_t d = 0;
  do { asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(d) : "r"(su(b)), "r"(ph) : "memory"); } while (!d);
}
__device__ __forceinline__ uint32_t swz(int row, int ch) {
  const int atom = ch >> 3, c8 = ch & 7;
  return atom * H * 128 + (row >> 3) * 1024 + (row & 7) * 128 + ((c8 ^ (row & 7)) << 4);
}

__global__ void __launch_bounds__(384, 1)
    bench(const uint16_t* x, int ldx, int nrows, const int* sel, int iters, int mode, int nwarps, const uint8_t* w,
          size_t wsize) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* wsm = sm + S * STAGE;
  uint64_t* full = (uint64_t*)(wsm + S * WST);
  uint64_t* empty = full + S;
  uint64_t* gathered = empty + S;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t crank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  uint32_t csize;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
  const uint32_t peer = crank ^ 2;
  const int nthr = nwarps * 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      // full: own gather threads + (mode 1) the expect_tx arrival for the peer's push + weights
      mbar_init(&full[s], nthr + (mode == 1 ? 1 : 0) + (w ? 1 : 0));
      mbar_init(&empty[s], mode == 1 ? 2 : 1);   // local consumer (+ the peer's consumer)
      mbar_init(&gathered[s], nthr);
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  // the token tile: shared by CTA c and c^2 (same rows); a new tile every 32 stages
  const int tile_id = csize == 4 ? blockIdx.x / 4 * 2 + (crank & 1) : blockIdx.x;
  if (warp == 10) {  // consumer: wait full, release local (+ peer) empty
    if (lane == 0)
      for (int it = 0; it < iters; ++it) {
        const int st = it % S;
        wait(&full[st], (it / S) & 1);
        arrive(&empty[st]);
        if (mode == 1) arrive_remote(mapa(su(&empty[st]), peer));
      }
  } else if (warp == 11 && w) {
    if (lane == 0)
      for (int it = 0; it < iters; ++it) {
        const int st = it % S;
        wait_cta(&empty[st], ((it / S) & 1) ^ 1);
        arrive_tx(&full[st], WST);
        const uint8_t* src = w + ((size_t)(blockIdx.x * (size_t)iters + it) * WST) % (wsize - WST) / 256 * 256;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su(wsm + st * WST)), "l"(src), "r"(WST), "r"(su(&full[st])) : "memory");
      }
  } else if (warp == 9 && mode == 1) {  // pusher: local half landed -> copy it into the peer's slot
    if (lane == 0)
      for (int it = 0; it < iters; ++it) {
        const int st = it % S;
        wait(&empty[st], ((it / S) & 1) ^ 1);          // both consumers released this slot everywhere
        arrive_tx(&full[st], STAGE / 2);               // the peer's push into MY slot
        wait_cta(&gathered[st], (it / S) & 1);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const int r0 = (crank >> 1) * (H / 2);        // my half of the rows
        for (int atom = 0; atom < 2; ++atom) {
          const uint32_t off = st * STAGE + atom * H * 128 + r0 * 128;
          asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(mapa(su(sm) + off, peer)), "r"(su(sm) + off), "r"(H / 2 * 128),
                       "r"(mapa(su(&full[st]), peer)) : "memory");
        }
      }
  } else if (warp < nwarps) {
    // source pointers / destinations per thread computed once per token tile (every
    // 32 stages), as the pair kernel does: a stage is then address add + cp.async
    const int tid = threadIdx.x, ch = tid & 15, rstep = nthr / 16;
    const int rows = mode == 1 ? H / 2 : H, r0 = mode == 1 ? (crank >> 1) * (H / 2) : 0;
    constexpr int MAXI = H / 4;  // 4 warps: 8 rows per pass
    const uint16_t* src[MAXI];
    uint32_t dst[MAXI];
    for (int it = 0; it < iters; ++it) {
      const int st = it % S;
      if (it % 32 == 0) {
        const int rbase = ((tile_id * 37 + it / 32) * H) % (nrows - H);
#pragma unroll
        for (int i = 0; i < MAXI; ++i) {
          const int row = r0 + (tid >> 4) + i * rstep;
          const bool ok = row < r0 + rows;
          src[i] = ok ? x + (size_t)sel[rbase + row] * ldx + ch * 8 : nullptr;
          dst[i] = ok ? swz(row, ch) : 0;
        }
      }
      wait_cta(&empty[st], ((it / S) & 1) ^ 1);
      const uint32_t b = su(sm + st * STAGE);
      const int col0 = (it * 128) % ldx;
#pragma unroll
      for (int i = 0; i < MAXI; ++i)
        if (src[i]) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(b + dst[i]), "l"(src[i] + col0) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(&full[st])) : "memory");
      if (mode == 1) asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(&gathered[st])) : "memory");
    }
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const int rows = 4096, cols = 4096;
  uint16_t* x; int* sel; uint8_t* wbuf;
  CK(cudaMalloc(&x, (size_t)rows * cols * 2));
  CK(cudaMemset(x, 0, (size_t)rows * cols * 2));
  std::vector<int> h(rows);
  for (int i = 0; i < rows; ++i) h[i] = (int)((i * 2654435761u) % rows);
  CK(cudaMalloc(&sel, rows * 4));
  CK(cudaMemcpy(sel, h.data(), rows * 4, cudaMemcpyHostToDevice));
  const size_t wsize = (size_t)1 << 30;
  CK(cudaMalloc(&wbuf, wsize));
  CK(cudaMemset(wbuf, 0, wsize));
  const int smem = S * (STAGE + WST) + 2048;
  CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const int iters = 3000;
  for (int cl : {1, 2, 4}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int nc = 0;
    CK(cudaOccupancyMaxActiveClusters(&nc, bench, &cfg));
    printf("cluster %d: max active clusters %d (%d CTAs)\n", cl, nc, nc * cl);
  }
  for (int ws : {0, 1})
    for (int nw : {4, 8})
      for (int mode : {2, 0, 1}) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
          cudaEventRecord(a);
          cudaLaunchConfig_t cfg = {};
          const int cl = mode == 2 ? 1 : 4;
          cfg.gridDim = dim3(mode == 2 ? 148 : 144); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = smem;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
          cfg.attrs = at; cfg.numAttrs = 1;
          CK(cudaLaunchKernelEx(&cfg, bench, (const uint16_t*)x, cols, rows, (const int*)sel, iters, mode == 2 ? 0 : mode, nw,
                                (const uint8_t*)(ws ? wbuf : nullptr), wsize));
          cudaEventRecord(b);
          CK(cudaEventSynchronize(b));
          CK(cudaGetLastError());
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (rep && ms < best) best = ms;
        }
        printf("weights %d gather warps %d %-26s %8.3f ms  stage %5.0f clk@1.9GHz (28 KB token stage per CTA)\n", ws, nw,
               mode == 1 ? "half gather + DSMEM push" : mode == 2 ? "full gather, no cluster" : "full gather per CTA (cl 4)", best, best * 1e-3 * 1.9e9 / iters);
      }
  return 0;
}
