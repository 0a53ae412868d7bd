// Microbenchmark: the CTA-pair sparse MMA floor on sm_100a.
//
// One cluster of 2 CTAs per TPC (74 clusters).  The leader issues R
// tcgen05.mma.sp.cta_group::2.kind::f16 (M=256, K=32 logical, N tokens) with
// 256-bit disable_output_lane masks:
//   PAT 0  one warp, back to back, two accumulators alternating (the pipe floor)
//   PAT 1  the R1' pattern of the real kernel: two issuer warps (slot 0 / slot 1),
//          per 4-window stage a tcgen05.cp of the E tile, 4 windows x 1 slot MMA
//          each with the A / B descriptors stepping through the stage, one commit
//          per stage
// A from shared memory (AT 0) or TMEM (AT 1).  Optionally a background stream of
// bulk copies (L2 -> smem, 4 in flight per CTA, the ring fills of the real kernel)
// competes for shared-memory bandwidth; its achieved fill rate is reported.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o pair_mma_bench pair_mma_bench.cu
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
__device__ __forceinline__ uint32_t ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t par) {
  uint32_t done = 0;
  do {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(done)
                 : "r"(bar), "r"(par)
                 : "memory");
  } while (!done);
}
__device__ __forceinline__ void mma_sp2(uint32_t d, uint64_t ad, uint32_t a_tmem, bool a_in_tmem, uint64_t bd,
                                        uint32_t idesc, const uint32_t (&m)[8], uint32_t e) {
  if (!a_in_tmem)
    asm volatile(
        "{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%12], "
        "%3, {%4, %5, %6, %7, %8, %9, %10, %11}, 1;}" ::"r"(d),
        "l"(ad), "l"(bd), "r"(idesc), "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "r"(m[4]), "r"(m[5]), "r"(m[6]),
        "r"(m[7]), "r"(e));
  else
    asm volatile(
        "{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], [%1], %2, [%12], "
        "%3, {%4, %5, %6, %7, %8, %9, %10, %11}, 1;}" ::"r"(d),
        "r"(a_tmem), "l"(bd), "r"(idesc), "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "r"(m[4]), "r"(m[5]),
        "r"(m[6]), "r"(m[7]), "r"(e));
}

template <int N, int AT, int PAT, int VAR = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    bench(int reps, int bg_bytes, const uint8_t* gsrc, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[2], bgbars[4], dummy[2];
  __shared__ volatile int stop;
  uint8_t* A = sm;                 // 16 KB (4 K-windows of 128 x 16 bf16, sw128)
  uint8_t* B = sm + 16384;         // N/2 rows x 256 B (2 K-atoms of 64)
  uint8_t* E = B + (N / 2) * 256;  // 2 KB
  uint8_t* S = E + 2048;           // background copy target (4 x bg bytes)
  const uint32_t rank = ctarank();
  for (int i = threadIdx.x; i < (16384 + (N / 2) * 256 + 2048) / 4; i += 128)
    ((uint32_t*)sm)[i] = (i >= (16384 + (N / 2) * 256) / 4) ? 0x44444444u : 0x3c003c00u;
  __shared__ __align__(16) uint32_t planes[64];  // VAR&2: per-window lane-mask words (as the index bit-planes)
  if (threadIdx.x < 64) planes[threadIdx.x] = (threadIdx.x * 0x9E3779B9u) ^ 0x5bd1e995u * (threadIdx.x + 7);
  if (VAR & 1) {  // random valid 2:4 codes: nibbles from {(0,1),(0,2),(0,3),(1,2),(1,3),(2,3)}
    const uint8_t nib[6] = {0x4, 0x8, 0xC, 0x9, 0xD, 0xE};
    for (int i = threadIdx.x; i < 2048; i += 128) {
      uint32_t h = (uint32_t)i * 2654435761u;
      E[i] = (uint8_t)(nib[(h >> 8) % 6] | (nib[(h >> 16) % 6] << 4));
    }
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    stop = 0;
    for (int q = 0; q < 2; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[q])));
    for (int q = 0; q < 2; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&dummy[q])));
    for (int q = 0; q < 4; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bgbars[q])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  csync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  const int warp = threadIdx.x >> 5;
  const int nissue = PAT == 1 ? 2 : 1;
  if (warp < nissue && rank == 0) {
    const uint32_t idesc = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (16u << 24);
    const uint32_t acol = 464;  // A in TMEM (the contents do not matter for timing)
    const uint32_t ecol = 496 + 8 * warp;
    uint32_t m[8] = {0xAAAAAAAAu, 0x55555555u, 0xF0F0F0F0u, 0x0F0F0F0Fu,
                     0x33333333u, 0xCCCCCCCCu, 0x00FF00FFu, 0xFF00FF00u};
    if (warp == 1)
      for (int q = 0; q < 8; ++q) m[q] = ~m[q];
    asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.cp.cta_group::2.128x128b [%0], %1;}" ::"r"(
                     tm + ecol),
                 "l"(dint(su(E))));
    const uint32_t dcols = 2 * N + 16 <= 464 ? N : 0;  // two accumulators when they fit
    __syncwarp();
    unsigned long long t0 = clock64();
    if (PAT == 0) {
      const uint64_t ad = dsw128(su(A)), bd = dsw128(su(B));
      for (int r = 0; r < reps; ++r)
        mma_sp2(tm + (r & 1) * dcols, ad, tm + acol, AT, bd, idesc | (r & 1), m, tm + ecol);
    } else {
      // warp w = slot w: accumulator w, 4 windows per stage, E re-copied per stage
      const uint32_t d = tm + warp * dcols;
      for (int st = 0; st < reps / 8; ++st) {
        asm volatile("{.reg .pred p; elect.sync _|p, 0xffffffff; @p tcgen05.cp.cta_group::2.128x128b [%0], %1;}" ::"r"(
                         tm + ecol + (st & 1) * 4),
                     "l"(dint(su(E))));
        uint32_t pl[4][8];
        if (VAR & 2) {
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            const uint4 v = *reinterpret_cast<const uint4*>(&planes[(st * 8 + kb * 4) & 63]);
            const uint4 u = *reinterpret_cast<const uint4*>(&planes[(st * 8 + kb * 4 + 16) & 63]);
            pl[kb][0] = __reduce_or_sync(0xffffffffu, v.x);
            pl[kb][1] = __reduce_or_sync(0xffffffffu, v.y);
            pl[kb][2] = __reduce_or_sync(0xffffffffu, v.z);
            pl[kb][3] = __reduce_or_sync(0xffffffffu, v.w);
            pl[kb][4] = __reduce_or_sync(0xffffffffu, u.x);
            pl[kb][5] = __reduce_or_sync(0xffffffffu, u.y);
            pl[kb][6] = __reduce_or_sync(0xffffffffu, u.z);
            pl[kb][7] = __reduce_or_sync(0xffffffffu, u.w);
          }
        }
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          if (VAR & 2) {
#pragma unroll
            for (int q = 0; q < 8; ++q) m[q] = warp ? ~pl[kb][q] : pl[kb][q];
          }
          if (VAR & 4) {  // varying masks without the load / REDUX work: a register rotation
#pragma unroll
            for (int q = 0; q < 8; ++q) m[q] = (m[q] << 1) | (m[q] >> 31);
          }
          const uint64_t ad = dsw128(su(A) + kb * 32);
          const uint64_t bd = dsw128(su(B) + (kb / 2) * (N / 2) * 128 + (kb % 2) * 64);
          mma_sp2(d, ad, tm + acol + 8 * kb, AT, bd, idesc | (kb & 1), m, tm + ecol + (st & 1) * 4 + (kb & 2));
        }
        asm volatile(
            "{.reg .pred p; elect.sync _|p, 0xffffffff; @p "
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;}" ::"r"(
                su(&dummy[warp])),
            "h"((uint16_t)3));
      }
    }
    asm volatile(
        "{.reg .pred p; elect.sync _|p, 0xffffffff; @p "
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;}" ::"r"(
            su(&bar[warp])),
        "h"((uint16_t)3));
    wait_bar(su(&bar[warp]), 0);
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && warp == 0) out[blockIdx.x] = t1 - t0;
    if (warp == 0) {
      stop = 1;
      uint32_t rstop;
      asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(rstop) : "r"(su((const void*)&stop)));
      if (threadIdx.x == 0) asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(rstop), "r"(1) : "memory");
    }
  } else if (warp < nissue && rank == 1) {
    wait_bar(su(&bar[warp]), 0);  // the leader's commits multicast here too
  } else if (warp == 2 && bg_bytes > 0) {
    // background: bulk copies L2 -> smem, 4 in flight, until the MMAs are done
    if ((threadIdx.x & 31) == 0) {
      uint32_t par[4] = {0, 0, 0, 0};
      unsigned long long nbytes = 0;
      const unsigned long long c0 = clock64();
      int it = 0;
      auto issue = [&](int q) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bgbars[q])), "r"(bg_bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su(S + q * bg_bytes)),
            "l"(gsrc + (size_t)(it & 7) * bg_bytes), "r"(bg_bytes), "r"(su(&bgbars[q]))
            : "memory");
        ++it;
      };
      for (int q = 0; q < 4; ++q) issue(q);
      int q = 0;
      while (!stop) {
        wait_bar(su(&bgbars[q]), par[q]);
        par[q] ^= 1;
        nbytes += bg_bytes;
        issue(q);
        q = (q + 1) & 3;
      }
      for (int j = 0; j < 4; ++j) {
        wait_bar(su(&bgbars[q]), par[q]);
        par[q] ^= 1;
        q = (q + 1) & 3;
      }
      out[148 + blockIdx.x] = nbytes;
      out[296 + blockIdx.x] = clock64() - c0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  csync();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int AT, int PAT, int VAR = 0>
void run(const char* name, int bg) {
  const int reps = 4096;
  const int smem = 16384 + (N / 2) * 256 + 2048 + 4 * 32768 + 1024;
  cudaFuncSetAttribute(bench<N, AT, PAT, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 3 * 148 * 8);
  cudaMemset(d, 0, 3 * 148 * 8);
  uint8_t* g;
  cudaMalloc(&g, 8 * 32768);
  cudaMemset(g, 0, 8 * 32768);
  bench<N, AT, PAT, VAR><<<148, 128, smem>>>(reps, bg, g, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  bench<N, AT, PAT, VAR><<<148, 128, smem>>>(reps, bg, g, d);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  if (e != cudaSuccess) {
    printf("%s: %s\n", name, cudaGetErrorString(e));
    exit(1);
  }
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[3 * 148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double clk = 0, bgb = 0, bgc = 0;
  int n = 0;
  for (int i = 0; i < 148; i += 2) clk += h[i], ++n;
  clk /= n;
  for (int i = 0; i < 148; ++i) bgb += h[148 + i], bgc += h[296 + i];
  const double flops = 2.0 * 256 * N * 32 * reps * 74;
  printf("%-30s N=%3d bg=%5d B  %7.1f clk/MMA (pipe %5.1f)  %7.1f TFLOP/s issued  bg fill %5.1f B/clk/SM\n", name,
         N, bg, clk / reps, N / 2.0, flops / (ms * 1e-3) / 1e12, bgc > 0 ? bgb / bgc : 0.0);
  cudaFree(d);
  cudaFree(g);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  run<128, 0, 0>("floor A:smem", 0);
  run<224, 0, 0>("floor A:smem", 0);
  run<256, 0, 0>("floor A:smem", 0);
  run<224, 1, 0>("floor A:tmem", 0);
  run<224, 0, 1>("R1' 2 issuers A:smem", 0);
  run<224, 1, 1>("R1' 2 issuers A:tmem", 0);
  run<128, 0, 1>("R1' 2 issuers A:smem", 0);
  run<224, 0, 1, 1>("R1' 2 iss. random E", 0);
  run<224, 0, 1, 2>("R1' 2 iss. planes+REDUX masks", 0);
  run<224, 0, 1, 3>("R1' 2 iss. random E+masks", 0);
  run<208, 0, 1, 3>("R1' 2 iss. random E+masks", 0);
  run<224, 0, 1, 4>("R1' 2 iss. rotating masks", 0);
  run<224, 0, 1, 5>("R1' 2 iss. rand E+rot masks", 0);
  run<208, 0, 1, 3>("R1' 2 iss. random E+masks", 32768);
  for (int bg : {8192, 32768}) {
    run<224, 0, 0>("floor A:smem", bg);
    run<224, 0, 1>("R1' 2 issuers A:smem", bg);
    run<224, 1, 1>("R1' 2 issuers A:tmem", bg);
  }
  return 0;
}
