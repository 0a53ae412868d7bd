// Microbenchmarks for the SIMT side of a remap on sm_100a (VERDICT r1 item 3,
// SURVEY §7 H1 "R2 / hybrid"): what it costs to move a tcgen05 partial product
// out of TMEM and add it into per-slot accumulators with CUDA cores.
//
//   1. FP32 pipe: FADD, FFMA, FADD2 (add.rn.f32x2), FFMA2 (fma.rn.f32x2) issue
//      rate per SM (8 independent chains per thread, 32 warps per SM).
//   2. tcgen05.ld bandwidth: 32x32b.x{16,32,64,128} with 4 / 8 / 16 warps per
//      SM, each warp reading its TMEM lane quadrant, bytes per clk per SM.
//   3. The R2 remap inner loop itself: per K-window partial P (128 lanes x N
//      fp32 columns in TMEM) -> registers -> acc[idx] += P (idx = the lane's
//      sub-row index bit), 4 and 8 warps, clk per window and N.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_bench tmem_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// ---------------------------------------------------------------- 1. FP32 pipes
template <int OP>  // 0 FADD, 1 FFMA, 2 FADD2, 3 FFMA2
__global__ void __launch_bounds__(1024, 1) fp_bench(int reps, float* sink, unsigned long long* clk) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  const float b = 1.0001f, c = 1e-7f;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) {
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[2 * i]) : "f"(c));
        asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(a[2 * i + 1]) : "f"(c));
      } else if (OP == 1) {
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[2 * i]) : "f"(b), "f"(c));
        asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[2 * i + 1]) : "f"(b), "f"(c));
      } else {
        uint64_t v = (uint64_t)__float_as_uint(a[2 * i]) | ((uint64_t)__float_as_uint(a[2 * i + 1]) << 32);
        const uint64_t bb = (uint64_t)__float_as_uint(b) | ((uint64_t)__float_as_uint(b) << 32);
        const uint64_t cc = (uint64_t)__float_as_uint(c) | ((uint64_t)__float_as_uint(c) << 32);
        if (OP == 2)
          asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v) : "l"(cc));
        else
          asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v) : "l"(bb), "l"(cc));
        a[2 * i] = __uint_as_float((uint32_t)v);
        a[2 * i + 1] = __uint_as_float((uint32_t)(v >> 32));
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
void run_fp(const char* name) {
  const int reps = 20000, threads = 1024;
  float* sink;
  unsigned long long* clk;
  cudaMalloc(&sink, 148 * threads * 4);
  cudaMalloc(&clk, 148 * 8);
  fp_bench<OP><<<148, threads>>>(reps, sink, clk);
  fp_bench<OP><<<148, threads>>>(reps, sink, clk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double lane_ops = 16.0 * reps * threads;  // fp32 element operations per SM
  const double instr = (OP >= 2 ? 8.0 : 16.0) * reps * threads / 32;
  printf("%-6s %7.1f fp32 element-ops/clk/SM  %6.2f warp-instr/clk/SM\n", name, lane_ops / c, instr / c);
  cudaFree(sink);
  cudaFree(clk);
}

// ---------------------------------------------------------------- 2. tcgen05.ld
template <int X>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[X]) {
  static_assert(X == 16 || X == 32 || X == 64 || X == 128, "x");
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  if constexpr (X == 16) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  } else {
#pragma unroll
    for (int h = 0; h < X / 16; ++h) {
      uint32_t* q = r + 16 * h;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]),
            "=r"(q[8]), "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15])
          : "r"(taddr + 16 * h));
    }
  }
}
__device__ __forceinline__ void tmem_ld32_one(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// MODE 0: x16 loads, 1: x32 (one instruction), 2: R2 remap (x16 loads + FADD2 into
// slot accumulators selected by a per-lane bit), 3: R2 remap with FADD (selp per element)
template <int MODE>
__global__ void tmem_bench(int reps, int ncols, float* sink, unsigned long long* clk) {
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  const int nwarps = blockDim.x >> 5;
  const int q = warp & 3, grp = warp >> 2, ngrp = nwarps >> 2;  // warps sharing a quadrant split the columns
  const uint32_t base = tm + ((uint32_t)(32 * q) << 16);
  float acc0[32], acc1[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc0[i] = acc1[i] = 0.f;
  const uint32_t bit = (lane * 0x9E3779B9u) >> 31;  // a per-lane "idx" (both values in every warp)
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int c = 32 * grp; c < ncols; c += 32 * ngrp) {
      float v[32];
      if (MODE == 1) {
        tmem_ld32_one(base + c, v);
      } else {
        tmem_ld<32>(base + c, v);
      }
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (MODE <= 1) {
#pragma unroll
        for (int i = 0; i < 32; ++i) acc0[i] += v[i];
      } else if (MODE == 2) {
        // acc_bit += v as FADD2 pairs: both slots get v masked by the lane's bit
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float m0 = bit ? 0.f : 1.f;
          uint64_t x = (uint64_t)__float_as_uint(v[i]) | ((uint64_t)__float_as_uint(v[i + 1]) << 32);
          uint64_t a0 = (uint64_t)__float_as_uint(acc0[i]) | ((uint64_t)__float_as_uint(acc0[i + 1]) << 32);
          uint64_t a1 = (uint64_t)__float_as_uint(acc1[i]) | ((uint64_t)__float_as_uint(acc1[i + 1]) << 32);
          const uint64_t mm0 = (uint64_t)__float_as_uint(m0) | ((uint64_t)__float_as_uint(m0) << 32);
          const uint64_t mm1 = (uint64_t)__float_as_uint(1.f - m0) | ((uint64_t)__float_as_uint(1.f - m0) << 32);
          asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a0) : "l"(x), "l"(mm0));
          asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a1) : "l"(x), "l"(mm1));
          acc0[i] = __uint_as_float((uint32_t)a0);
          acc0[i + 1] = __uint_as_float((uint32_t)(a0 >> 32));
          acc1[i] = __uint_as_float((uint32_t)a1);
          acc1[i + 1] = __uint_as_float((uint32_t)(a1 >> 32));
        }
      } else {
        // sum-and-slot1 form: acc0 accumulates everything, acc1 only the bit-1 lanes
        // (slot 0 = acc0 - acc1 at the end): one FADD + one FFMA per element
        const float m1 = bit ? 1.f : 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          acc0[i] += v[i];
          acc1[i] = fmaf(v[i], m1, acc1[i]);
        }
      }
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc0[i] + acc1[i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int MODE>
void run_tmem(const char* name, int warps, int ncols) {
  const int reps = 2000;
  float* sink;
  unsigned long long* clk;
  cudaMalloc(&sink, 148 * 1024 * 4);
  cudaMalloc(&clk, 148 * 8);
  tmem_bench<MODE><<<148, 32 * warps>>>(reps, ncols, sink, clk);
  tmem_bench<MODE><<<148, 32 * warps>>>(reps, ncols, sink, clk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148];
  cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double bytes = 128.0 * ncols * 4 * reps;  // the whole 128-lane x ncols region per rep
  printf("%-28s warps=%2d cols=%3d  %7.1f clk per 128x%d fp32 region  %6.1f B/clk/SM\n", name, warps, ncols,
         c / reps, ncols, bytes / c);
  cudaFree(sink);
  cudaFree(clk);
}

int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  run_fp<0>("FADD");
  run_fp<1>("FFMA");
  run_fp<2>("FADD2");
  run_fp<3>("FFMA2");
  for (int w : {4, 8, 16}) {
    run_tmem<0>("tcgen05.ld 32x32b.x16", w, 256);
    run_tmem<1>("tcgen05.ld 32x32b.x32", w, 256);
  }
  for (int w : {4, 8, 16}) {
    run_tmem<2>("R2 remap ld+FFMA2 (2 slots)", w, 224);
    run_tmem<3>("R2 remap ld+FADD+FFMA", w, 224);
  }
  return 0;
}
