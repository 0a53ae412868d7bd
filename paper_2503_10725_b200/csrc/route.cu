// Routing (top-k + gate weights) and warp-level index compaction into
// per-expert selection arrays (§2.1 routing; P:239/P:303 SEL).
//
// Deterministic by construction: positions inside an expert's SEL are ranks
// by ascending token id, computed from per-warp expert bitmasks
// (popc(mask & lanemask_lt)) and fixed-order prefix sums -- no atomics decide
// any output position, so SEL is bit-exact against the oracle.
#include "internal.h"

namespace smy {

constexpr int kRouteThreads = 256;  // tokens per block
constexpr int kRouteWarps = kRouteThreads / 32;
constexpr int kMaxK = 16;  // top-k plus appended shared experts
constexpr int kMaxE = 256;

template <int V>
__device__ __forceinline__ void topk_warp(const float* __restrict__ lg, int E, int k, int gating, int lane,
                                          int32_t* __restrict__ ids, float* __restrict__ w) {
  float v[V];
  int rank[V];
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int e = lane + 32 * j;
    v[j] = e < E ? lg[e] : -INFINITY;
    if (isnan(v[j])) v[j] = -INFINITY;  // a NaN logit ranks as -inf (include/samoyeds.h, samoyeds_route)
    rank[j] = 0;
  }
#pragma unroll
  for (int jj = 0; jj < V; ++jj) {
    const int cols = min(32, E - 32 * jj);
    for (int src = 0; src < cols; ++src) {
      const float o = __shfl_sync(0xffffffffu, v[jj], src);
      const int oe = src + 32 * jj;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int e = lane + 32 * j;
        rank[j] += (o > v[j] || (o == v[j] && oe < e)) ? 1 : 0;
      }
    }
  }
  // the maximum logit (rank 0) and the normaliser
  float m = -INFINITY;
#pragma unroll
  for (int j = 0; j < V; ++j)
    if (lane + 32 * j < E) m = fmaxf(m, v[j]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < V; ++j)
    if (lane + 32 * j < E && (gating == SMY_GATE_SOFTMAX_ALL || rank[j] < k)) s += expf(v[j] - m);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
#pragma unroll
  for (int j = 0; j < V; ++j) {
    const int e = lane + 32 * j;
    if (e < E && rank[j] < k) {
      ids[rank[j]] = e;
      w[rank[j]] = expf(v[j] - m) / s;
    }
  }
}

// Writes the token's k routed entries, then its ns shared-expert entries (ids E..E+ns-1,
// weight 1: every token passes through every shared expert; reading R15) --
// the compaction then gives each shared expert a SEL of all tokens, so the grouped
// SSMM launches run shared and routed experts together.
__device__ __forceinline__ void topk_token(const float* __restrict__ lg, int E, int k, int gating, int lane,
                                           int32_t* __restrict__ ids, float* __restrict__ w, int ns = 0) {
  const int g = gating & ~SMY_GATE_SHARED_SIGMOID;
  if (E <= 32) topk_warp<1>(lg, E, k, g, lane, ids, w);
  else if (E <= 64) topk_warp<2>(lg, E, k, g, lane, ids, w);
  else if (E <= 128) topk_warp<4>(lg, E, k, g, lane, ids, w);
  else topk_warp<8>(lg, E, k, g, lane, ids, w);
  if (lane < ns) {
    ids[k + lane] = E + lane;
    // reading R15 (weight 1) or R15b (sigmoid of the shared expert's own logit column)
    w[k + lane] = (gating & SMY_GATE_SHARED_SIGMOID) ? 1.f / (1.f + expf(-lg[E + lane])) : 1.f;
  }
}

// Build per-warp expert masks for this block's tokens (from ids).
__device__ __forceinline__ void build_masks(const int32_t* __restrict__ ids, int64_t T, int E, int k,
                                            uint32_t (*mask)[kMaxE]) {
  for (int i = threadIdx.x; i < kRouteWarps * E; i += kRouteThreads) mask[i / E][i % E] = 0u;
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * kRouteThreads + threadIdx.x;
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (t < T)
    for (int i = 0; i < k; ++i) {
      const int key = ids[t * k + i];
      if (key >= 0 && key < E) atomicOr(&mask[w][key], 1u << l);  // keys outside [0, E): no entry
    }
  __syncthreads();
}

// Warp 0: exclusive scans over experts e < E of the counts c[e] and of the two
// SSMM launches' tile counts mt * ceil(c / nt) (lane l owns experts l*8 .. l*8+7,
// so the order is kept); writes off[e] (smem) and prefix0/1 (global, nullable).
__device__ __forceinline__ void scan_experts(const int32_t* __restrict__ cnt, int E, int lane, int32_t* __restrict__ off,
                                             int nt0, int mt0, int32_t* __restrict__ prefix0, int nt1, int mt1,
                                             int32_t* __restrict__ prefix1) {
  constexpr int PER = kMaxE / 32;
  int c[PER];
  int s0 = 0, s1 = 0, s2 = 0;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = lane * PER + j;
    c[j] = e < E ? cnt[e] : 0;
    s0 += c[j];
    s1 += prefix0 ? mt0 * ((c[j] + nt0 - 1) / nt0) : 0;
    s2 += prefix1 ? mt1 * ((c[j] + nt1 - 1) / nt1) : 0;
  }
  int i0 = s0, i1 = s1, i2 = s2;  // inclusive warp scans
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y0 = __shfl_up_sync(0xffffffffu, i0, o), y1 = __shfl_up_sync(0xffffffffu, i1, o),
              y2 = __shfl_up_sync(0xffffffffu, i2, o);
    if (lane >= o) {
      i0 += y0;
      i1 += y1;
      i2 += y2;
    }
  }
  int r0 = i0 - s0, r1 = i1 - s1, r2 = i2 - s2;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int e = lane * PER + j;
    if (e < E) {
      off[e] = r0;
      if (prefix0) prefix0[e] = r1;
      if (prefix1) prefix1[e] = r2;
    }
    r0 += c[j];
    r1 += prefix0 ? mt0 * ((c[j] + nt0 - 1) / nt0) : 0;
    r2 += prefix1 ? mt1 * ((c[j] + nt1 - 1) / nt1) : 0;
  }
  if (lane == 31) {
    off[E] = i0;
    if (prefix0) prefix0[E] = i1;
    if (prefix1) prefix1[E] = i2;
  }
}

// One warp per token over the whole grid (8 tokens per 256-thread block).
__global__ void route_topk_kernel(const float* __restrict__ logits, int64_t T, int E, int k, int gating,
                                  int32_t* __restrict__ ids, float* __restrict__ w, int ns) {
  const int lane = threadIdx.x % 32;
  const int64_t t = (int64_t)blockIdx.x * kRouteWarps + threadIdx.x / 32;
  if (t >= T) return;
  const int kk = k + ns;  // row stride: routed entries, then shared
  const int ld = E + ((gating & SMY_GATE_SHARED_SIGMOID) ? ns : 0);  // logits row: E router (+ ns shared-gate)
  topk_token(logits + t * ld, E, k, gating, lane, ids + t * kk, w + t * kk, ns);
}

__global__ void route_count_kernel(const int32_t* __restrict__ ids, int64_t T, int E, int k,
                                   int32_t* __restrict__ blk_counts) {
  __shared__ uint32_t mask[kRouteWarps][kMaxE];
  build_masks(ids, T, E, k, mask);
  for (int e = threadIdx.x; e < E; e += kRouteThreads) {
    int c = 0;
    for (int ww = 0; ww < kRouteWarps; ++ww) c += __popc(mask[ww][e]);
    blk_counts[(int64_t)blockIdx.x * E + e] = c;
  }
}

// T <= kRouteThreads: the whole routing + compaction in one block / one launch
// (top-k, masks, counts, offsets, tile prefixes, scatter).
__device__ __forceinline__ void small_route(const float* __restrict__ logits, int64_t T, int E, int k, int ns,
                                            int gating, int32_t* __restrict__ ids, float* __restrict__ w,
                                            int32_t* __restrict__ counts, int32_t* __restrict__ offsets, int nt0,
                                            int mt0, int32_t* __restrict__ prefix0, int nt1, int mt1,
                                            int32_t* __restrict__ prefix1, int32_t* __restrict__ sel,
                                            float* __restrict__ gw) {
  __shared__ uint32_t mask[kRouteWarps][kMaxE];
  __shared__ int32_t wbase[kRouteWarps][kMaxE];
  const int wp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (logits != nullptr) {
    // E, k here include the ns shared experts; the router covers the first E - ns
    for (int t = wp; t < T; t += kRouteWarps)
      topk_token(logits + (int64_t)t * ((gating & SMY_GATE_SHARED_SIGMOID) ? E : E - ns), E - ns, k - ns, gating,
                 lane, ids + (int64_t)t * k, w + (int64_t)t * k, ns);
  }
  __syncthreads();
  build_masks(ids, T, E, k, mask);
  __shared__ int32_t cnt[kMaxE];
  __shared__ int32_t off[kMaxE + 1];
  for (int e = threadIdx.x; e < E; e += kRouteThreads) {
    int c = 0;
    for (int ww = 0; ww < kRouteWarps; ++ww) c += __popc(mask[ww][e]);
    cnt[e] = c;
    counts[e] = c;
  }
  __syncthreads();
  if (wp == 0) scan_experts(cnt, E, lane, off, nt0, mt0, prefix0, nt1, mt1, prefix1);
  __syncthreads();
  for (int e = threadIdx.x; e <= E; e += kRouteThreads) {
    offsets[e] = off[e];
    if (e < E) wbase[0][e] = off[e];  // the expert's first row
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += kRouteThreads) {
    int run = wbase[0][e];
    for (int ww = 0; ww < kRouteWarps; ++ww) {
      wbase[ww][e] = run;
      run += __popc(mask[ww][e]);
    }
  }
  __syncthreads();
  const int t = threadIdx.x;
  if (t >= T) return;
  const uint32_t lt = (1u << lane) - 1u;
  for (int i = 0; i < k; ++i) {
    const int e = ids[(int64_t)t * k + i];
    if (e < 0 || e >= E) continue;
    const int pos = wbase[wp][e] + __popc(mask[wp][e] & lt);
    sel[pos] = t;
    gw[pos] = w[(int64_t)t * k + i];
  }
}

__global__ void route_small_kernel(const float* __restrict__ logits, int64_t T, int E, int k, int ns, int gating,
                                   int32_t* __restrict__ ids, float* __restrict__ w, int32_t* __restrict__ counts,
                                   int32_t* __restrict__ offsets, int nt0, int mt0, int32_t* __restrict__ prefix0,
                                   int nt1, int mt1, int32_t* __restrict__ prefix1, int32_t* __restrict__ sel,
                                   float* __restrict__ gw) {
  small_route(logits, T, E, k, ns, gating, ids, w, counts, offsets, nt0, mt0, prefix0, nt1, mt1, prefix1, sel, gw);
}

// 32 < T <= 64 in ONE launch: a cluster of 8 CTAs, one warp per token (token t on CTA
// t % 8), a cluster barrier (release / acquire at cluster scope) publishes ids / w, and
// CTA 0 compacts (small_route without the top-k).  (4 tokens per warp for T <= 256
// measured slower than the grid-wide top-k launch + one-block compaction.)
constexpr int kRouteCluster = 8;
__global__ void __cluster_dims__(kRouteCluster, 1, 1)
    route_cluster_kernel(const float* __restrict__ logits, int64_t T, int E, int k, int ns, int gating,
                         int32_t* __restrict__ ids, float* __restrict__ w, int32_t* __restrict__ counts,
                         int32_t* __restrict__ offsets, int nt0, int mt0, int32_t* __restrict__ prefix0, int nt1,
                         int mt1, int32_t* __restrict__ prefix1, int32_t* __restrict__ sel, float* __restrict__ gw) {
  const int wp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int ld = (gating & SMY_GATE_SHARED_SIGMOID) ? E : E - ns;  // logits row (E, k include the ns shared)
  for (int t = (int)blockIdx.x + kRouteCluster * wp; t < T; t += kRouteCluster * kRouteWarps)
    topk_token(logits + (int64_t)t * ld, E - ns, k - ns, gating, lane, ids + (int64_t)t * k, w + (int64_t)t * k, ns);
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (blockIdx.x != 0) return;
  small_route(nullptr, T, E, k, ns, gating, ids, w, counts, offsets, nt0, mt0, prefix0, nt1, mt1, prefix1, sel, gw);
}

// Single block: counts, offsets, per-block bases and SSMM tile prefixes.
__global__ void route_scan_kernel(const int32_t* __restrict__ blk_counts, int nblk, int E, int32_t* __restrict__ counts,
                                  int32_t* __restrict__ offsets, int32_t* __restrict__ blk_base, int nt0, int mt0,
                                  int32_t* __restrict__ prefix0, int nt1, int mt1, int32_t* __restrict__ prefix1) {
  __shared__ int32_t cnt[kMaxE];
  __shared__ int32_t off[kMaxE + 1];
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int c = 0;
    for (int b = 0; b < nblk; ++b) c += blk_counts[(int64_t)b * E + e];
    cnt[e] = c;
  }
  __syncthreads();
  if (threadIdx.x < 32) scan_experts(cnt, E, threadIdx.x, off, nt0, mt0, prefix0, nt1, mt1, prefix1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    counts[e] = cnt[e];
    offsets[e] = off[e];
    int run = off[e];
    for (int b = 0; b < nblk; ++b) {
      blk_base[(int64_t)b * E + e] = run;
      run += blk_counts[(int64_t)b * E + e];
    }
  }
  if (threadIdx.x == 0) offsets[E] = off[E];
}

__global__ void route_scatter_kernel(const int32_t* __restrict__ ids, const float* __restrict__ w, int64_t T, int E,
                                     int k, const int32_t* __restrict__ blk_base, int32_t* __restrict__ sel,
                                     float* __restrict__ gw) {
  __shared__ uint32_t mask[kRouteWarps][kMaxE];
  __shared__ int32_t wbase[kRouteWarps][kMaxE];
  build_masks(ids, T, E, k, mask);
  for (int e = threadIdx.x; e < E; e += kRouteThreads) {
    int run = blk_base[(int64_t)blockIdx.x * E + e];
    for (int ww = 0; ww < kRouteWarps; ++ww) {
      wbase[ww][e] = run;
      run += __popc(mask[ww][e]);
    }
  }
  __syncthreads();
  const int64_t t = (int64_t)blockIdx.x * kRouteThreads + threadIdx.x;
  if (t >= T) return;
  const int ww = threadIdx.x / 32, l = threadIdx.x % 32;
  const uint32_t lt = (1u << l) - 1u;
  for (int i = 0; i < k; ++i) {
    const int e = ids[t * k + i];
    if (e < 0 || e >= E) continue;
    const int pos = wbase[ww][e] + __popc(mask[ww][e] & lt);
    sel[pos] = (int32_t)t;
    gw[pos] = w[t * k + i];
  }
}

size_t route_ws_bytes(int64_t T, int E) {
  const int64_t nblk = (T + kRouteThreads - 1) / kRouteThreads;
  return (size_t)(2 * nblk * E) * sizeof(int32_t) + 256;
}

// Generic deterministic compaction of keys[T x k] (negative = no entry) into
// per-bucket lists of ascending row ids (and the aligned vals).
smy_status compact_launch(const int32_t* keys, const float* vals, int64_t T, int nb, int k, int32_t* counts,
                          int32_t* offsets, int32_t* sel, float* gw, void* ws, size_t ws_bytes, const int* tile_nt,
                          const int* tile_mt, int n_tile_cfgs, int32_t* tile_prefix, cudaStream_t s) {
  return route_launch(nullptr, T, nb, k, 0, const_cast<int32_t*>(keys), const_cast<float*>(vals), counts, offsets, sel,
                      gw, ws, ws_bytes, tile_nt, tile_mt, n_tile_cfgs, tile_prefix, s, 0);
}

smy_status route_launch(const float* logits, int64_t T, int E, int k, int gating, int32_t* ids, float* w,
                        int32_t* counts, int32_t* offsets, int32_t* sel, float* gw, void* ws, size_t ws_bytes,
                        const int* tile_nt, const int* tile_mt, int n_tile_cfgs, int32_t* tile_prefix,
                        cudaStream_t s, int ns) {
  // routed experts E, k; with ns shared experts appended the compaction runs over
  // E + ns buckets and k + ns entries per token (ids / w rows of stride k + ns)
  if (ns < 0 || ns > 32 || (ns > 0 && logits == nullptr)) return SMY_E_CONFIG;
  if (E + ns > kMaxE || k + ns > kMaxK || k < 1 || (logits != nullptr && k > E)) return SMY_E_CONFIG;
  const int Er = E, kr = k;
  E += ns;
  k += ns;
  if (ws_bytes < route_ws_bytes(T, E)) return SMY_E_WORKSPACE;
  const int nblk = (int)((T + kRouteThreads - 1) / kRouteThreads);
  int32_t* blk_counts = static_cast<int32_t*>(ws);
  int32_t* blk_base = blk_counts + (int64_t)nblk * E;
  const int nt0 = n_tile_cfgs > 0 ? tile_nt[0] : 1, mt0 = n_tile_cfgs > 0 ? tile_mt[0] : 0;
  const int nt1 = n_tile_cfgs > 1 ? tile_nt[1] : 1, mt1 = n_tile_cfgs > 1 ? tile_mt[1] : 0;
  int32_t* pre0 = n_tile_cfgs > 0 ? tile_prefix : nullptr;
  int32_t* pre1 = n_tile_cfgs > 1 ? tile_prefix + (E + 1) : nullptr;
  if (T <= kRouteThreads) {  // one block for the compaction (decode sizes)
    // up to 4 tokens per warp: top-k inside the same launch; more: a grid-wide
    // top-k launch first (one warp per token) so the block only compacts
    // (16 per warp measured slower than two launches; so were, at T = 64, E = 64: one
    // 1024-thread block doing both, top-k by argmax rounds, and one cooperative launch
    // with a grid barrier -- probes/route_ab.sh)
    // (fused top-k in the one block: one token per warp; 9..64 tokens: the cluster launch)
    const bool fused_topk = T <= ((debug_flags() & 268435456) ? 4 * kRouteWarps : kRouteWarps);
    if (logits != nullptr && !fused_topk && T <= kRouteCluster * kRouteWarps && !(debug_flags() & 268435456)) {
      // one launch: a cluster of 8 CTAs (SMY_DEBUG & 268435456: the two-launch path)
      route_cluster_kernel<<<kRouteCluster, kRouteThreads, 0, s>>>(logits, T, E, k, ns, gating, ids, w, counts,
                                                                  offsets, nt0, mt0, pre0, nt1, mt1, pre1, sel, gw);
      count_launch();
      return cuda_status(cudaGetLastError());
    }
    if (logits != nullptr && !fused_topk) {
      route_topk_kernel<<<(unsigned)((T + kRouteWarps - 1) / kRouteWarps), kRouteThreads, 0, s>>>(logits, T, Er, kr,
                                                                                                 gating, ids, w, ns);
      count_launch();
    }
    route_small_kernel<<<1, kRouteThreads, 0, s>>>(fused_topk ? logits : nullptr, T, E, k, ns, gating, ids, w, counts,
                                                   offsets, nt0, mt0, pre0, nt1, mt1, pre1, sel, gw);
    count_launch();
    return cuda_status(cudaGetLastError());
  }
  if (logits != nullptr) {
    route_topk_kernel<<<(unsigned)((T + kRouteWarps - 1) / kRouteWarps), kRouteThreads, 0, s>>>(logits, T, Er, kr,
                                                                                               gating, ids, w, ns);
    count_launch();
  }
  route_count_kernel<<<nblk, kRouteThreads, 0, s>>>(ids, T, E, k, blk_counts);
  count_launch();
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e);
  }
  route_scan_kernel<<<1, 256, 0, s>>>(blk_counts, nblk, E, counts, offsets, blk_base, nt0, mt0, pre0, nt1, mt1, pre1);
  count_launch();
  route_scatter_kernel<<<nblk, kRouteThreads, 0, s>>>(ids, w, T, E, k, blk_base, sel, gw);
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
