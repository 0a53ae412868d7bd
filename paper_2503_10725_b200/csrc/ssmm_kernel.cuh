#pragma once
// Samoyeds dual-side sparse SSMM for sm_100a (B200).
//
// C[t, o] = sum_k W[o, k] * x[sel[t], k]     (Alg. 1)
//
// B200 design:
//  * persistent CTAs (one per SM) walk a static tile schedule; a tile is 128
//    compressed weight rows (TMEM lanes) x NT selected tokens of one expert.
//    Grouped (MoE) launches decode the expert from a device-side tile prefix
//    written by the routing kernels -- the host never sees the counts;
//  * warp 4 is the producer: one cp.async.bulk per stage and weight streams the
//    pre-packed weight image (A smem image | E metadata TMEM image | index
//    bit-planes).  Token rows: when the expert's rows are contiguous (the
//    compact intermediate feeding down_proj -- the paper's compressed output
//    layout) warp 4 also issues one 2D TMA tile per stage; when they are
//    selected through SEL (gate/up) warps 6-9 gather x[sel[t]] with
//    cp.async straight from the token-major activations into the 128B-swizzled
//    K-major tile -- x is never permuted or copied (measured on B200: cp.async
//    sustains ~27 B/clk/SM of 128-B row gathers vs ~8 for tile::gather4,
//    probes/gather_bench.cu);
//  * warp 5 (one lane) copies E smem->TMEM (tcgen05.cp) and issues
//    tcgen05.mma.sp (bf16 -> fp32, K=32 = one V=32 sub-row window per MMA);
//  * the data-stationary remap of §4.3 ("the output of the SpTC must
//    be remapped to different rows ... according to the indices matrix") is done
//    by the tensor core: one TMEM accumulator per in-block sub-row slot p < M;
//    every MMA carries a 128-bit disable_output_lane mask built from the index
//    bit-planes so lane r only accumulates into slot idx[r][j];
//  * warps 0-3 run the fused epilogue straight from TMEM (compact store /
//    SiLU(gate)*up -> bf16 / routing-weight scale + scatter-add) and then
//    re-zero the accumulators for the next tile, while the producer is already
//    streaming that tile's operands.
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "ptx.cuh"

namespace smy {

// L2 prefetch distance (stages) of the row-expansion kernels' weight stream (0 = off)
#ifndef SMY_XP_PREFETCH
#define SMY_XP_PREFETCH 0
#endif
// expanded-stage ring depth of the (N, 2N, 32) row expansion (shared-memory units of 37 KB)
#ifndef SMY_XP_SLOTS
#define SMY_XP_SLOTS 2
#endif
template <int NT, int NW, int MS, int REP, int XP = 0>
struct Cfg {
  static constexpr int kWStride = 19456;                  // A|E|planes, 1024-aligned stride
  static constexpr int kBBytes = NT * 128 * (2 / REP);     // token tile per stage
  static constexpr int kStageBytes = NW * kWStride + kBBytes;
  // XP (in-smem row expansion of an (N, 2N, 32) image, N > 1): ring of expanded stages,
  // each = two 128-row A halves | their two E images | the enabled-lane masks
  static constexpr int kXMask = 2 * kABytes + 2 * kEBytes;
  static constexpr int kXUnit = XP ? kXMask + 1024 : 0;
  static constexpr int kXFit = (232448 - 1024 - 2048 - 2 * kStageBytes) / (kXMask + 1024);  // keep >= 2 stages
  static constexpr int kXSlots = XP ? (SMY_XP_SLOTS < kXFit ? SMY_XP_SLOTS : kXFit) : 0;
  static constexpr int kAccCols = NW * MS * NT;
  // two accumulator sets when they fit: the epilogue drains tile i while the
  // MMAs of tile i+1 run (decode-sized tiles)
  static constexpr int kAccBufs = 2 * kAccCols + 16 <= 512 ? 2 : 1;
  static constexpr int kECol = (kAccBufs * kAccCols + 3) / 4 * 4;
  static constexpr int kColsNeeded = kECol + 16;           // E: 2 stage buffers x 2 issuer warps x 4 cols
  static constexpr int kTmemCols = kColsNeeded <= 32    ? 32
                                   : kColsNeeded <= 64  ? 64
                                   : kColsNeeded <= 128 ? 128
                                   : kColsNeeded <= 256 ? 256
                                                        : 512;
  static constexpr int kAux = 2048;                        // barriers + gather row ids
  static constexpr int kSmemCap = 232448 - 1024 - kAux;
  static constexpr int kStagesRaw = (kSmemCap - kXSlots * kXUnit) / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kSmemBytes = kStages * kStageBytes + kXSlots * kXUnit + 1024 + kAux;
  static constexpr int kPlanes = MS == 1 ? 0 : MS == 2 ? 1 : MS == 4 ? 2 : MS == 8 ? 3 : 4;
  static_assert(kColsNeeded <= 512, "TMEM budget");
  static_assert(kStages >= 2, "smem budget");
  static_assert(NT % 16 == 0 && NT >= 16 && NT <= 256, "UMMA N");
};

// (SMY_SINGLE_FAST_GATHER_NT, internal.h: the widest token tile whose gather
// precomputes per-thread source pointers, NT/8 of them)
constexpr int kThreads = 352;  // warps 0-3 epilogue, 4 producer, 5 + 10 MMA, 6-9 gather
constexpr int kGatherThreads = 128;
// XP launches add warps 11-14: the in-smem row expansion
// XP expander warps 11-18 (thread = compressed row x window pair); 4 warps (all four
// windows per thread) measured slower: decode (4,8,32) 212 K vs 146 K tokens/s
#ifndef SMY_XP_WARPS
#define SMY_XP_WARPS 8
#endif
constexpr int kXWarps = SMY_XP_WARPS;
constexpr int threads_of(int xp) { return xp ? kThreads + 32 * kXWarps : kThreads; }

// Expanded row (0..255 of an m-tile's 2 x 128 TMEM lanes) of logical output row o of
// an (N, 2N, V) m-tile.  Interleaved gate/up weights (reading R20: blocks of 32 gate |
// 32 up output rows) are laid out so that every warp's 32 lanes hold 16 gate rows and
// the up rows of the same 16 outputs (lanes 0-15 / 16-31, the N = M epilogue pairing);
// other weights keep o.  Either way the rows of compressed rows [32w, 32w + 32) stay in
// [64w, 64w + 64).
__device__ __forceinline__ int xp_pos(int o, bool ilv) {
  if (!ilv) return o;
  const int i = o & 31, up = (o >> 5) & 1;
  return (o & ~63) + ((i >> 4) << 5) + (up << 4) + (i & 15);
}

struct TileInfo {
  int g, m_tile, t0, n_local, row0, k0, k1;  // k-stage range [k0, k1)
};

// Static schedule: tile index -> (expert, m_tile, n_tile).  n is the fastest
// index so CTAs running concurrently share the weight tile in L2.
//
// Stream-K tail (a.streamk, scatter-add epilogues only -- partial sums add): with
// `total` tiles over P workers, the first total - total % P tiles run whole; each
// of the last rem = total % P tiles is cut into s = P / rem K-ranges, so the last
// wave costs 1/s of a tile instead of a whole one.
__device__ __forceinline__ bool decode_tile(const SsmmArgs& a, int nt, int tile, TileInfo& ti) {
  int kpiece = 0, kpieces = 1;
  if (a.streamk) {
    const int total = a.tile_prefix != nullptr ? a.tile_prefix[a.num_groups] : a.max_tiles;
    const int P = a.workers, rem = total % P, full = total - rem;
    int s = rem ? P / rem : 1;
    if (s > a.k_stages) s = a.k_stages;
    if (s < 1) s = 1;
    if (tile >= full + rem * s) return false;
    if (tile >= full) {
      kpiece = (tile - full) % s;
      kpieces = s;
      tile = full + (tile - full) / s;
    }
  }
  int g = 0, local = tile;
  if (a.tile_prefix != nullptr) {
    if (tile >= a.tile_prefix[a.num_groups]) return false;
    int lo = 0, hi = a.num_groups - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (a.tile_prefix[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    g = lo;
    local = tile - a.tile_prefix[g];
  } else if (tile >= a.max_tiles) {
    return false;
  }
  const int row0 = a.offsets ? a.offsets[g] : 0;
  const int n_g = a.offsets ? a.offsets[g + 1] - row0 : a.n_sel;
  const int n_tiles = (n_g + nt - 1) / nt;
  ti.g = g;
  int mk, n_tile;                              // mk = (m_tile, k_split), k_split fastest
  if (a.m_fastest && n_tiles > 1) {
    // m fastest: concurrently running tiles share the token tile (B) in L2 -- the
    // down launch, whose B (the compact intermediate) is larger than its weights
    const int mk_count = a.tile_prefix != nullptr ? (a.tile_prefix[g + 1] - a.tile_prefix[g]) / n_tiles
                                                   : a.max_tiles / n_tiles;
    n_tile = local / mk_count;
    mk = local % mk_count;
  } else {
    mk = local / n_tiles;
    n_tile = local % n_tiles;
  }
  const int ksplits = a.k_splits > 1 ? a.k_splits : 1;
  ti.m_tile = mk / ksplits;
  const int kspl = mk % ksplits;
  const int per = (a.k_stages + ksplits - 1) / ksplits;
  ti.k0 = kspl * per;
  ti.k1 = min(a.k_stages, ti.k0 + per);
  if (kpieces > 1) {
    ti.k0 = kpiece * a.k_stages / kpieces;
    ti.k1 = (kpiece + 1) * a.k_stages / kpieces;
  }
  // the group's tokens are cut into n_tiles near-equal tiles (widths rounded up to
  // 16, the MMA N granule) rather than full tiles plus a ragged one: equal-cost
  // tiles balance the static schedule
  const int tper = (a.debug & 8192) ? nt : min(nt, (((n_g + n_tiles - 1) / n_tiles) + 15) & ~15);
  ti.t0 = n_tile * tper;
  ti.n_local = min(tper, n_g - ti.t0);
  ti.row0 = row0;
  return true;
}

// silu(g) * u (MUFU ex2 + rcp; measured faster here than hand-written .ftz PTX and
// than a one-MUFU tanh form -- the epilogue is not MUFU-bound)
#if SMY_SILU_TANH
// silu(g) = g/2 (1 + tanh(g/2)): one MUFU op (tanh.approx) instead of ex2 + rcp
__device__ __forceinline__ float silu_mul(float g, float u) {
  const float h = 0.5f * g;
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
  return fmaf(h, t, h) * u;
}
#else
__device__ __forceinline__ float silu_mul(float g, float u) { return __fdividef(g, 1.f + __expf(-g)) * u; }
#endif

// grid-stride zeroing of a.zero_ptr by `nthreads` threads (16-byte stores)
__device__ __forceinline__ void zero_slice(const SsmmArgs& a, int64_t tid, int64_t nthreads) {
  float4* z = reinterpret_cast<float4*>(a.zero_ptr);
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t i = tid; i < a.zero_elems / 4; i += nthreads) z[i] = zero;
}

// Row of gathered index rid: the local activations, or (expert parallelism over
// peer memory) the source rank's token row through its NVLink-mapped pointer.
__device__ __forceinline__ const uint16_t* x_row(const SsmmArgs& a, int rid) {
  if (a.row_map != nullptr) {
    const int m = a.row_map[rid];
    return a.x_peers[m >> 24] + (int64_t)(m & 0xFFFFFF) * a.ldx;
  }
  return a.x + (int64_t)rid * a.ldx;
}
// fp32 destination row of a scatter-add (EP: the source rank's output, P2P reductions)
__device__ __forceinline__ float* out_row(const SsmmArgs& a, int dst) {
  if (a.row_map != nullptr) {
    const int m = a.row_map[dst];
    return a.out_peers[m >> 24] + (int64_t)(m & 0xFFFFFF) * a.ldo;
  }
  return static_cast<float*>(a.out) + (int64_t)dst * a.ldo;
}

// Scatter-add of one 16-token chunk for the default (1,2,V) weights: lane l holds
// output columns (2 grp, 2 grp + 1) of 16 tokens (v0 / v1 = slot 0 / 1).  Lane pairs
// (l even, l + 1) cover 4 adjacent columns, so each token pair (j, j + 1) costs one
// shuffle of two values and ONE 16-byte red.add.v4 per lane -- even lanes write token
// j, odd lanes token j + 1 -- instead of one 8-byte reduction per lane and token.
// my_row / my_s: destination row and routing weight of token (lane & 15); n: tokens
// of the chunk this lane may write (0 if its rows are invalid).
__device__ __forceinline__ void scatter_chunk_v4(const float (&v0)[16], const float (&v1)[16], float* my_row,
                                                 float my_s, int n, int grp, int lane) {
  const int odd = lane & 1;
  const int col = 2 * (grp - odd);
#pragma unroll
  for (int j = 0; j < 16; j += 2) {
    const int mine = j + odd;                                  // the token this lane writes
    float* row = reinterpret_cast<float*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), mine));
    const float s = __shfl_sync(0xffffffffu, my_s, mine);
    const float r0 = __shfl_xor_sync(0xffffffffu, odd ? v0[j] : v0[j + 1], 1);
    const float r1 = __shfl_xor_sync(0xffffffffu, odd ? v1[j] : v1[j + 1], 1);
    if (mine < n) {
      float* o = row + col;
      if (odd) red_add_v4(o, s * r0, s * r1, s * v0[j + 1], s * v1[j + 1]);
      else red_add_v4(o, s * v0[j], s * v1[j], s * r0, s * r1);
    }
  }
}

// Interleaved gate/up epilogue (kEpiSiluMulIlv, reading R20) for one 16-column
// chunk of one warp: its 32 TMEM lanes are 16 gate rows (lanes 0-15) and the up
// rows of the same 16 output pairs (lanes 16-31); v[slot][col].  Per column one
// shuffle swaps what each half lacks -- the gate lane takes u of slot 0, the up
// lane g of slot 1 -- so all 32 lanes compute one bf16(silu(g) * u) and the warp
// stores 32 consecutive outputs (64 B).  No shared memory, no barrier.
__device__ __forceinline__ void ilv_chunk(const float (&v)[2][16], bool valid, int jmax, uint16_t* out, int64_t ldo,
                                          int64_t row_base, int cg, int lane, const int32_t* rows_out = nullptr) {
  const bool is_up = lane >= 16;
  // token pair (c, c+1): the gate lane finishes both slots of token c, the up lane
  // both slots of token c+1 -- two shuffles swap what each lacks, and each lane
  // stores its two adjacent outputs as one bf16x2 (the epilogue is issue-bound)
  uint32_t packed[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = 2 * j;
    const float r0 = __shfl_xor_sync(0xffffffffu, is_up ? v[0][c] : v[0][c + 1], 16);
    const float r1 = __shfl_xor_sync(0xffffffffu, is_up ? v[1][c] : v[1][c + 1], 16);
    const float g0 = is_up ? r0 : v[0][c], u0 = is_up ? v[0][c + 1] : r0;
    const float g1 = is_up ? r1 : v[1][c], u1 = is_up ? v[1][c + 1] : r1;
    const __nv_bfloat162 h = __floats2bfloat162_rn(silu_mul(g0, u0), silu_mul(g1, u1));
    packed[j] = *reinterpret_cast<const uint32_t*>(&h);
  }
  const int n = valid ? jmax : 0;
  if (rows_out != nullptr) {  // ablation only (SMY_VARIANT_DENSE_INTER): row r goes to rows_out[r]
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = 2 * j + (is_up ? 1 : 0);
      if (t < n) *reinterpret_cast<uint32_t*>(out + (int64_t)rows_out[row_base + t] * ldo + 2 * cg) = packed[j];
    }
    return;
  }
  uint32_t* o = reinterpret_cast<uint32_t*>(out + (row_base + (is_up ? 1 : 0)) * ldo + 2 * cg);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (2 * j + (is_up ? 1 : 0) < n) *o = packed[j];
    o += ldo;  // two rows of ldo bf16 = ldo 32-bit words
  }
}

// The same for N = M weights (one accumulator slot): lanes 0-15 gate, 16-31 up
// rows of the same 16 outputs; per column pair one shuffle, the gate lane computes
// the even token, the up lane the odd one.
__device__ __forceinline__ void ilv_chunk_ms1(const float (&v)[16], bool valid, int jmax, uint16_t* out, int64_t ldo,
                                              int64_t row_base, int cg, int lane) {
  const bool is_up = lane >= 16;
  uint16_t act[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float recv = __shfl_xor_sync(0xffffffffu, is_up ? v[2 * j] : v[2 * j + 1], 16);
    act[j] = __bfloat16_as_ushort(
        __float2bfloat16_rn(is_up ? silu_mul(recv, v[2 * j + 1]) : silu_mul(v[2 * j], recv)));
  }
  uint16_t* o = out + (row_base + (is_up ? 1 : 0)) * ldo + cg;
  const int n = valid ? jmax : 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (2 * j + (is_up ? 1 : 0) < n) *o = act[j];
    o += 2 * ldo;
  }
}

__device__ __forceinline__ void tma_tile2d(void* dst, const CUtensorMap* map, int col, int row, uint64_t* bar,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(col), "r"(row), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

template <int NT, int NW, int MS, int REP, int XP = 0>
__global__ void __launch_bounds__(threads_of(XP), 1) ssmm_kernel(const __grid_constant__ SsmmArgs a) {
  constexpr int kIssuers = (NW == 2 || MS >= 2) ? 2 : 1;  // MMA-issuing warps
  using C = Cfg<NT, NW, MS, REP, XP>;
  constexpr int S = C::kStages;
  // XP: the weight image is an (N, 2N, 32) format, N > 1.  Warps 11-14
  // expand each compressed stage into two 128-row halves of output rows: compressed row
  // r's window-j values / metadata move to expanded row (r / N) * 2N + idx[r][j] and the
  // MMA of half h enables only the lanes some compressed row landed on.  Two unmasked-
  // layout MMAs per window (as the (1,2,V) remap issues), whatever M is.
  static_assert(!XP || (NW == 1 && MS == 2 && REP == 1), "XP: one weight, two halves");
  constexpr int XS = C::kXSlots;
  // a dependent launch (the down SSMM after gate/up, SsmmArgs::pdl) may start its
  // prologue and weight stream on SMs this grid has left
  if (threadIdx.x == 0) griddep_launch_dependents();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aux = smem + S * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;      // [kAccBufs]
  uint64_t* acc_empty = acc_full + 2;  // [kAccBufs]
  uint64_t* xfull = acc_empty + 2;     // [XS <= 4] expanded stage written (4 expander warps)
  uint64_t* xempty = xfull + 4;        // [XS <= 4] expanded stage consumed (issuer commits)
  // XP + SEL gather: the gathered token rows complete on their own barrier, so the
  // expander (which needs only the weight block) is not held behind the gather
  uint64_t* bfull = XP ? xempty + 4 : full;  // [S]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty + 4 + (XP ? 8 : 0));
  static_assert(C::kXSlots <= 4, "XP barrier slots");
  constexpr int AB = C::kAccBufs;
  int32_t* rows = reinterpret_cast<int32_t*>(aux + 1024);  // gather row ids of the current tile
  const bool gather = a.sel_in != nullptr;

  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], gather && !XP ? 1 + kGatherThreads : 1);
      if (XP && gather) mbar_init(&bfull[s], kGatherThreads);
      mbar_init(&empty[s], kIssuers + (XP ? kXWarps : 0));  // XP: the expander warps also read the stage
    }
    for (int b = 0; b < AB; ++b) {
      mbar_init(&acc_full[b], kIssuers);
      mbar_init(&acc_empty[b], 4);
    }
    for (int x = 0; x < XS; ++x) {
      mbar_init(&xfull[x], kXWarps);  // every expander warp
      mbar_init(&xempty[x], kIssuers);
    }
    fence_mbar_init();
  }
  if (warp == 5) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto wsm = [&](int st, int w) { return smem + st * C::kStageBytes + w * C::kWStride; };
  auto bsm = [&](int st) { return smem + st * C::kStageBytes + NW * C::kWStride; };
  auto xsm = [&](int x) { return smem + S * C::kStageBytes + x * C::kXUnit; };
  const int ks = a.k_stages;
  const int tile0 = blockIdx.x, tstep = gridDim.x;
  // SMY_DEBUG & 128: per-role cycle counters (same slots as the pair kernel)
  const bool prof = a.prof != nullptr;
  unsigned long long pc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  auto clk = []() { unsigned long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; };

  if (warp == 4) {
    // ========== producer: weight image (bulk) + contiguous token tile (2D TMA) ==========
    if (lane == 0) {
      const uint32_t wbytes = kABytes + kEBytes + 64 * (XP ? a.planes : C::kPlanes);
      const uint32_t stage_bytes = NW * wbytes + (gather ? 0u : (uint32_t)C::kBBytes);
      const uint64_t pol_w = a.weights_stream ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_x = policy_evict_last();
      uint32_t it = 0;
      TileInfo ti;
      // programmatic dependent launch: the first ring of stages gets its weights at once,
      // their token loads (the previous kernel's output) wait for griddepcontrol.wait
      const bool defer = a.pdl && !gather;
      int npend = 0, pend_k[S], pend_row[S];
      auto load_b = [&](int st, int k, int xrow) {
#pragma unroll
        for (int atom = 0; atom < 2 / REP; ++atom)
          tma_tile2d(bsm(st) + atom * (NT * 128), &a.tmap_x, k * (128 / REP) + atom * 64, xrow, &full[st], pol_x);
      };
      auto flush = [&]() {
        griddep_wait();
        for (int i = 0; i < npend; ++i) load_b(i, pend_k[i], pend_row[i]);
        npend = -1;
      };
      for (int tile = tile0; decode_tile(a, NT, tile, ti); tile += tstep) {
        const uint8_t* src0 = a.img0[ti.g] + (size_t)ti.m_tile * ks * a.block;
        const uint8_t* src1 = NW == 2 ? a.img1[ti.g] + (size_t)ti.m_tile * ks * a.block : nullptr;
        const int xrow = ti.row0 + ti.t0;
        for (int k = ti.k0; k < ti.k1; ++k, ++it) {
          const int st = it % S;
          if (defer && npend >= 0 && it >= (uint32_t)S) flush();  // the ring is full: tokens next
          const unsigned long long t0 = prof ? clk() : 0;
          mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
          if (prof) pc[5] += clk() - t0;
          const bool skip_w = a.debug & 2;
          mbar_arrive_expect_tx(&full[st], stage_bytes - (skip_w ? NW * wbytes : 0u));
          if (!skip_w) {
            bulk_g2s(wsm(st, 0), src0 + (size_t)k * a.block, wbytes, &full[st], pol_w);
            // XP: the expanded units leave fewer stages in flight -- pull the block
            // SMY_XP_PREFETCH stages ahead into L2 (no shared memory needed for that)
            if (XP && SMY_XP_PREFETCH > 0 && k + SMY_XP_PREFETCH < ti.k1)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src0 + (size_t)(k + SMY_XP_PREFETCH) * a.block),
                           "r"(wbytes)
                           : "memory");
            if (NW == 2) bulk_g2s(wsm(st, 1), src1 + (size_t)k * a.block, wbytes, &full[st], pol_w);
          }
          if (!gather) {
            if (defer && npend >= 0) {
              pend_k[npend] = k;
              pend_row[npend] = xrow;
              ++npend;
            } else {
              load_b(st, k, xrow);
            }
          }
        }
      }
      if (defer && npend >= 0) flush();
    }
  } else if (warp == 5 || warp == 10) {
    // ============ MMA issuers (warps 5 and 10; whole warp, one elected lane) ============
    // Per-stage issue work (plane words -> uniform lane masks, descriptors,
    // elect) is as long as the MMAs at decode sizes, so two warps split it:
    // NW == 2 -> warp mi issues weight mi; NW == 1 -> slots p = mi (mod 2).
    // tcgen05.commit tracks the issuing thread's MMAs, so each issuer commits and
    // `empty` / `acc_full` expect kIssuers arrivals.  Each warp copies the E tile
    // it uses into its own TMEM columns (ordered before its own MMAs).
    const int mi = warp == 10 ? 1 : 0;
    if (mi < kIssuers) {
    // N of a tile = its token count rounded up to 16 (ragged tiles issue narrower MMAs)
    constexpr uint32_t idesc0 = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 4) << 24);
    const int we = NW == 2 ? mi : 0;  // the weight whose E this warp needs
    const uint32_t smem_base = smem_u32(smem);
    // redux.sync results live in uniform registers: keeps every MMA operand uniform
    // so the compiler issues UTCHMMA without a per-instruction R2UR waterfall
    const uint32_t tm = __reduce_or_sync(0xffffffffu, tmem);
    uint32_t it = 0, tcount = 0;
    TileInfo ti;
    const unsigned long long tstart = prof ? clk() : 0;
    for (int tile = tile0; decode_tile(a, NT, tile, ti); tile += tstep, ++tcount) {
      unsigned long long t0 = prof ? clk() : 0;
      const int ab = tcount % AB;
      const uint32_t tacc = tm + ab * C::kAccCols;
      mbar_wait(&acc_empty[ab], (tcount / AB) & 1);  // this accumulator set drained and re-zeroed
      if (prof) pc[1] += clk() - t0;
      tc_fence_after();
      const uint32_t idesc =
          __reduce_or_sync(0xffffffffu, idesc0 | ((uint32_t)(((ti.n_local + 15) >> 4) << 4) >> 3) << 17);
      for (int k = ti.k0; k < ti.k1; ++k, ++it) {
        const int st = it % S;
        t0 = prof ? clk() : 0;
        mbar_wait(&full[st], (it / S) & 1);
        if (prof) pc[0] += clk() - t0;
        tc_fence_after();
        const uint32_t sbase = smem_base + st * C::kStageBytes;
        // E double-buffered in TMEM: this stage's copy does not overwrite columns
        // the previous stage's MMAs may still be reading
        const uint32_t ecol = C::kECol + (it & 1) * 8 + 4 * mi;
        if constexpr (XP != 0) {
          // expanded half mi of this stage: A rows, E image, enabled-lane masks
          const int xs = it % XS;
          t0 = prof ? clk() : 0;
          if (gather) mbar_wait(&bfull[st], (it / S) & 1);
          mbar_wait(&xfull[xs], (it / XS) & 1);
          if (prof) pc[0] += clk() - t0;
          tc_fence_after();
          const uint32_t xb = smem_base + S * C::kStageBytes + xs * C::kXUnit;
          tc_cp_128x128b_elect(tm + ecol, desc_interleave(xb + 2 * kABytes + mi * kEBytes));
          uint4 ens[4];  // all four windows' masks first: the LDS latency off the MMA issue chain
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) ens[kb] = lds_v4(xb + C::kXMask + (mi * 4 + kb) * 16);
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            const uint4 en = ens[kb];
            const uint64_t bdesc = desc_sw128(sbase + C::kWStride + (kb / 2) * (NT * 128) + (kb % 2) * 64);
            // (SMY_DEBUG & 16777216: both halves' MMAs read half 0's A -- timing probe, results wrong)
            const uint64_t adesc = desc_sw128(xb + ((a.debug & 16777216) ? 0 : mi) * kABytes + kb * 32);
            if (!(a.debug & 4))
              tc_mma_sp_elect(tacc + mi * NT, adesc, bdesc, idesc | (uint32_t)(kb & 1), ~en.x, ~en.y, ~en.z, ~en.w,
                              tm + ecol + (kb & 2));
          }
          tc_commit_elect(&empty[st]);
          tc_commit_elect(&xempty[xs]);
          continue;
        }
        tc_cp_128x128b_elect(tm + ecol, desc_interleave(sbase + we * C::kWStride + kABytes));
        // index bit-planes of this stage (this warp's weight): LDS, no redux (see ssmm_pair.cuh)
        uint32_t pl[4][C::kPlanes > 0 ? C::kPlanes : 1][4];
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
          for (int b = 0; b < C::kPlanes; ++b) {
            const uint4 v = lds_v4(smem_u32(wsm(st, we)) + kABytes + kEBytes + (kb * C::kPlanes + b) * 16);
            pl[kb][b][0] = v.x;
            pl[kb][b][1] = v.y;
            pl[kb][b][2] = v.z;
            pl[kb][b][3] = v.w;
          }
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          const int e0 = (kb / REP) * 32;  // first B element of this K=32 window
          const uint64_t bdesc = desc_sw128(sbase + NW * C::kWStride + (e0 / 64) * (NT * 128) + (e0 % 64) * 2);
          const uint64_t adesc = desc_sw128(sbase + we * C::kWStride + kb * 32);
#pragma unroll
          for (int p = 0; p < MS; ++p) {
            if (NW == 1 && kIssuers == 2 && (p & 1) != mi) continue;
            uint32_t mask[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t en = 0xffffffffu;
#pragma unroll
              for (int b = 0; b < C::kPlanes; ++b) en &= ((p >> b) & 1) ? pl[kb][b][q] : ~pl[kb][b][q];
              mask[q] = MS == 1 ? 0u : ~en;
            }
            // metadata column of this K=32 window: even part in the address,
            // the odd bit in idesc.sparse_id2 (bits [0,2))
            if (!(a.debug & 4))
              tc_mma_sp_elect(tacc + (we * MS + p) * NT, adesc, bdesc, idesc | (uint32_t)(kb & 1), mask[0], mask[1],
                              mask[2], mask[3], tm + ecol + (kb & 2));
          }
        }
        tc_commit_elect(&empty[st]);
      }
      tc_commit_elect(&acc_full[ab]);
      pc[7] += 1;
    }
    if (prof) pc[2] = clk() - tstart;
    }
  } else if (warp >= 11) {
    if constexpr (XP != 0) {
    // ============ XP: in-smem row expansion (warps 11-14, thread = compressed row) ============
    // Thread = (compressed row t of the m-tile, window group wp): per stage it moves the
    // row's values / metadata of windows [XW wp, XW wp + XW) from the TMA-staged compressed
    // block to their expanded rows (all loads first, then the stores).
    constexpr int XW = 16 / kXWarps;  // windows per thread
    const int tt = threadIdx.x - kThreads, t = tt & 127, wp = tt >> 7, w4 = t >> 5;
    const int P = a.planes, N = a.n_fmt, M = a.m_fmt;
    const bool ilvp = a.epi == kEpiSiluMulIlv;
    const int gbase = (t / N) * M;  // first logical output row of this row's group (in the m-tile)
    const uint32_t a_src = (uint32_t)((t >> 3) * 1024 + (t & 7) * 128), a_sw = (uint32_t)(t & 7);
    const uint32_t e_src0 = kABytes + 16u * ((t & 7) + 16 * (t >> 4)) + 2u * ((t >> 3) & 1);
    // stale rows are never enabled; start from zero values and valid (0,1) metadata anyway
    for (int i = tt; i < XS * C::kXUnit / 16; i += 32 * kXWarps) {
      const int off = (i * 16) % C::kXUnit;
      const uint32_t v = off >= 2 * kABytes && off < C::kXMask ? 0x44444444u : 0u;
      reinterpret_cast<uint4*>(xsm(0))[i] = make_uint4(v, v, v, v);
    }
    uint32_t it = 0;
    TileInfo ti;
    for (int tile = tile0; decode_tile(a, NT, tile, ti); tile += tstep) {
      for (int k = ti.k0; k < ti.k1; ++k, ++it) {
        const int st = it % S, xs = it % XS;
        unsigned long long tx0 = prof ? clk() : 0;
        mbar_wait(&full[st], (it / S) & 1);
        if (prof) { const unsigned long long t1 = clk(); pc[8] += t1 - tx0; tx0 = t1; }
        const uint8_t* cw = wsm(st, 0);
        uint4 av[2 * XW];
#pragma unroll
        for (int c = 0; c < 2 * XW; ++c)
          av[c] = *reinterpret_cast<const uint4*>(cw + a_src + (((2 * XW * wp + c) ^ a_sw) << 4));
        uint16_t ev[XW][2];
        int p[XW];
#pragma unroll
        for (int j = 0; j < XW; ++j) {
          const int kb = XW * wp + j;
          p[j] = 0;
#pragma unroll
          for (int k1 = 0; k1 < 2; ++k1) ev[j][k1] = *reinterpret_cast<const uint16_t*>(cw + e_src0 + 128 * k1 + 4 * kb);
          for (int b = 0; b < P; ++b)
            p[j] |= (int)((*reinterpret_cast<const uint32_t*>(cw + kABytes + kEBytes + (kb * P + b) * 16 + w4 * 4) >>
                           lane) & 1u) << b;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // the compressed block is read (the MMAs release B)
        mbar_wait(&xempty[xs], ((it / XS) & 1) ^ 1);
        if (prof) { const unsigned long long t1 = clk(); pc[9] += t1 - tx0; tx0 = t1; }
        uint8_t* xu = xsm(xs);
#pragma unroll
        for (int j = 0; j < XW; ++j) {
          const int kb = XW * wp + j;
          const int pos = xp_pos(gbase + p[j], ilvp);  // in [64 w4, 64 w4 + 64)
          const int h = pos >> 7, r = pos & 127;
          uint8_t* arow = xu + h * kABytes + (r >> 3) * 1024 + (r & 7) * 128;
          // A: the window's two 16-B chunks (128B swizzle: chunk c of row r at c ^ (r % 8))
          *reinterpret_cast<uint4*>(arow + (((2 * kb) ^ (r & 7)) << 4)) = av[2 * j];
          *reinterpret_cast<uint4*>(arow + (((2 * kb + 1) ^ (r & 7)) << 4)) = av[2 * j + 1];
          // E: the row's 16-bit code word of each K-half (lane (row % 8) + 8 k1 + 16 (row / 16),
          // bits 16 ((row / 8) % 2) of the window's 32-bit column)
          uint8_t* erow = xu + 2 * kABytes + h * kEBytes + 16 * ((r & 7) + 16 * (r >> 4)) + 4 * kb + 2 * ((r >> 3) & 1);
          *reinterpret_cast<uint16_t*>(erow) = ev[j][0];
          *reinterpret_cast<uint16_t*>(erow + 128) = ev[j][1];
          const int loc = pos - 64 * w4;
          const uint32_t m0 = __reduce_or_sync(0xffffffffu, loc < 32 ? 1u << loc : 0u);
          const uint32_t m1 = __reduce_or_sync(0xffffffffu, loc >= 32 ? 1u << (loc - 32) : 0u);
          if (lane == 0)
            *reinterpret_cast<uint2*>(xu + C::kXMask + ((w4 >> 1) * 4 + kb) * 16 + 8 * (w4 & 1)) = make_uint2(m0, m1);
        }
        if (prof) { const unsigned long long t1 = clk(); pc[11] += t1 - tx0; tx0 = t1; }
        // generic-proxy writes -> tcgen05.cp / tcgen05.mma reads (SMY_DEBUG & 33554432: skipped, timing probe)
        if (!(a.debug & 33554432)) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xfull[xs]);
        if (prof) pc[6] += clk() - tx0;
      }
    }
    }
  } else if (warp >= 6 && warp < 10) {
    // ================== SEL gather of token rows (warps 6-9, cp.async) ==================
    if (gather && REP == 1 && NT <= SMY_SINGLE_FAST_GATHER_NT) {
      // Thread tb owns 16-B chunk ch = tb % 16 of rows tb/16 + 8i of the tile for
      // every k-stage: sources and swizzled destinations are computed once per tile
      // (as in the pair kernel); rows past the tile's tokens are not loaded.
      const int tb = threadIdx.x - 6 * 32;
      constexpr int NI = NT / 8;
      const int r0 = tb >> 4, ch = tb & 15;
      const uint32_t dst0 = (uint32_t)((ch >> 3) * (NT * 128) + r0 * 128 + (((ch & 7) ^ r0) << 4));
      // (no L2::cache_hint on these cp.async: measured neutral, and ptxas 12.9 emitted an
      // illegal LDGSTS descriptor operand for it in this kernel)
      uint32_t it = 0;
      TileInfo ti;
      for (int tile = tile0; decode_tile(a, NT, tile, ti); tile += tstep) {
        const uint16_t* src[NI];
        uint32_t valid = 0;
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int t = r0 + 8 * i;
          const int rid = t < ti.n_local ? a.sel_in[ti.row0 + ti.t0 + t] : -1;
          src[i] = (rid >= 0 ? x_row(a, rid) : a.x) + ch * 8;
          valid |= (rid >= 0 ? 1u : 0u) << i;
        }
        for (int k = ti.k0; k < ti.k1; ++k, ++it) {
          const int st = it % S;
          unsigned long long tg0 = prof ? clk() : 0;
          mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
          if (prof) { const unsigned long long t1 = clk(); pc[10] += t1 - tg0; tg0 = t1; }
          const int64_t kcol0 = (int64_t)k * 128;
          const uint32_t bs = smem_u32(bsm(st)) + dst0;
          if (!(a.debug & 1)) {
#pragma unroll
            for (int i = 0; i < NI; ++i)
              if ((valid >> i) & 1u)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(bs + 1024u * i), "l"(src[i] + kcol0)
                             : "memory");
          }
          cp_async_mbar_arrive_noinc(&bfull[st]);
          if (prof) pc[11] += clk() - tg0;
        }
      }
    } else if (gather) {
      const int tb = threadIdx.x - 6 * 32;
      constexpr int CPR = 16 / REP;  // 16-byte chunks per token row per stage
      constexpr int CHUNKS = NT * CPR;
      uint32_t it = 0;
      TileInfo ti;
      for (int tile = tile0; decode_tile(a, NT, tile, ti); tile += tstep) {
        named_bar_sync(1, kGatherThreads);  // previous tile's rows no longer read
        for (int i = tb; i < NT; i += kGatherThreads)
          rows[i] = i < ti.n_local ? a.sel_in[ti.row0 + ti.t0 + i] : -1;
        named_bar_sync(1, kGatherThreads);
        for (int k = ti.k0; k < ti.k1; ++k, ++it) {
          const int st = it % S;
          unsigned long long tg0 = prof ? clk() : 0;
          mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
          if (prof) { const unsigned long long t1 = clk(); pc[10] += t1 - tg0; tg0 = t1; }
          const int64_t kcol0 = (int64_t)k * (128 / REP);
          uint8_t* bs = bsm(st);
          for (int idx = tb; idx < ((a.debug & 1) ? 0 : CHUNKS); idx += kGatherThreads) {
            const int row = idx / CPR, ch = idx % CPR;
            const int atom = ch >> 3, c8 = ch & 7;
            const int rid = rows[row];
            const uint16_t* src = rid >= 0 ? x_row(a, rid) + kcol0 + ch * 8 : a.x;
            uint8_t* dst = bs + atom * (NT * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((c8 ^ (row & 7)) << 4);
            cp_async16(dst, src, rid >= 0 ? 16u : 0u);
          }
          // the barrier completes when every gather thread's copies have landed;
          // the thread moves on to the next stage immediately
          cp_async_mbar_arrive_noinc(&bfull[st]);
          if (prof) pc[11] += clk() - tg0;
        }
      }
    }
  } else {
    // ============ epilogue (warps 0-3): TMEM -> fused epilogue -> re-zero ============
    if (a.pdl) griddep_wait();  // outputs (zeroed by the previous kernel) are written below
    if (a.zero_ptr != nullptr) zero_slice(a, (int64_t)blockIdx.x * 128 + threadIdx.x, (int64_t)gridDim.x * 128);
    const int q = warp;  // TMEM lane quarter
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int nf = a.n_fmt;
    auto zero_acc = [&](int b) {
      for (int c = 0; c < C::kAccCols; c += 16) tmem_st16_zero(tmem + lane_base + b * C::kAccCols + c);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    };
    for (int b = 0; b < AB; ++b) zero_acc(b);
    uint32_t tcount = 0;
    TileInfo ti;
    for (int tile = tile0; decode_tile(a, NT, tile, ti); tile += tstep, ++tcount) {
      const int cr = ti.m_tile * kTileM + 32 * q + lane;  // compressed row of this lane
      const bool valid = cr < a.R;
      const int grp = cr / nf;
      unsigned long long t0 = prof ? clk() : 0;
      const int ab = tcount % AB;
      mbar_wait(&acc_full[ab], (tcount / AB) & 1);
      if (prof) { const unsigned long long t1 = clk(); pc[3] += t1 - t0; t0 = t1; }
      tc_fence_after();
      if constexpr (XP != 0) {
        // lane l of warp q in half h = expanded row pos = 128 h + 32 q + l of the m-tile
        for (int h = 0; h < 2; ++h) {
          const uint32_t tcol = tmem + lane_base + ab * C::kAccCols + h * NT;
          if (a.epi == kEpiSiluMulIlv) {
            // lanes 0-15 gate / 16-31 up of the same 16 outputs (xp_pos)
            const int cg = ti.m_tile * 128 + 64 * h + 16 * q + (lane & 15);
            for (int c0 = 0; c0 < ti.n_local; c0 += 16) {
              float v[16];
              tmem_ld16(tcol + c0, v);
              tmem_ld_wait();
              ilv_chunk_ms1(v, cg < a.m_out && !(a.debug & 8), min(16, ti.n_local - c0),
                            static_cast<uint16_t*>(a.out), a.ldo, ti.row0 + ti.t0 + c0, cg, lane);
            }
            continue;
          }
          const int o = ti.m_tile * 256 + 128 * h + 32 * q + lane;  // output row of this lane
          const bool ok = o < a.m_out && !(a.debug & 8);
          for (int c0 = 0; c0 < ti.n_local; c0 += 16) {
            float v[16];
            tmem_ld16(tcol + c0, v);
            tmem_ld_wait();
            const int jmax = min(16, ti.n_local - c0);
            if (a.epi == kEpiScatter) {
              const int rl = ti.row0 + ti.t0 + c0 + (lane & 15);
              float* my_row = (lane & 15) < jmax ? out_row(a, a.sel_out ? a.sel_out[rl] : rl) : nullptr;
              const float my_s = (lane & 15) < jmax ? (a.scale ? a.scale[rl] : 1.f) : 0.f;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                float* orow = reinterpret_cast<float*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j));
                const float sj = __shfl_sync(0xffffffffu, my_s, j);
                if (ok && j < jmax) atomicAdd(orow + o, sj * v[j]);  // 32 lanes: 128 contiguous bytes
              }
              continue;
            }
            if (!ok) continue;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j >= jmax) break;
              const int64_t r = ti.row0 + ti.t0 + c0 + j;
              if (a.out_bf16)
                static_cast<uint16_t*>(a.out)[r * a.ldo + o] = __bfloat16_as_ushort(__float2bfloat16_rn(v[j]));
              else
                static_cast<float*>(a.out)[r * a.ldo + o] = v[j];
            }
          }
        }
        tc_fence_before();
        zero_acc(ab);
        if (prof) pc[4] += clk() - t0;
        continue;
      }
      if (NW == 1 && MS == 1 && REP == 1 && a.epi == kEpiSiluMulIlv) {
        // N = M: lanes 0-15 gate / 16-31 up of the same 16 outputs (reading R20)
        const int cg = 16 * (4 * ti.m_tile + q) + (lane & 15);
        for (int c0 = 0; c0 < ti.n_local; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + lane_base + ab * C::kAccCols + c0, v);
          tmem_ld_wait();
          ilv_chunk_ms1(v, cg < a.R / 2 && !(a.debug & 8), min(16, ti.n_local - c0), static_cast<uint16_t*>(a.out),
                        a.ldo, ti.row0 + ti.t0 + c0, cg, lane);
        }
        tc_fence_before();
        zero_acc(ab);
        if (prof) pc[4] += clk() - t0;
        continue;
      }
      if (NW == 1 && MS == 2 && a.epi == kEpiSiluMulIlv) {
        // lanes 0-15 gate / 16-31 up of the same 16 output pairs (reading R20)
        const int cg = 16 * (4 * ti.m_tile + q) + (lane & 15);
        for (int c0 = 0; c0 < ti.n_local; c0 += 16) {
          float v[2][16];
          tmem_ld16(tmem + lane_base + ab * C::kAccCols + c0, v[0]);
          tmem_ld16(tmem + lane_base + ab * C::kAccCols + NT + c0, v[1 % MS]);
          tmem_ld_wait();
          ilv_chunk(v, cg < a.R / 2 && !(a.debug & 8), min(16, ti.n_local - c0), static_cast<uint16_t*>(a.out), a.ldo,
                    ti.row0 + ti.t0 + c0, cg, lane, a.rows_out);
        }
        tc_fence_before();
        zero_acc(ab);
        if (prof) pc[4] += clk() - t0;
        continue;
      }
      for (int c0 = 0; c0 < ti.n_local; c0 += 16) {
        float v[NW][MS][16];
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int p = 0; p < MS; ++p)
            tmem_ld16(tmem + lane_base + ab * C::kAccCols + (w * MS + p) * NT + c0, v[w][p]);
        tmem_ld_wait();
        if (MS > 1 && nf > 1) {  // N>1: sum the N lanes of a block (compressed rows of one group)
#pragma unroll
          for (int w = 0; w < NW; ++w)
#pragma unroll
            for (int p = 0; p < MS; ++p)
#pragma unroll
              for (int j = 0; j < 16; ++j)
                for (int off = nf >> 1; off > 0; off >>= 1) v[w][p][j] += __shfl_xor_sync(0xffffffffu, v[w][p][j], off);
        }
        const int jmax = min(16, ti.n_local - c0);
        if (a.epi == kEpiScatter) {
          // destination rows / gate weights of these 16 tokens: one load per lane,
          // broadcast by shuffle (all lanes take part, so no early exit above)
          const int rl = ti.row0 + ti.t0 + c0 + (lane & 15);
          float* my_row = (lane & 15) < jmax ? out_row(a, a.sel_out ? a.sel_out[rl] : rl) : nullptr;
          const float my_s = (lane & 15) < jmax ? (a.scale ? a.scale[rl] : 1.f) : 0.f;
          const int nv = (valid && !(a.debug & 8)) ? jmax : 0;
          if (MS == 2 && nf == 1) {  // the default (1,2,V): 16 independent predicated reductions
            scatter_chunk_v4(v[0][0], v[0][1 % MS], my_row, my_s, nv, grp, lane);
            continue;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float* o = reinterpret_cast<float*>(
                __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j));
            const float s = __shfl_sync(0xffffffffu, my_s, j);
            if (j >= nv) continue;
            if (MS == 1) {
              atomicAdd(o + cr, s * v[0][0][j]);
            } else if (MS == 2 && nf == 1) {
              red_add_v2(o + 2 * grp, s * v[0][0][j], s * v[0][1 % MS][j]);
            } else {
#pragma unroll
              for (int p = 0; p < MS; ++p)
                if ((p % nf) == (cr % nf)) atomicAdd(o + grp * MS + p, s * v[0][p][j]);
            }
          }
          continue;
        }
        if (!valid || (a.debug & 8)) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j >= jmax) break;
          const int r = ti.row0 + ti.t0 + c0 + j;  // compact row of this token
          if (NW == 2) {  // SiLU(gate) * up -> bf16
            uint16_t* o = static_cast<uint16_t*>(a.out) + (int64_t)r * a.ldo;
            if (MS == 2 && nf == 1) {
              float act[2];
#pragma unroll
              for (int p = 0; p < 2; ++p) act[p] = silu_mul(v[0][p % MS][j], v[NW - 1][p % MS][j]);
              const __nv_bfloat162 h = __floats2bfloat162_rn(act[0], act[1]);
              *reinterpret_cast<__nv_bfloat162*>(o + 2 * grp) = h;
            } else {
#pragma unroll
              for (int p = 0; p < MS; ++p) {
                if (MS > 1 && nf > 1 && (p % nf) != (cr % nf)) continue;
                const float act = silu_mul(v[0][p][j], v[NW - 1][p][j]);
                o[MS == 1 ? cr : grp * MS + p] = __bfloat16_as_ushort(__float2bfloat16_rn(act));
              }
            }
          } else if (a.out_bf16) {
            uint16_t* o = static_cast<uint16_t*>(a.out) + (int64_t)r * a.ldo;
#pragma unroll
            for (int p = 0; p < MS; ++p) {
              if (MS > 1 && nf > 1 && (p % nf) != (cr % nf)) continue;
              o[MS == 1 ? cr : grp * MS + p] = __bfloat16_as_ushort(__float2bfloat16_rn(v[0][p][j]));
            }
          } else {
            float* o = static_cast<float*>(a.out) + (int64_t)r * a.ldo;
            if (MS == 2 && nf == 1) {
              *reinterpret_cast<float2*>(o + 2 * grp) = make_float2(v[0][0][j], v[0][1 % MS][j]);
            } else {
#pragma unroll
              for (int p = 0; p < MS; ++p) {
                if (MS > 1 && nf > 1 && (p % nf) != (cr % nf)) continue;
                o[MS == 1 ? cr : grp * MS + p] = v[0][p][j];
              }
            }
          }
        }
      }
      tc_fence_before();
      zero_acc(ab);  // hand this accumulator set back
      if (prof) pc[4] += clk() - t0;
    }
  }
  tc_fence_before();
  if (prof) {
    unsigned long long* o = a.prof + ((size_t)(a.epi == kEpiScatter) * 148 + blockIdx.x) * 16;
    if (warp == 5 && lane == 0) { atomicAdd(o + 0, pc[0]); atomicAdd(o + 1, pc[1]); atomicAdd(o + 2, pc[2]); atomicAdd(o + 7, pc[7]); }
    if (warp == 6 && lane == 0) { atomicAdd(o + 10, pc[10]); atomicAdd(o + 11, pc[11]); }
    if (warp == 0 && lane == 0) { atomicAdd(o + 3, pc[3]); atomicAdd(o + 4, pc[4]); }
    if (warp == 4 && lane == 0) { atomicAdd(o + 5, pc[5]); }
    if (XP && warp == 11 && lane == 0) {
      atomicAdd(o + 6, pc[6]); atomicAdd(o + 8, pc[8]); atomicAdd(o + 9, pc[9]); atomicAdd(o + 12, pc[11]);
    }
  }
  __syncthreads();
  tc_fence_after();
  if (warp == 5) tmem_dealloc(tmem, C::kTmemCols);
}

// ------------------------------------------------------------------ host side

template <int NT, int NW, int MS, int REP, int XP = 0>
smy_status launch_t(const SsmmArgs& a, cudaStream_t s) {
  using C = Cfg<NT, NW, MS, REP, XP>;
  constexpr int kThreadsL = threads_of(XP);
  static bool configured = false;
  static int num_sms = 0;
  auto kern = ssmm_kernel<NT, NW, MS, REP, XP>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return cuda_status(e);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    configured = true;
  }
  if (a.max_tiles <= 0) return SMY_OK;
  SsmmArgs b = a;
  b.streamk = a.epi == kEpiScatter && a.k_splits <= 1 && !(a.debug & 512);
  const int grid = (b.streamk || a.max_tiles >= num_sms) ? num_sms : a.max_tiles;
  b.workers = grid;
  // m-tile fastest (concurrent tiles share the token tile in L2) for the scatter (down)
  // launches, and for SEL-gather launches whose token pool does not fit in L2 (their
  // n-fastest order would re-stream the gathered rows from HBM for every m-tile)
  b.m_fastest = (a.epi == kEpiScatter || (a.sel_in != nullptr && (int64_t)a.x_rows * a.ldx * 2 > kGatherL2Bytes)) &&
                !(a.debug & 2048);
  if (b.pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreadsL);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, b);
    count_launch();
    return cuda_status(e);
  }
  kern<<<grid, kThreadsL, C::kSmemBytes, s>>>(b);
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
