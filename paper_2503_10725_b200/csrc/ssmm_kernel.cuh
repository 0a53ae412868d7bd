#pragma once
// Samoyeds dual-side sparse SSMM for sm_100a (B200).
//
// C[t, o] = sum_k W[o, k] * x[sel[t], k]     (Alg. 1)
//
// B200 design:
//  * one CTA = one tile of 128 compressed weight rows (TMEM lanes) x NT
//    selected tokens, for one expert (grouped launches decode the expert from
//    a device-side tile prefix -- no host sync on routing counts);
//  * warp 0 streams the pre-packed weight image (A smem image | E metadata
//    TMEM image | index bit-planes) with one cp.async.bulk per stage/weight;
//  * warps 2-7 gather the routed token rows x[sel[t]] straight from the
//    token-major activations into a 128B-swizzled K-major tile with cp.async
//    (the paper's SEL gather; no permuted copy of x is ever made);
//  * warp 1 (one lane) copies E smem->TMEM (tcgen05.cp) and issues
//    tcgen05.mma.sp (bf16, K=32 = one V=32 sub-row window per MMA);
//  * the data-stationary remap of §4.3 ("the output of the SpTC
//    must be remapped to different rows ... according to the indices") is done
//    by the tensor core itself: one TMEM accumulator per in-block sub-row slot
//    p < M, and every MMA carries a 128-bit disable_output_lane mask built from
//    the index bit-planes so lane r only accumulates into slot idx[r][j];
//  * warps 4-7 zero the accumulators, then run the fused epilogue
//    (compact store / SiLU*up -> bf16 / routing-weight scale + scatter-add,
//    P:337) straight from TMEM (tcgen05.ld).
#include <cuda_bf16.h>

#include <cstdio>

#include "internal.h"
#include "ptx.cuh"

namespace smy {

template <int NT, int NW, int MS, int REP>
struct Cfg {
  static constexpr int kWStride = 19456;                  // A|E|planes, 1024-aligned stride
  static constexpr int kBBytes = NT * 128 * (2 / REP);     // token tile per stage
  static constexpr int kStageBytes = NW * kWStride + kBBytes;
  static constexpr int kAccCols = NW * MS * NT;
  static constexpr int kECol = (kAccCols + 3) / 4 * 4;
  static constexpr int kColsNeeded = kECol + 4 * NW;
  static constexpr int kTmemCols = kColsNeeded <= 32    ? 32
                                   : kColsNeeded <= 64  ? 64
                                   : kColsNeeded <= 128 ? 128
                                   : kColsNeeded <= 256 ? 256
                                                        : 512;
  static constexpr int kAux = 2048;                        // barriers + row ids
  static constexpr int kSmemCap = 232448 - 1024 - kAux;
  static constexpr int kStagesRaw = kSmemCap / kStageBytes;
  static constexpr int kStages = kStagesRaw > 6 ? 6 : kStagesRaw;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + kAux;
  static constexpr int kPlanes = MS == 1 ? 0 : MS == 2 ? 1 : MS == 4 ? 2 : MS == 8 ? 3 : 4;
  static constexpr int kLag = kStages >= 3 ? 2 : 1;
  static_assert(kColsNeeded <= 512, "TMEM budget");
  static_assert(kStages >= 2, "smem budget");
  static_assert(NT % 16 == 0 && NT >= 16 && NT <= 256, "UMMA N");
};

constexpr int kThreads = 256;
constexpr int kLoaderThreads = 192;  // warps 2..7

template <int NT, int NW, int MS, int REP>
__global__ void __launch_bounds__(kThreads, 1) ssmm_kernel(const __grid_constant__ SsmmArgs a) {
  using C = Cfg<NT, NW, MS, REP>;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aux = smem + S * C::kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(aux);
  uint64_t* empty = full + S;
  uint64_t* acc_full = empty + S;
  uint64_t* tmem_ready = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_ready + 1);
  int32_t* rows = reinterpret_cast<int32_t*>(aux + 1024);

  // ---- tile -> (group, m_tile, n_tile)
  int g = 0, local = blockIdx.x;
  if (a.tile_prefix != nullptr) {
    if (local >= a.tile_prefix[a.num_groups]) return;
    int lo = 0, hi = a.num_groups - 1;
    while (lo < hi) {  // last g with prefix[g] <= local
      int mid = (lo + hi + 1) >> 1;
      if (a.tile_prefix[mid] <= local) lo = mid; else hi = mid - 1;
    }
    g = lo;
    local -= a.tile_prefix[g];
  }
  const int m_tile = local % a.m_tiles;
  const int n_tile = local / a.m_tiles;
  const int row0 = a.offsets ? a.offsets[g] : 0;
  const int n_g = a.offsets ? a.offsets[g + 1] - row0 : a.n_sel;
  const int t0 = n_tile * NT;
  const int n_local = min(NT, n_g - t0);
  if (n_local <= 0) return;

  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1 + kLoaderThreads / 32);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(tmem_ready, 4);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::kTmemCols);
  for (int i = threadIdx.x; i < NT; i += kThreads)
    rows[i] = (i < n_local) ? (a.sel_in ? a.sel_in[row0 + t0 + i] : row0 + t0 + i) : -1;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto wsm = [&](int st, int w) { return smem + st * C::kStageBytes + w * C::kWStride; };
  auto bsm = [&](int st) { return smem + st * C::kStageBytes + NW * C::kWStride; };
  const int ks = a.k_stages;

  if (warp == 0) {
    // ======================= weight-image producer =======================
    if (lane == 0) {
      const uint32_t bytes = kABytes + kEBytes + 64 * C::kPlanes;
      const uint64_t pol = policy_evict_last();
      const uint8_t* src0 = a.img0[g] + (size_t)m_tile * ks * a.block;
      const uint8_t* src1 = NW == 2 ? a.img1[g] + (size_t)m_tile * ks * a.block : nullptr;
      for (int it = 0; it < ks; ++it) {
        const int st = it % S;
        mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
        mbar_arrive_expect_tx(&full[st], NW * bytes);
        bulk_g2s(wsm(st, 0), src0 + (size_t)it * a.block, bytes, &full[st], pol);
        if (NW == 2) bulk_g2s(wsm(st, 1), src1 + (size_t)it * a.block, bytes, &full[st], pol);
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer =============================
    if (lane == 0) {
      constexpr uint32_t idesc = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) |
                                 ((uint32_t)(128 >> 4) << 24);
      mbar_wait(tmem_ready, 0);
      tc_fence_after();
      for (int it = 0; it < ks; ++it) {
        const int st = it % S;
        mbar_wait(&full[st], (it / S) & 1);
        tc_fence_after();
#pragma unroll
        for (int w = 0; w < NW; ++w)
          tc_cp_128x128b(tmem + C::kECol + 4 * w, desc_interleave(smem_u32(wsm(st, w) + kABytes)));
#pragma unroll
        for (int kb = 0; kb < 4; ++kb) {
          const int e0 = (kb / REP) * 32;  // first B element of this K=32 window
          const uint64_t bdesc =
              desc_sw128(smem_u32(bsm(st)) + (e0 / 64) * (NT * 128) + (e0 % 64) * 2);
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const uint64_t adesc = desc_sw128(smem_u32(wsm(st, w)) + kb * 32);
            uint32_t pl[C::kPlanes > 0 ? C::kPlanes : 1][4];
#pragma unroll
            for (int b = 0; b < C::kPlanes; ++b) {
              const uint4 v = *reinterpret_cast<const uint4*>(wsm(st, w) + kABytes + kEBytes + (kb * C::kPlanes + b) * 16);
              pl[b][0] = v.x; pl[b][1] = v.y; pl[b][2] = v.z; pl[b][3] = v.w;
            }
#pragma unroll
            for (int p = 0; p < MS; ++p) {
              uint32_t mask[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                uint32_t en = 0xffffffffu;
#pragma unroll
                for (int b = 0; b < C::kPlanes; ++b) en &= ((p >> b) & 1) ? pl[b][q] : ~pl[b][q];
                mask[q] = MS == 1 ? 0u : ~en;
              }
              // metadata column of this K=32 window: even part in the address, the
              // odd bit in idesc.sparse_id2 (bits [0,2))
              tc_mma_sp(tmem + (w * MS + p) * NT, adesc, bdesc, idesc | (uint32_t)(kb & 1), 1u, mask,
                        tmem + C::kECol + 4 * w + (kb & 2));
            }
          }
        }
        tc_commit(&empty[st]);
      }
      tc_commit(acc_full);
    }
  } else {
    // ============== token gather (warps 2-7) + epilogue (warps 4-7) ==============
    const int tb = threadIdx.x - 64;
    if (warp >= 4) {
      const uint32_t lane_base = (uint32_t)(32 * (warp - 4)) << 16;
      for (int c = 0; c < C::kAccCols; c += 16) tmem_st16_zero(tmem + lane_base + c);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tmem_ready);
    }
    constexpr int CPR = 16 / REP;  // 16-byte chunks per token row per stage
    constexpr int CHUNKS = NT * CPR;
    constexpr int LAG = C::kLag;
    for (int it = 0; it < ks; ++it) {
      const int st = it % S;
      mbar_wait(&empty[st], ((it / S) & 1) ^ 1);
      const int64_t kcol0 = (int64_t)it * (128 / REP);
      uint8_t* bs = bsm(st);
      for (int idx = tb; idx < CHUNKS; idx += kLoaderThreads) {
        const int row = idx / CPR, ch = idx % CPR;
        const int atom = ch >> 3, c8 = ch & 7;
        const int rid = rows[row];
        const uint16_t* src = rid >= 0 ? a.x + (int64_t)rid * a.ldx + kcol0 + ch * 8 : a.x;
        uint8_t* dst = bs + atom * (NT * 128) + (row >> 3) * 1024 + (row & 7) * 128 + ((c8 ^ (row & 7)) << 4);
        cp_async16(dst, src, rid >= 0 ? 16u : 0u);
      }
      cp_async_commit();
      if (it >= LAG) {
        cp_async_wait<LAG>();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[(it - LAG) % S]);
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0)
      for (int it = ks - LAG < 0 ? 0 : ks - LAG; it < ks; ++it) mbar_arrive(&full[it % S]);

    if (warp >= 4) {
      // =============================== epilogue ===============================
      const int q = warp - 4;
      const uint32_t lane_base = (uint32_t)(32 * q) << 16;
      const int cr = m_tile * kTileM + 32 * q + lane;  // compressed row of this lane
      const bool valid = cr < a.R;
      const int nf = a.n_fmt;
      mbar_wait(acc_full, 0);
      tc_fence_after();
      for (int c0 = 0; c0 < n_local; c0 += 16) {
        float v[NW][MS][16];
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int p = 0; p < MS; ++p) tmem_ld16(tmem + lane_base + (w * MS + p) * NT + c0, v[w][p]);
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
        if (!valid) continue;
        const int grp = cr / nf;
        const int jmax = min(16, n_local - c0);
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j >= jmax) break;
          const int r = row0 + t0 + c0 + j;  // compact row of this token
          if (a.epi == kEpiScatter) {
            const int dst = a.sel_out ? a.sel_out[r] : r;
            const float s = a.scale ? a.scale[r] : 1.f;
            float* o = static_cast<float*>(a.out) + (int64_t)dst * a.ldo;
            if (MS == 1) {
              atomicAdd(o + cr, s * v[0][0][j]);
            } else if (MS == 2 && nf == 1) {
              red_add_v2(o + 2 * grp, s * v[0][0][j], s * v[0][1 % MS][j]);
            } else {
#pragma unroll
              for (int p = 0; p < MS; ++p)
                if ((p % nf) == (cr % nf)) atomicAdd(o + grp * MS + p, s * v[0][p][j]);
            }
          } else if (NW == 2) {  // SiLU(gate) * up -> bf16
            uint16_t* o = static_cast<uint16_t*>(a.out) + (int64_t)r * a.ldo;
#pragma unroll
            for (int p = 0; p < MS; ++p) {
              if (MS > 1 && nf > 1 && (p % nf) != (cr % nf)) continue;
              const float gv = v[0][p][j], uv = v[NW - 1][p][j];
              const float act = gv / (1.f + expf(-gv)) * uv;
              const int orow = MS == 1 ? cr : grp * MS + p;
              o[orow] = __bfloat16_as_ushort(__float2bfloat16_rn(act));
            }
          } else if (a.out_bf16) {
            uint16_t* o = static_cast<uint16_t*>(a.out) + (int64_t)r * a.ldo;
#pragma unroll
            for (int p = 0; p < MS; ++p) {
              if (MS > 1 && nf > 1 && (p % nf) != (cr % nf)) continue;
              const int orow = MS == 1 ? cr : grp * MS + p;
              o[orow] = __bfloat16_as_ushort(__float2bfloat16_rn(v[0][p][j]));
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
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc(tmem, C::kTmemCols);
}

// ------------------------------------------------------------------ host side

template <int NT, int NW, int MS, int REP>
smy_status launch_t(const SsmmArgs& a, cudaStream_t s) {
  using C = Cfg<NT, NW, MS, REP>;
  static bool configured = false;
  auto kern = ssmm_kernel<NT, NW, MS, REP>;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return cuda_status(e);
    configured = true;
  }
  if (a.max_tiles <= 0) return SMY_OK;
  kern<<<a.max_tiles, kThreads, C::kSmemBytes, s>>>(a);
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
