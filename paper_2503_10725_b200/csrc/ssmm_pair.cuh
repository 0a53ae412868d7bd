#pragma once
// SSMM on CTA pairs (tcgen05 cta_group::2) -- the prefill path.
//
// Same computation and epilogues as ssmm_kernel.cuh, restructured around the
// measured B200 limits (probes/mma_bench.cu, probes/gather_bench.cu, DESIGN.md
// §7.1): a sparse M=128 MMA streams its A (4 KB) and B (64 B per token) from
// shared memory at 128 B/clk, and the SEL gather is re-done for every weight
// tile.  A CTA pair (one cluster of 2 on a TPC) issues M=256 MMAs: each CTA
// holds its own 128 compressed rows of A and HALF of the token tile, each half
// of B is read once for both SMs, and each CTA gathers only half the tokens.
//
// Roles per CTA (480 threads): warps 0-3 + 10-13 epilogue, 4 producer (TMA
// loads of the weight image and the contiguous B half), 5 + 14 MMA issuers
// (leader CTA) or gather relay (warp 5 of the peer), 6-9 SEL gather
// (cp.async).  Both CTAs' TMA loads use .cta_group::2 and complete on the
// LEADER's `full` barrier, so the peer's weights / contiguous B need no relay;
// only the peer's cp.async gather is forwarded (peer-local `full` -> one remote
// arrive).  The leader's MMA commits multicast to both CTAs' `empty` /
// `acc_full`; both epilogues arrive on the leader's `acc_empty`.
#include "ssmm_kernel.cuh"

#ifndef SMY_PAIR_MIN_WSLOTS
#define SMY_PAIR_MIN_WSLOTS 3  // weight slots kept beside the token ring of a SPLIT launch
#endif
#ifndef SMY_PW_ACC
#define SMY_PW_ACC 0  // per-weight accumulator hand-off of the m-tile-paired gate/up (measured slower)
#endif
#ifndef SMY_GATHER_SPIN
#define SMY_GATHER_SPIN 0
#endif
#ifndef SMY_PAIR_W_EVICT_FIRST
#define SMY_PAIR_W_EVICT_FIRST 0
#endif
#ifndef SMY_RELAY_TRYWAIT
#define SMY_RELAY_TRYWAIT 0
#endif
#ifndef SMY_GATHER_EVICT_LAST
#define SMY_GATHER_EVICT_LAST 0
#endif
#ifndef SMY_TOKEN_ACQ_CTA
#define SMY_TOKEN_ACQ_CTA 0
#endif
#ifndef SMY_CLUSTER_ACQ_ALL
#define SMY_CLUSTER_ACQ_ALL 0
#endif

namespace smy {

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar), done = 0;
  do {
#ifdef SMY_SPIN_CLUSTER_WAIT
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
#endif
  } while (!done);
}
// CTA-scope acquire (no L1 invalidation): waits whose consumers are tcgen05 /
// TMA / cp.async operations ordered by the tcgen05 fences, not generic loads of
// the peer CTA's writes (the pattern CUTLASS's 2-SM pipelines use)
__device__ __forceinline__ void mbar_wait_cta(uint64_t* bar, uint32_t parity) {
  if (SMY_CLUSTER_ACQ_ALL) {
    mbar_wait_acq_cluster(bar, parity);
    return;
  }
  uint32_t addr = smem_u32(bar), done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
// non-suspending poll: the stage relay forwards completions with minimum latency
__device__ __forceinline__ void mbar_spin(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar), done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_cp2_elect(uint32_t taddr, uint64_t sdesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.cp.cta_group::2.128x128b [%0], %1;\n\t}" ::"r"(taddr),
      "l"(sdesc)
      : "memory");
}
__device__ __forceinline__ void tc_mma_sp2_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 const uint32_t (&m)[8], uint32_t e_tmem) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.mma.sp.cta_group::2.kind::f16 [%0], %1, %2, [%12], %3, {%4, %5, %6, %7, %8, %9, %10, %11}, 1;\n\t}" ::"r"(
          d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "r"(m[4]), "r"(m[5]), "r"(m[6]),
      "r"(m[7]), "r"(e_tmem)
      : "memory");
}
// D = 0 over this pair's 256 lanes x N columns: a dense MMA of an all-zero A and B
// (both descriptors alias one zeroed 128-B core matrix, LBO = SBO = 0) with
// enable_input_d = 0 -- clears the accumulator the lane-masked MMAs then add into
__device__ __forceinline__ void tc_mma2_zero_elect(uint32_t d_tmem, uint64_t zdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %1, %2, 0;\n\t}" ::"r"(d_tmem),
      "l"(zdesc), "r"(idesc)
      : "memory");
}
// arrive on the same-offset mbarrier in every CTA of `cta_mask` once all prior
// tcgen05 ops of this thread complete
__device__ __forceinline__ void tc_commit2_mc_elect(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\t"
      "@p tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}

// TMA 2D tile load into this CTA's shared memory whose complete_tx lands on
// the pair leader's mbarrier (`bar` is a shared::cluster address)
__device__ __forceinline__ void tma2d_pair(void* dst, const CUtensorMap* map, int c0, int c1, uint32_t bar,
                                           uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}

constexpr int kPairEpiWarps = 8;                    // warps 0-3 and 10-13

// tokens held by each CTA of a pair for a tile of n tokens: MMA N = 2 * half must
// be a multiple of 16, so a half is a whole number of 8-row swizzle atoms
__device__ __forceinline__ int pair_half(int n) { return ((n + 15) >> 4) << 3; }
constexpr int kPairThreads = 32 * (11 + kPairEpiWarps - 4);  // + producer, 2 MMA issuers, 4 gather
// SEL-gather launches (SPLIT) add 4 gather warps (15-18): the cp.async gather is what
// binds the gate/up ring (probes/gather2_bench.cu: 28 KB stages with 19.5 KB of
// weights beside them, 1344 clk per stage with 4 warps, 1185 with 8)
#ifndef SMY_PAIR_GATHER_WARPS
#define SMY_PAIR_GATHER_WARPS 8
#endif
// (w gather warps cover 2w token rows per pass: 8 warps for halves of a multiple of
// 16 rows, 7 for multiples of 14 -- the NT = 112 m-tile-paired gate/up)
constexpr int pair_gather_warps(int split, int nt) {
  return !split ? 4 : (nt / 2) % (2 * SMY_PAIR_GATHER_WARPS) == 0 ? SMY_PAIR_GATHER_WARPS
                    : (SMY_PAIR_GATHER_WARPS >= 7 && (nt / 2) % 14 == 0) ? 7 : 4;
}
// lock-step (SPLIT = 0) kernels carry 4 more warps (15-18): a fourth epilogue warp per
// TMEM lane quadrant when the token rows are contiguous (the down), idle otherwise
#ifndef SMY_PAIR_EPI4
#define SMY_PAIR_EPI4 1
#endif
constexpr int pair_threads(int split, int nt) {
  return kPairThreads + 32 * (pair_gather_warps(split, nt) - 4) + (!split && SMY_PAIR_EPI4 ? 128 : 0);
}
constexpr int pair_gather_threads(int split, int nt) { return 32 * pair_gather_warps(split, nt); }

// MS = accumulator slots per weight: 2 for (1,2,V) (the lane-masked remap), 1 for
// N == M (plain 2:4, no remap -- the weight-only-sparse baseline formats)
// SPLIT: separate weight / token rings (own barriers, deeper token ring) -- the SEL
// gather launches (gate/up), whose token-row loads show the longest latency; the
// contiguous-row launches (down) keep both in one lock-step ring
template <int NT, int NW, int MS_ = 2, int SPLIT = 0>
struct PairCfg {
  static constexpr int MS = MS_;
  static constexpr int kHalf = NT / 2;                      // tokens per CTA
  static constexpr int kWStride = 19456;                    // A|E|planes (kWRows rows of 128 B)
  static constexpr int kWRows = (kABytes + kEBytes + 64 + 127) / 128;  // TMA box rows of one weight tile
  static constexpr int kBBytes = kHalf * 256;               // 2 K-atoms x kHalf rows x 128 B
  static constexpr int kPeerPl = MS == 2 ? 128 : 0;         // the peer m-tile's index planes (leader)
  static constexpr int kWStage = (NW * kWStride + kPeerPl + 1023) / 1024 * 1024;  // weight slot (+ peer planes)
  static constexpr int kBStage = (kBBytes + 1023) / 1024 * 1024;                  // token-row slot
  static constexpr int kAccCols = NW * MS * NT;
  // two accumulator sets when they fit (NT <= 112 at NW = 1): the epilogue drains
  // tile i while the MMAs of tile i+1 run -- for short-K launches whose epilogue is
  // as long as their main loop
  static constexpr int kAccBufs = 2 * kAccCols + 16 <= 512 ? 2 : 1;
  static constexpr int kECol = (kAccBufs * kAccCols + 3) / 4 * 4;
  static constexpr int kColsNeeded = kECol + 16;            // E: 2 buffers x 2 issuer warps x 4 cols
  static constexpr int kTmemCols = kColsNeeded <= 128 ? 128 : kColsNeeded <= 256 ? 256 : 512;
  static constexpr int kAux = 2048;
  static constexpr int kSmemCap = 232448 - 1024 - kAux;
  static constexpr int kStagesRaw = kSmemCap / (kWStage + kBStage);
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;          // lock-step ring depth
  // split rings: 5 token slots (measured: their depth matters more than the weights'),
  // the rest of shared memory to weight slots
  static constexpr int kBFit = (kSmemCap - SMY_PAIR_MIN_WSLOTS * kWStage) / kBStage;
  static constexpr int kBStages = SPLIT ? (SMY_TOKEN_SLOTS < kBFit ? SMY_TOKEN_SLOTS : kBFit) : kStages;
  static constexpr int kWStagesRaw = SPLIT ? (kSmemCap - kBStages * kBStage) / kWStage : kStages;
  static constexpr int kWStages = kWStagesRaw > 8 ? 8 : kWStagesRaw;
  static constexpr int kSmemBytes = kWStages * kWStage + kBStages * kBStage + 1024 + kAux;
  static_assert(kColsNeeded <= 512, "TMEM budget");
  static_assert(kBStages >= 2 && kWStages >= 2, "smem budget");
  static_assert(NT % 16 == 0 && (NT / 2) % 8 == 0 && NT >= 32 && NT <= 256, "UMMA N (cta_group::2) / 8-row halves");
};

template <int NT, int NW, int MS, int SPLIT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair_threads(SPLIT, NT), 1)
    ssmm_pair_kernel(const __grid_constant__ SsmmArgs a) {
  using C = PairCfg<NT, NW, MS, SPLIT>;
  constexpr int SW = C::kWStages, SB = C::kBStages;
  if (threadIdx.x == 0) griddep_launch_dependents();  // see ssmm_kernel
  constexpr int kIssuers = (NW == 2 || MS == 2) ? 2 : 1;  // MMA-issuing warps
  constexpr int H = C::kHalf;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* aux = smem + SW * C::kWStage + SB * C::kBStage;
  // lock-step: wfull / wempty serve both rings; split: bfull / bempty for the tokens
  uint64_t* wfull = reinterpret_cast<uint64_t*>(aux);  // [SW]
  uint64_t* wempty = wfull + 8;                        // [SW]
  uint64_t* bfull = SPLIT ? wempty + 8 : wfull;        // [SB]
  uint64_t* bempty = SPLIT ? wempty + 16 : wempty;     // [SB]
  constexpr int AB = C::kAccBufs;
  // per-weight accumulator hand-off (m-tile-paired ILV gate/up, one accumulator set):
  // acc_full[w] / acc_empty[w] per weight, so issuer w starts its next tile as soon as
  // both epilogues have drained weight w -- the weight-0 MMAs of tile i+1 overlap the
  // weight-1 half of tile i's epilogue
  const bool PW = SMY_PW_ACC && NW == 2 && MS == 2 && AB == 1 && a.mtp_half && a.epi == kEpiSiluMulIlv;
  uint64_t* acc_full = wempty + 24;    // [AB]
  uint64_t* acc_empty = acc_full + 2;  // [AB]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t cta = cluster_rank();
  const bool leader = cta == 0;
  const bool gather = a.sel_in != nullptr;
  // launches with contiguous token rows leave the gather warps 6-9 idle: they join the
  // epilogue as a third warp per TMEM lane quadrant (the scatter-add epilogue of short-K
  // down launches is what the MMA waits for; SMY_DEBUG & 134217728 turns it off)
  const bool epi3 = !gather && !(a.debug & 134217728);
  const bool epi4 = epi3 && !SPLIT && SMY_PAIR_EPI4;  // + warps 15-18
  const int NHW = epi4 ? 4 : epi3 ? 3 : 2;  // epilogue warps per lane quadrant
  const int warp = warp_id(), lane = lane_id();
  uint8_t* zbuf = aux + 1024;  // 1 KB of zeros: the operand of the accumulator-clearing MMA
  // SMY_DEBUG & 128: clock at which the leader's gather thread 0 issued each token slot
  volatile unsigned long long* ts_issue = reinterpret_cast<volatile unsigned long long*>(aux + 512);
  // TMEM allocation first, ordered before every other shared-memory write of the
  // prologue (compute-sanitizer racecheck flagged the allocator's slot write
  // against the prologue's stores when they were unordered)
  if (warp_id() == 5) tmem_alloc2(tmem_slot, C::kTmemCols);
  __syncthreads();
  if (threadIdx.x < 256) {
    reinterpret_cast<uint32_t*>(zbuf)[threadIdx.x] = 0u;
    fence_proxy_async_smem();
  }
  if (threadIdx.x < 8) ts_issue[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    if constexpr (SPLIT) {
      for (int s = 0; s < SW; ++s) {
        mbar_init(&wfull[s], 1);          // the leader's expect_tx (both CTAs' weight bytes + planes)
        mbar_init(&wempty[s], kIssuers);  // every issuer warp's commit
      }
      for (int s = 0; s < SB; ++s) {
        // gather: own gather threads (+ the peer's relay on the leader); contiguous
        // rows: the leader's expect_tx (both CTAs' TMA bytes)
        mbar_init(&bfull[s], gather ? pair_gather_threads(SPLIT, NT) + (leader ? 1 : 0) : 1);
        mbar_init(&bempty[s], kIssuers);
      }
    } else {
      for (int s = 0; s < SW; ++s) {
        // leader: its producer's expect_tx (all TMA bytes of both CTAs) + its gather
        // threads + the peer's gather relay; peer: its gather threads (relayed)
        mbar_init(&wfull[s], leader ? 1 + (gather ? kGatherThreads + 1 : 0) : (gather ? kGatherThreads : 1));
        mbar_init(&wempty[s], kIssuers);  // every issuer warp's commit
      }
    }
    for (int b = 0; b < (PW ? 2 : AB); ++b) {
      mbar_init(&acc_full[b], PW ? 1 : kIssuers);  // every issuer warp's commit (PW: its weight's)
      mbar_init(&acc_empty[b], 2 * 4 * NHW);  // every epilogue warp of both CTAs
    }
    fence_mbar_init();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrive
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto wsm = [&](int st, int w) { return smem + st * C::kWStage + w * C::kWStride; };
  auto psm = [&](int st) { return smem + st * C::kWStage + NW * C::kWStride; };
  auto bsm = [&](int st) { return smem + SW * C::kWStage + st * C::kBStage; };
  const int ks = a.k_stages;
  const int pair0 = blockIdx.x >> 1, pstep = gridDim.x >> 1;
  const uint32_t wfull_lead = mapa_shared(smem_u32(wfull), 0);  // the leader's barriers, cluster window
  const uint32_t bfull_lead = mapa_shared(smem_u32(bfull), 0);

  const bool prof = a.prof != nullptr;
  unsigned long long pc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  auto gtime = []() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  const unsigned long long g_start = prof ? gtime() : 0;
  auto clk = []() { unsigned long long c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; };
  if (warp == 4) {
    // ========= producer: own weight tiles + contiguous B half (TMA, completing on
    // the leader's full) + (leader) the peer m-tile's index planes =========
    if (lane == 0) {
      const uint32_t wbytes = (a.debug & 2) ? 0u : (uint32_t)C::kWRows * 128;
      const uint32_t w_pair_bytes = 2 * NW * wbytes + (MS == 2 ? NW * 64u : 0u);
      const uint32_t b_pair_bytes = gather ? 0u : 2 * (uint32_t)C::kBBytes;
      // prefill: the pairs on the same m-tile read its weights at about the same
      // time; evict_normal measured better than evict_first (fewer re-reads)
      const uint64_t pol_w = (a.weights_stream || SMY_PAIR_W_EVICT_FIRST) ? policy_evict_first() : policy_evict_normal();
      const uint64_t pol_x = policy_evict_last();
      const int brows = a.block >> 7;
      uint32_t it = 0;
      TileInfo ti;
      // programmatic dependent launch (SsmmArgs::pdl): the lock-step ring's first SW
      // stages get their weights at once, their token halves after griddepcontrol.wait
      const bool defer = a.pdl && !gather && !SPLIT;
      if (a.pdl && !gather && SPLIT) griddep_wait();
      int npend = 0, pend_k[SW], pend_row[SW];
      auto load_b = [&](int sb, int k, int xrow) {
#pragma unroll
        for (int atom = 0; atom < 2; ++atom)
          tma2d_pair(bsm(sb) + atom * (H * 128), &a.tmap_x, k * 128 + atom * 64, xrow, bfull_lead + sb * 8, pol_x);
      };
      auto flush = [&]() {
        griddep_wait();
        for (int i = 0; i < npend; ++i) load_b(i, pend_k[i], pend_row[i]);
        npend = -1;
      };
      for (int tile = pair0; decode_tile(a, NT, tile, ti); tile += pstep) {
        // an odd m-tile count leaves the last pair's peer without a tile: it loads the
        // last real tile again (valid memory) and its epilogue stores nothing
        const int m_own = min(2 * ti.m_tile + (int)cta, a.m_tiles - 1), m_peer = min(2 * ti.m_tile + 1, a.m_tiles - 1);
        const int hh = pair_half(ti.n_local);
        const uint8_t* src[2] = {a.img0[ti.g], NW == 2 ? a.img1[ti.g] : nullptr};
        int wrow[2];
#pragma unroll
        for (int w = 0; w < NW; ++w) wrow[w] = (int)((src[w] - a.wbase) >> 7) + m_own * ks * brows;
        const int xrow = ti.row0 + ti.t0 + (int)cta * hh;
        for (int k = ti.k0; k < ti.k1; ++k, ++it) {
          const int st = it % SW;
          if (defer && npend >= 0 && it >= (uint32_t)SW) flush();
          const unsigned long long t0 = prof ? clk() : 0;
          mbar_wait_cta(&wempty[st], ((it / SW) & 1) ^ 1);
          if (prof) pc[5] += clk() - t0;
          if (leader) mbar_arrive_expect_tx(&wfull[st], SPLIT ? w_pair_bytes : w_pair_bytes + b_pair_bytes);
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            if (!(a.debug & 2)) tma2d_pair(wsm(st, w), &a.tmap_w, 0, wrow[w] + k * brows, wfull_lead + st * 8, pol_w);
            if (MS == 2 && leader)
              bulk_g2s(psm(st) + 64 * w, src[w] + ((size_t)m_peer * ks + k) * a.block + kABytes + kEBytes, 64,
                       &wfull[st], pol_w);
          }
          if (!gather) {
            const int sb = it % SB;
            if constexpr (SPLIT) {
              mbar_wait_cta(&bempty[sb], ((it / SB) & 1) ^ 1);
              if (leader) mbar_arrive_expect_tx(&bfull[sb], b_pair_bytes);
            }
            if (defer && npend >= 0) {  // lock-step: sb == st == it for the first SW stages
              pend_k[npend] = k;
              pend_row[npend] = xrow;
              ++npend;
            } else {
              load_b(sb, k, xrow);
            }
          }
        }
      }
      if (defer && npend >= 0) flush();
    }
  } else if (warp == 5 || warp == 14) {
    if (leader && (warp == 5 || kIssuers == 2)) {
      // ==================== MMA issuers (leader CTA, warps 5 and 14) ====================
      // The per-stage issue work (plane words -> uniform lane masks, descriptors,
      // elect) costs about as much as the tensor work itself, so two warps split
      // the MMAs: NW == 2 -> warp mi issues weight mi; NW == 1 -> slot p = mi.
      // tcgen05.commit tracks the issuing thread's MMAs, so both warps commit and
      // `empty` / `acc_full` expect two arrivals per pair.  Each warp copies the
      // E image it uses into its own TMEM columns (ordered before its MMAs).
      const int mi = warp == 14 ? 1 : 0;
      const int w = NW == 2 ? mi : 0;
      constexpr int NP = NW == 2 ? MS : 1;  // slots this warp issues
      // N of a tile = 2 * its per-CTA half (runtime: ragged tiles issue narrower MMAs)
      constexpr uint32_t idesc0 = (1u << 2) | (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 4) << 24);
      constexpr uint32_t zidesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 4) << 24);  // dense
      const uint64_t zdesc = (uint64_t)((smem_u32(zbuf) & 0x3FFFF) >> 4) | ((uint64_t)1 << 46);  // no swizzle, LBO = SBO = 0
      const uint32_t smem_base = smem_u32(smem);
      const uint32_t tm = __reduce_or_sync(0xffffffffu, tmem);
      uint32_t it = 0, tcount = 0;
      TileInfo ti;
      const unsigned long long tstart = prof ? clk() : 0;
      for (int tile = pair0; decode_tile(a, NT, tile, ti); tile += pstep, ++tcount) {
        unsigned long long t0 = prof ? clk() : 0;
        const int ab = tcount % AB;
        const uint32_t tacc = tm + ab * C::kAccCols;
        mbar_wait_cta(&acc_empty[PW ? w : ab], (tcount / AB) & 1);  // both epilogues have read the accumulator
        if (prof) pc[1] += clk() - t0;
        tc_fence_after();
        const uint32_t nbits = __reduce_or_sync(0xffffffffu, ((uint32_t)(2 * pair_half(ti.n_local)) >> 3) << 17);
        const uint32_t idesc = idesc0 | nbits;
        // clear this warp's accumulator regions (the masked MMAs only add into the
        // lanes they enable); ordered before them as MMAs of the same thread
#pragma unroll
        for (int pp = 0; pp < NP; ++pp)
          tc_mma2_zero_elect(tacc + (w * MS + (NW == 2 ? pp : mi)) * NT, zdesc, zidesc | nbits);
        for (int k = ti.k0; k < ti.k1; ++k, ++it) {
          const int st = it % SW, sb = it % SB;
          t0 = prof ? clk() : 0;
          if constexpr (SPLIT) {
            // weight slots: TMA / bulk copies only (CTA-scope acquire); token slots
            // include the peer's cp.async writes, made visible by its relay's release
            mbar_wait_cta(&wfull[st], (it / SW) & 1);
            if (prof) { const unsigned long long t1 = clk(); pc[0] += t1 - t0; t0 = t1; }
#if SMY_TOKEN_ACQ_CTA
            mbar_wait_cta(&bfull[sb], (it / SB) & 1);
#else
            mbar_wait_acq_cluster(&bfull[sb], (it / SB) & 1);
#endif
            if (prof) {  // token-ring share of the operand waits; issue -> ready latency of the slot
              const unsigned long long t1 = clk(), ts = ts_issue[sb];
              pc[6] += t1 - t0;
              // (the gather's generic store of ts is not ordered by its async arrive:
              // skip the first round's unwritten slots)
              if (ts != 0 && t1 > ts && t1 - ts < (1ull << 24)) pc[8] += t1 - ts;
              t0 = clk();
            }
          } else {
            mbar_wait_acq_cluster(&wfull[st], (it / SW) & 1);  // both CTAs' stage (peer bytes + relay)
          }
          if (prof) pc[0] += clk() - t0;
          tc_fence_after();
          const uint32_t sbase = smem_base + st * C::kWStage;
          const uint32_t bbase = smem_base + SW * C::kWStage + sb * C::kBStage;
          const uint32_t ecol = C::kECol + (it & 1) * 8 + 4 * mi;
          tc_cp2_elect(tm + ecol, desc_interleave(sbase + w * C::kWStride + kABytes));
          // lane planes: words 0-3 this CTA's 128 lanes, 4-7 the peer's.  Plain LDS into
          // registers (the same value in every lane); the masks reach the MMA through
          // the elected lane's R2UR -- redux.sync per word made the issuer warp the
          // bottleneck (probes/pair_mma_bench.cu: 122 vs 113 clk per MMA)
          uint32_t pl[4][8];
#pragma unroll
          for (int kb = 0; kb < 4 && MS == 2; ++kb) {
            const uint4 v = lds_v4(sbase + w * C::kWStride + kABytes + kEBytes + kb * 16);
            const uint4 u = lds_v4(sbase + NW * C::kWStride + 64 * w + kb * 16);
            pl[kb][0] = v.x;
            pl[kb][1] = v.y;
            pl[kb][2] = v.z;
            pl[kb][3] = v.w;
            pl[kb][4] = u.x;
            pl[kb][5] = u.y;
            pl[kb][6] = u.z;
            pl[kb][7] = u.w;
          }
#pragma unroll
          for (int kb = 0; kb < 4; ++kb) {
            const int e0 = kb * 32;
            const uint64_t bdesc = desc_sw128(bbase + (e0 / 64) * (H * 128) + (e0 % 64) * 2);
            const uint64_t adesc = desc_sw128(sbase + w * C::kWStride + kb * 32);
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
              const int p = NW == 2 ? pp : mi;
              uint32_t mask[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) mask[q] = MS == 1 ? 0u : p ? ~pl[kb][q] : pl[kb][q];  // disable idx != p
              if (!(a.debug & 4))
                tc_mma_sp2_elect(tacc + (w * MS + p) * NT, adesc, bdesc, idesc | (uint32_t)(kb & 1), mask,
                                 tm + ecol + (kb & 2));
            }
          }
          tc_commit2_mc_elect(&wempty[st], 0x3);
          if constexpr (SPLIT) tc_commit2_mc_elect(&bempty[sb], 0x3);
        }
        tc_commit2_mc_elect(&acc_full[PW ? w : ab], 0x3);
        pc[7] += 1;
      }
      if (prof) pc[2] = clk() - tstart;
    } else if (!leader && warp == 5 && lane == 0 && gather) {
      // ============== peer: forward "gather landed" to the leader's full ==============
      uint32_t it = 0;
      TileInfo ti;
      for (int tile = pair0; decode_tile(a, NT, tile, ti); tile += pstep)
        for (int k = ti.k0; k < ti.k1; ++k, ++it) {
          const int sb = it % SB;
          if (SMY_RELAY_TRYWAIT)
            mbar_wait_cta(&bfull[sb], (it / SB) & 1);
          else
            mbar_spin(&bfull[sb], (it / SB) & 1);
          mbar_arrive_cluster(bfull_lead + sb * 8);
        }
    }
  } else if (warp >= 15 && !SPLIT && !epi4) {
    // idle: the lock-step kernel's fourth epilogue warps on a SEL-gather launch
  } else if ((warp >= 6 && warp < 10 && !epi3) || warp >= 15 && SPLIT) {
    // ============ SEL gather of this CTA's half of the token rows (cp.async) ============
    // Thread tb owns the 16-B chunk ch = tb % 16 of rows tb/16 + RS*i (i < H/RS,
    // RS = gather threads / 16) of the tile for every k-stage, so the row lookups,
    // source pointers and swizzled destination offsets are computed once per tile;
    // a stage is then H/RS (address add + cp.async) per thread.
    if (gather) {
      constexpr int GT = pair_gather_threads(SPLIT, NT), RS = GT / 16;
      const int tb = warp < 10 ? threadIdx.x - 6 * 32 : threadIdx.x - 15 * 32 + kGatherThreads;
      static_assert(GT % 32 == 0 && H % RS == 0, "gather mapping");
      const uint64_t pol_g = SMY_GATHER_EVICT_LAST ? policy_evict_last() : 0;
      constexpr int NI = H / RS;
      const int r0 = tb >> 4, ch = tb & 15;
      const uint32_t dst0 = (uint32_t)((ch >> 3) * (H * 128) + r0 * 128 + (((ch & 7) ^ (r0 & 7)) << 4));
      // swizzled destination of row r0 + RS*i relative to dst0 (RS % 8 == 0: the same
      // XOR pattern for every i; RS = 14 -- 7 gather warps -- changes it per row)
      auto dst_off = [&](int i) -> uint32_t {
        if (RS % 8 == 0) return 128u * RS * i;
        const int row = r0 + RS * i;
        return (uint32_t)((ch >> 3) * (H * 128) + row * 128 + (((ch & 7) ^ (row & 7)) << 4)) - dst0;
      };
      uint32_t it = 0;
      TileInfo ti;
      for (int tile = pair0; decode_tile(a, NT, tile, ti); tile += pstep) {
        const uint16_t* src[NI];
        uint32_t valid = 0;
        const int hh = pair_half(ti.n_local);
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          const int tl = r0 + RS * i;  // row within this CTA's half
          const int t = (int)cta * hh + tl;
          const int rid = (tl < hh && t < ti.n_local) ? a.sel_in[ti.row0 + ti.t0 + t] : -1;
          src[i] = (rid >= 0 ? x_row(a, rid) : a.x) + ch * 8;
          valid |= (rid >= 0 ? 1u : 0u) << i;
        }
        for (int k = ti.k0; k < ti.k1; ++k, ++it) {
          const int st = it % SB;
          unsigned long long tg0 = prof ? clk() : 0;
          if (SMY_GATHER_SPIN)
            mbar_spin(&bempty[st], ((it / SB) & 1) ^ 1);
          else
            mbar_wait_cta(&bempty[st], ((it / SB) & 1) ^ 1);
          if (prof) {
            const unsigned long long t1 = clk();
            pc[10] += t1 - tg0;
            tg0 = t1;
            if (tb == 0 && leader) {  // slot round trip: issue of stage it - SB -> this slot free again
              if (it >= (uint32_t)SB) pc[9] += t1 - ts_issue[st];
              ts_issue[st] = t1;
            }
          }
          const int64_t kcol0 = (int64_t)k * 128;
          const uint32_t bs = smem_u32(bsm(st)) + dst0;
          if (!(a.debug & 1)) {
            // rows past the tile's tokens are not loaded: their D columns are never read
#pragma unroll
            for (int i = 0; i < NI; ++i)
              if ((valid >> i) & 1u)
              {
                if (SMY_GATHER_EVICT_LAST)
                  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(bs + dst_off(i)),
                               "l"(src[i] + kcol0), "l"(pol_g)
                               : "memory");
                else
                  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(bs + dst_off(i)), "l"(src[i] + kcol0)
                               : "memory");
              }
          }
          cp_async_mbar_arrive_noinc(&bfull[st]);
          if (prof) pc[11] += clk() - tg0;
        }
      }
    }
  } else {
    // ==== epilogue (warps 0-3 and 10-13): this CTA's 128 lanes x all NT tokens ====
    // warp w reaches TMEM lanes 32*(w%4)..+31; warps w and w+10 split the
    // 16-column chunks (even / odd) so two warps per SM sub-partition hide the
    // epilogue's dependent-latency chains.
    const int q = warp & 3;
    const int h = warp >= 15 ? 3 : warp >= 10 ? 1 : warp >= 6 ? 2 : 0;  // this warp's share of the chunks
    const int cstep = 16 * NHW;
    if (a.pdl) griddep_wait();  // outputs (zeroed by the previous kernel) are written below
    if (a.zero_ptr != nullptr)
      zero_slice(a, (int64_t)blockIdx.x * 128 * NHW + (q + 4 * h) * 32 + lane, (int64_t)gridDim.x * 128 * NHW);
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const uint32_t acc_empty_leader = mapa_shared(smem_u32(acc_empty), 0);
    // the accumulator is cleared by the issuer's zero MMA at the start of each tile,
    // so a warp hands its TMEM columns back right after its last load of a tile
    auto release = [&](int b) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc_empty_leader + 8 * b);
    };
    for (int b = 0; b < (PW ? 2 : AB); ++b) release(b);
    uint32_t tcount = 0;
    TileInfo ti;
    const bool ilv = (NW == 1 || a.mtp_half) && a.epi == kEpiSiluMulIlv;
    for (int tile = pair0; decode_tile(a, NT, tile, ti); tile += pstep, ++tcount) {
      const int m_own = 2 * ti.m_tile + (int)cta;
      const int cr = m_own * kTileM + 32 * q + lane;
      const bool valid = m_own < a.m_tiles && cr < a.R;
      const int grp = cr;  // (1,2,V): one compressed row per group
      unsigned long long t0 = prof ? clk() : 0;
      const int ab = tcount % AB;
      const uint32_t tacc = tmem + ab * C::kAccCols;
      if (PW) {  // per-weight hand-off: drain weight 0, release it, then weight 1
        const int cg = 16 * (4 * m_own + q) + (lane & 15);
        const bool gvalid = m_own < a.m_tiles && cg < a.R / 2 && !(a.debug & 8);
#pragma unroll 1
        for (int w = 0; w < 2; ++w) {
          mbar_wait_cta(&acc_full[w], tcount & 1);
          tc_fence_after();
          const int cgw = cg + w * a.mtp_half * 64;  // a 128-lane m-tile holds 64 outputs
          for (int c0 = 16 * h; c0 < ti.n_local; c0 += cstep) {
            float v[2][16];
            tmem_ld16(tacc + lane_base + (2 * w) * NT + c0, v[0]);
            tmem_ld16(tacc + lane_base + (2 * w + 1) * NT + c0, v[1]);
            tmem_ld_wait();
            if (c0 + cstep >= ti.n_local) release(w);
            if (!(a.debug & 32))
              ilv_chunk(v, gvalid && cgw < a.R / 2, min(16, ti.n_local - c0), static_cast<uint16_t*>(a.out), a.ldo,
                        ti.row0 + ti.t0 + c0, cgw, lane, a.rows_out);
          }
          if (16 * h >= ti.n_local) release(w);  // no chunk of this tile for this warp
        }
        if (prof) pc[4] += clk() - t0;
        continue;
      }
      mbar_wait_cta(&acc_full[ab], (tcount / AB) & 1);
      if (prof) { const unsigned long long t1 = clk(); pc[3] += t1 - t0; t0 = t1; }
      tc_fence_after();
      if (ilv) {
        // lanes 0-15 gate / 16-31 up of the same 16 output pairs (reading R20)
        const int cg = 16 * (4 * m_own + q) + (lane & 15);
        const bool gvalid = m_own < a.m_tiles && cg < a.R / 2 && !(a.debug & 8);
        for (int c0 = 16 * h; c0 < ti.n_local; c0 += cstep) {
          const unsigned long long tl0 = prof ? clk() : 0;
          if constexpr (MS == 2 && NW == 2) {  // m-tile pairing: weight 1 = m-tiles [half, 2 half)
            float v[2][2][16];
#pragma unroll
            for (int w = 0; w < 2; ++w) {
              tmem_ld16(tacc + lane_base + (2 * w) * NT + c0, v[w][0]);
              tmem_ld16(tacc + lane_base + (2 * w + 1) * NT + c0, v[w][1]);
            }
            tmem_ld_wait();
            if (c0 + cstep >= ti.n_local) release(ab);
            if (prof) pc[8] += clk() - tl0;
            const int cg1 = cg + a.mtp_half * 64;  // a 128-lane m-tile holds 64 outputs
            if (!(a.debug & 32)) {
              ilv_chunk(v[0], gvalid, min(16, ti.n_local - c0), static_cast<uint16_t*>(a.out), a.ldo,
                        ti.row0 + ti.t0 + c0, cg, lane, a.rows_out);
              ilv_chunk(v[1], gvalid && cg1 < a.R / 2, min(16, ti.n_local - c0), static_cast<uint16_t*>(a.out),
                        a.ldo, ti.row0 + ti.t0 + c0, cg1, lane, a.rows_out);
            }
          } else if constexpr (MS == 2) {
            float v[2][16];
            tmem_ld16(tacc + lane_base + c0, v[0]);
            tmem_ld16(tacc + lane_base + NT + c0, v[1]);
            tmem_ld_wait();
            if (c0 + cstep >= ti.n_local) release(ab);
            if (prof) pc[8] += clk() - tl0;
            if (!(a.debug & 32))
              ilv_chunk(v, gvalid, min(16, ti.n_local - c0), static_cast<uint16_t*>(a.out), a.ldo,
                        ti.row0 + ti.t0 + c0, cg, lane, a.rows_out);
          } else {  // N = M: one slot
            float v[16];
            tmem_ld16(tacc + lane_base + c0, v);
            tmem_ld_wait();
            if (c0 + cstep >= ti.n_local) release(ab);
            if (prof) pc[8] += clk() - tl0;
            if (!(a.debug & 32))
              ilv_chunk_ms1(v, gvalid, min(16, ti.n_local - c0), static_cast<uint16_t*>(a.out), a.ldo,
                            ti.row0 + ti.t0 + c0, cg, lane);
          }
        }
      }
      for (int c0 = 16 * h; !ilv && c0 < ti.n_local; c0 += cstep) {
        float v[NW][MS][16];
        const unsigned long long tl0 = prof ? clk() : 0;
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int p = 0; p < MS; ++p) tmem_ld16(tacc + lane_base + (w * MS + p) * NT + c0, v[w][p]);
        tmem_ld_wait();
        if (c0 + cstep >= ti.n_local) release(ab);
        if (prof) pc[8] += clk() - tl0;
        const int jmax = min(16, ti.n_local - c0);
        const int n = (valid && !(a.debug & 8)) ? jmax : 0;
        if (a.epi == kEpiScatter) {
          // destination rows / gate weights of these 16 tokens: one load per lane,
          // broadcast by shuffle; then 16 independent predicated reductions
          const int rl = ti.row0 + ti.t0 + c0 + (lane & 15);
          float* my_row = (lane & 15) < jmax ? out_row(a, a.sel_out ? a.sel_out[rl] : rl) : nullptr;
          const float my_s = (lane & 15) < jmax ? (a.scale ? a.scale[rl] : 1.f) : 0.f;
          if constexpr (MS == 2) {
            scatter_chunk_v4(v[0][0], v[0][1], my_row, my_s, n, grp, lane);
            if (NW == 2 && a.mtp_half) {  // m-tile pairing: weight 1 = compressed rows + mtp_half * 128
              const int g1 = grp + a.mtp_half * kTileM;
              scatter_chunk_v4(v[NW - 1][0], v[NW - 1][1], my_row, my_s,
                               (valid && g1 < a.R && !(a.debug & 8)) ? jmax : 0, g1, lane);
            }
          } else if (NW == 2) {  // m-tile pairing: weight w = output rows offset by w * mtp_half * 128
            const int off1 = a.mtp_half * kTileM;
            const int n1 = (valid && cr + off1 < a.R && !(a.debug & 8)) ? jmax : 0;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float* o = reinterpret_cast<float*>(
                  __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j));
              const float sc = __shfl_sync(0xffffffffu, my_s, j);
              if (j < n) atomicAdd(o + cr, sc * v[0][0][j]);
              if (j < n1) atomicAdd(o + cr + off1, sc * v[NW - 1][0][j]);
            }
          } else {  // N == M: lane = output row
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              float* o = reinterpret_cast<float*>(
                  __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(my_row), j));
              const float sc = __shfl_sync(0xffffffffu, my_s, j);
              if (j < n) atomicAdd(o + cr, sc * v[0][0][j]);
            }
          }
          continue;
        }
        if (MS == 1 && NW == 2 && a.mtp_half) {  // m-tile pairing, compact fp32 / bf16
          const int64_t r0 = ti.row0 + ti.t0 + c0;
          const int off1 = a.mtp_half * kTileM;
          const int n1 = (valid && cr + off1 < a.R && !(a.debug & 8)) ? jmax : 0;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const int col = cr + w * off1, nw_ = w ? n1 : n;
            if (a.out_bf16) {
              uint16_t* o = static_cast<uint16_t*>(a.out) + r0 * a.ldo + col;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if (j < nw_) *o = __bfloat16_as_ushort(__float2bfloat16_rn(v[w][0][j]));
                o += a.ldo;
              }
            } else {
              float* o = static_cast<float*>(a.out) + r0 * a.ldo + col;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                if (j < nw_) *o = v[w][0][j];
                o += a.ldo;
              }
            }
          }
          continue;
        }
        if constexpr (MS == 1 && NW == 2) {  // N == M, gate and up: lane = output row
          const int64_t r0 = ti.row0 + ti.t0 + c0;
          uint16_t* o = static_cast<uint16_t*>(a.out) + r0 * a.ldo + cr;
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < n) *o = __bfloat16_as_ushort(__float2bfloat16_rn(silu_mul(v[0][0][j], v[1][0][j])));
            o += a.ldo;
          }
          continue;
        }
        if constexpr (MS == 1) {  // N == M compact: lane = output row, fp32 or bf16
          const int64_t r0 = ti.row0 + ti.t0 + c0;
          if (a.out_bf16) {
            uint16_t* o = static_cast<uint16_t*>(a.out) + r0 * a.ldo + cr;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j < n) *o = __bfloat16_as_ushort(__float2bfloat16_rn(v[0][0][j]));
              o += a.ldo;
            }
          } else {
            float* o = static_cast<float*>(a.out) + r0 * a.ldo + cr;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              if (j < n) *o = v[0][0][j];
              o += a.ldo;
            }
          }
          continue;
        }
        // compact epilogues: values first, then predicated stores walking one row pointer
        uint32_t packed[16];
        float2 f2[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (NW == 2) {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(silu_mul(v[0][0][j], v[NW - 1][0][j]),
                                                            silu_mul(v[0][1 % MS][j], v[NW - 1][1 % MS][j]));
            packed[j] = *reinterpret_cast<const uint32_t*>(&h2);
          } else {
            const __nv_bfloat162 h2 = __floats2bfloat162_rn(v[0][0][j], v[0][1 % MS][j]);
            packed[j] = *reinterpret_cast<const uint32_t*>(&h2);
            f2[j] = make_float2(v[0][0][j], v[0][1 % MS][j]);
          }
        }
        const int64_t r0 = ti.row0 + ti.t0 + c0;
        if (NW == 2 || a.out_bf16) {
          uint32_t* o = reinterpret_cast<uint32_t*>(static_cast<uint16_t*>(a.out) + r0 * a.ldo + 2 * grp);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < n) *o = packed[j];
            o += a.ldo / 2;
          }
        } else {
          float2* o = reinterpret_cast<float2*>(static_cast<float*>(a.out) + r0 * a.ldo + 2 * grp);
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (j < n) *o = f2[j];
            o += a.ldo / 2;
          }
        }
      }
      if (16 * h >= ti.n_local) release(ab);  // no chunk of this tile for this warp
      if (prof) pc[4] += clk() - t0;
    }
  }
  if (prof) {
    unsigned long long* o = a.prof + ((size_t)(a.epi == kEpiScatter) * 148 + blockIdx.x) * 16;
    if (warp == 5 && lane == 0) {
      atomicAdd(o + 0, pc[0] + pc[6]); atomicAdd(o + 1, pc[1]); atomicAdd(o + 2, pc[2]); atomicAdd(o + 6, pc[6]);
      atomicAdd(o + 7, pc[7]);
    }
    if (warp == 6 && lane == 0) { atomicAdd(o + 10, pc[10]); atomicAdd(o + 11, pc[11]); atomicAdd(o + 9, pc[9]); }
    if (warp == 5 && lane == 0 && SPLIT) atomicAdd(o + 12, pc[8]);
    if (warp == 0 && lane == 0) { atomicAdd(o + 3, pc[3]); atomicAdd(o + 4, pc[4]); atomicAdd(o + 8, pc[8]); }
    if (warp == 4 && lane == 0) { atomicAdd(o + 5, pc[5]); }
  }
  if (prof) {  // CTA lifetime (ns) up to here, and the time its MMA work ended
    unsigned long long* o = a.prof + ((size_t)(a.epi == kEpiScatter) * 148 + blockIdx.x) * 16;
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long g_end = gtime();
      atomicAdd(o + 13, g_end - g_start);
      o[14] = g_start;  // the last call's start / end (absolute ns)
      o[15] = g_end;
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 5) tmem_dealloc2(tmem, C::kTmemCols);
}

template <int NT, int NW, int MS, int SPLIT>
smy_status launch_pair_t(const SsmmArgs& a, cudaStream_t s) {
  using C = PairCfg<NT, NW, MS, SPLIT>;
  static bool configured = false;
  static int num_sms = 0;
  auto kern = ssmm_pair_kernel<NT, NW, MS, SPLIT>;
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
  // stream-K launches use every pair: with fewer tiles than pairs the K pieces fill them
  const int pairs = (b.streamk || a.max_tiles >= num_sms / 2) ? num_sms / 2 : a.max_tiles;
  b.workers = pairs;
  // m-tile fastest (concurrent tiles share the token tile in L2) for the scatter (down)
  // launches, and for SEL-gather launches whose token pool does not fit in L2 (their
  // n-fastest order would re-stream the gathered rows from HBM for every m-tile)
  b.m_fastest = (a.epi == kEpiScatter || (a.sel_in != nullptr && (int64_t)a.x_rows * a.ldx * 2 > kGatherL2Bytes)) &&
                !(a.debug & 2048);
  if (b.pdl) {  // programmatic dependent launch (SsmmArgs::pdl); cluster dims are compiled in
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(pair_threads(SPLIT, NT));
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
  kern<<<2 * pairs, pair_threads(SPLIT, NT), C::kSmemBytes, s>>>(b);
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
