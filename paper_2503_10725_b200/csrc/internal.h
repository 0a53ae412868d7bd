// Internal declarations shared by the library's translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "samoyeds.h"

namespace smy {

constexpr int kTileM = 128;       // compressed rows per tile (TMEM lanes)
constexpr int kStageVK = 128;     // virtual logical K per pipeline stage (4 x K32)
constexpr int kABytes = 16384;    // A smem image per stage
constexpr int kEBytes = 2048;     // E TMEM image per stage
constexpr int kMaxGroups = 128;   // experts per grouped launch
constexpr int kMaxPeers = 8;      // ranks of one NVLink/NVSwitch node (expert parallelism)

// widest token tile of the (1,2,V) single-weight kernels (interleaved gate/up, down);
// a build knob for A/B experiments (probes/), 224 by default
#ifndef SMY_NT_WIDE
#define SMY_NT_WIDE 224
#endif
// token tile of the m-tile-paired (1,2,V) gate/up on the CTA pair (two m-tiles x two
// slots x SMY_MTP_NT accumulator columns must fit TMEM beside the E columns)
#ifndef SMY_MTP_NT
#define SMY_MTP_NT 112
#endif
// token-ring depth of the SEL-gather pair launches (SPLIT rings; capped by what fits
// beside 3 weight slots: 7 at NT = 112 (the m-tile-paired gate/up), 5 at NT = 224;
// 5 -> 7 at NT = 112: token-ring waits 495 k -> 391 k cycles, gate/up -2 to -3 %)
#ifndef SMY_TOKEN_SLOTS
#define SMY_TOKEN_SLOTS 7
#endif

struct Geometry {
  int64_t R;        // compressed rows = rows * N / M
  int m_tiles, k_stages, planes, rep, block;
  int ms;           // accumulator slots per weight: M, or 1 when N == M
};

smy_status geometry(const smy_wdesc* d, Geometry* g);
void set_last_error(const char* msg);
smy_status cuda_status(cudaError_t e);

// ---------------------------------------------------------------- SSMM
enum EpiKind { kEpiCompact = 0, kEpiSiluMul = 1, kEpiScatter = 2, kEpiSiluMulIlv = 3 };
// kEpiSiluMulIlv: one weight whose compressed rows alternate 16 gate / 16 up rows
// (the interleaved gate/up weight, reading R20); the epilogue pairs TMEM
// lane l (gate) with lane l + 16 (up) of the same warp by shuffles.

struct SsmmArgs {
  CUtensorMap tmap_x;               // contiguous x rows: 2D TMA box 64 x NT, 128B swizzle
  CUtensorMap tmap_w;       // pair kernel: all weight images as rows of 128 B from `wbase`
  const uint8_t* wbase;
  const uint8_t* img0[kMaxGroups];  // weight image per group (gate / single)
  const uint8_t* img1[kMaxGroups];  // up weight image (SILU_MUL only)
  int num_groups;
  // weight geometry (identical for every group)
  int R, m_out, n_fmt, m_fmt, m_tiles, k_stages, planes, block;
  // activations
  const uint16_t* x;
  int64_t ldx, x_rows;
  const int32_t* sel_in;   // gather rows: x row = sel_in[row0 + t]; NULL: x row = row0 + t
  const int32_t* offsets;  // per-group row ranges [G+1]; NULL: single group of n_sel rows
  const int32_t* tile_prefix;  // per-group tile prefix [G+1]; NULL: single group
  int n_sel;
  // epilogue
  int epi, out_bf16;
  void* out;
  int64_t ldo;
  const int32_t* sel_out;  // scatter destinations (SCATTER only)
  const int32_t* rows_out;  // SILU_MUL_ILV output row of compact row r (ablation variant only; NULL: r)
  // m-tile pairing (N = M single weights on the pair kernel, NW = 2): "weight" 1 is the
  // same weight's m-tiles [mtp_half, 2 mtp_half) (img1 = img0 + mtp_half m-tiles), so every
  // token stage feeds two accumulators; output rows of weight w are offset by
  // w * mtp_half * 128; m_tiles = mtp_half; 0 = off
  int mtp_half;
  // in-smem row expansion of an (N, 2N, 32) image, N > 1 (ssmm_kernel<..., XP = 1>): set by
  // ssmm_launch from the format; 0 = the lane-masked M-slot remap
  int xp;
  // programmatic dependent launch: the launch may start while the previous kernel of
  // the stream (the gate/up SSMM) still runs; its producer streams the first ring of
  // WEIGHT stages, then waits (griddepcontrol.wait) before the dependent token loads,
  // and the epilogue waits before its first output write (contiguous-B launches only)
  int pdl;
  const float* scale;      // scatter scale, NULL = 1
  int max_tiles;           // tile count (single group) / upper bound (grouped)
  int weights_stream;      // 1: weights read once per call (decode) -> L2 evict_first
  int k_splits;            // >1: split K across tiles (SCATTER epilogue only; partial sums add)
  int streamk;             // 1: last partial wave of tiles split along K over all workers (SCATTER only)
  int workers;             // CTAs (single) / CTA pairs (pair kernel) of the launch; set by the launcher
  int m_fastest;           // tile order: m-tile fastest (B shared in L2) instead of n-tile fastest
  // expert parallelism over peer memory (NVLink P2P): gathered row i is token
  // row_map[i] & 0xFFFFFF of rank row_map[i] >> 24, read from x_peers[rank]; the
  // scatter-add of row i goes to out_peers[rank] (ldo) -- no dispatched copies
  const int32_t* row_map;
  // zero this fp32 buffer (zero_elems, multiple of 4) on the way: the layer's output,
  // cleared by the gate/up launch's epilogue warps before their first tile instead
  // of a separate memset launch (the down launch that adds into it runs after)
  float* zero_ptr;
  int64_t zero_elems;
  const uint16_t* x_peers[kMaxPeers];
  float* out_peers[kMaxPeers];
  int debug;               // profiling switches (env SMY_DEBUG): 1 no gather copies, 2 no weight
                           // copies, 4 no MMAs, 8 no epilogue math/stores -- results are garbage;
                           // 128: per-role cycle counters into `prof` (results valid)
  unsigned long long* prof;  // [2 epilogue kinds][148][16] role cycle counters (SMY_DEBUG & 128)
};
unsigned long long* debug_prof_buffer(int ctas);
int debug_flags();

// K-split count for a scatter-add launch with `tiles` (expert, m, n) tiles.
int ssmm_pick_ksplit(int64_t tiles, int k_stages);

// Tensor map over a token-major bf16 activation matrix [rows x cols] (ld elements):
// boxes of 64 elements x box_rows rows, 128-byte swizzle (the UMMA K-major atom).
smy_status make_w_tmap(CUtensorMap* map, const void* base, int64_t rows, int box_rows);
smy_status make_x_tmap(CUtensorMap* map, const void* x, int64_t cols, int64_t rows, int64_t ld, int box_rows);

struct SsmmPlan {
  int nt, nw, ms, rep;
};
// Choose the token tile for a launch given the expected tokens per group.
int ssmm_pick_nt(int nw, int ms, int rep, int64_t tokens_per_group, int xp = 0);
// gathered token pools larger than this run their tiles m-tile fastest (L2 is 126 MB;
// the weight tiles in flight and the outputs share it)
constexpr int64_t kGatherL2Bytes = 64ll << 20;
smy_status ssmm_launch(const SsmmArgs& a, int nt, int nw, int ms, int rep, cudaStream_t s);
// CTA-pair (cta_group::2) kernel: a.m_tiles / tile prefixes count m-tile PAIRS, tmap box = nt/2 rows
// returns the cluster size to use (2: one MMA pair, 4: two pairs sharing weights) or 0 (single CTA)
// gather: the launch reads x through SEL.  Such launches with the lane-masked
// (1,2,V) remap and tiles of <= SMY_SINGLE_FAST_GATHER_NT tokens stay on the
// single-CTA kernel (weight-streaming regime: its deeper weight ring and
// precomputed-pointer gather beat the CTA pair there, profiles/r2_midrange.md)
#ifndef SMY_SINGLE_FAST_GATHER_NT
#define SMY_SINGLE_FAST_GATHER_NT 128
#endif
int ssmm_pair_cluster(int nt, int nw, int ms, int rep, int m_tiles, int64_t tokens_per_group, int gather);
smy_status ssmm_launch_pair(const SsmmArgs& a, int nt, int nw, int ms, int cl, cudaStream_t s);
// can one tensor map address all these images (else: single-CTA kernel)
bool ssmm_pair_images_ok(const smy_weight* const* w0, const smy_weight* const* w1, int groups, size_t img_bytes);

// --------------------------------------------------------------- routing
smy_status route_launch(const float* logits, int64_t T, int E, int k, int gating, int32_t* ids, float* w,
                        int32_t* counts, int32_t* offsets, int32_t* sel, float* gw, void* ws, size_t ws_bytes,
                        const int* tile_nt, const int* tile_mt, int n_tile_cfgs, int32_t* tile_prefix,
                        cudaStream_t s, int num_shared = 0);
size_t route_ws_bytes(int64_t T, int E);
smy_status compact_launch(const int32_t* keys, const float* vals, int64_t T, int nb, int k, int32_t* counts,
                          int32_t* offsets, int32_t* sel, float* gw, void* ws, size_t ws_bytes, const int* tile_nt,
                          const int* tile_mt, int n_tile_cfgs, int32_t* tile_prefix, cudaStream_t s);

// --------------------------------------------------------------- compress
smy_status decompress_launch(const smy_weight* src, uint16_t* w, int64_t ldw, int32_t* d_status, cudaStream_t s);
smy_status sel_check_launch(const int32_t* sel, int32_t n, int64_t x_rows, int32_t* d_status, cudaStream_t s);
constexpr int kDebugValidate = 65536;  // SMY_DEBUG bit: validate SEL in samoyeds_ssmm (synchronising)
// interleaved gate/up weight (reading R20): canonical rows moved, image re-packed
smy_status interleave_launch(const smy_weight* gate, const smy_weight* up, const smy_wdesc& d, const Geometry& g,
                             smy_weight* gu, cudaStream_t s);
// formats with an interleaved gate/up epilogue: (1,2,V) and N = M (plain 2:4), V % 32 == 0
// formats whose SSMMs run the in-smem row expansion: N > 1, M = 2N,
// V % 32 == 0 -- (4,8,32), (8,16,32), (2,4,32); SMY_DEBUG=8388608 keeps the M-slot remap
constexpr int kDebugNoXp = 8388608;
inline bool xp_format(const smy_format& f) { return f.n > 1 && f.m == 2 * f.n && f.v % 32 == 0; }
bool xp_on(const smy_format& f);  // xp_format and not disabled by SMY_DEBUG
inline bool ilv_format(const smy_format& f) {
  return f.v % 32 == 0 && ((f.n == 1 && f.m == 2) || f.n == f.m || xp_format(f));
}
smy_status compress_launch(const smy_wdesc* d, const Geometry& g, const uint16_t* w, int64_t ldw, int flags,
                           smy_weight* out, int32_t* d_status, cudaStream_t s);

// --------------------------------------------------------------- helpers
smy_status silu_mul_launch(const float* g, const float* u, int64_t rows, int64_t cols, uint16_t* out,
                           cudaStream_t s);
smy_status check_arch();
void count_launch(int n = 1);
size_t ep_plan_ws_bytes(int64_t T, int world, int k);
smy_status ep_plan_launch(const int32_t* ids, const float* w, int64_t T, int k, int E, int world, int32_t* counts,
                          int32_t* offsets, int32_t* sel, int32_t* tag_ids, float* tag_w, void* ws, size_t ws_bytes,
                          cudaStream_t s);
smy_status ep_pack_launch(const uint16_t* x, int64_t ldx, int64_t d, const int32_t* offsets, int world,
                          const int32_t* sel, int64_t max_rows, uint16_t* xs, cudaStream_t s);
smy_status ep_combine_launch(const float* back, int64_t d, const int32_t* offsets, int world, const int32_t* sel,
                             int64_t max_rows, float* out, cudaStream_t s);
// expert parallelism over peer memory: where a received row's token lives / its output goes
struct PeerRows {
  int world;
  const int32_t* row_map;              // dev [rows]: (source rank << 24) | token id
  const uint16_t* x_peers[kMaxPeers];  // source ranks' bf16 token rows (NVLink-mapped)
  float* out_peers[kMaxPeers];         // source ranks' fp32 outputs (P2P reductions)
  int64_t ldx, ldo;
};
smy_status moe_core(const smy_moe_config* c, const smy_weight* experts, const smy_weight* shared, const void* x,
                    const float* logits, const int32_t* keys, const float* vals, int64_t T, float* out,
                    void* workspace, size_t ws_bytes, cudaStream_t s, const PeerRows* peers = nullptr);
smy_status moe_workspace_bytes(const smy_moe_config* c, int64_t T, size_t* bytes);
smy_status ep_unique_id(void* out128);
smy_status ep_comm_create(const void* id128, int rank, int world, smy_ep_comm** out);
smy_status ep_comm_destroy(smy_ep_comm* c);
int ep_comm_world(const smy_ep_comm* c);
smy_status ep_workspace_bytes(const smy_moe_config* c, int64_t T, int world, size_t* bytes);
smy_status ep_layer(const smy_moe_config* c, const smy_weight* experts, const void* x, const float* logits, int64_t T,
                    float* out, void* workspace, size_t ws_bytes, smy_ep_comm* comm, cudaStream_t s);
smy_status ep_row_ids_launch(const int32_t* sel, const int32_t* offsets, int world, int rank, int64_t max_rows,
                             int32_t* row_ids, cudaStream_t s);
void record_phase(int i, cudaStream_t s);  // no-op unless bench hooks are set
smy_status moe_variant_bytes(const smy_moe_config* c, int64_t T, int v, size_t* bytes);
smy_status moe_set_variant(int v, void* scratch, size_t bytes);

}  // namespace smy
