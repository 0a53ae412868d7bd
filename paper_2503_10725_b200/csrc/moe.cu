// samoyeds_moe_layer: the whole permutation-free MoE expert path on one GPU
// (§3.1 P:187-189 redundancy removed; §4.5 P:374 compressed output
// layout; §6.2 P:493 shared experts):
//
//   route + compaction (3 small kernels)  ->  memset(out)
//   grouped gate/up SSMM, fused SiLU*up, compact bf16 intermediate [sum n_e x f]
//   grouped down SSMM, fused routing-weight scale + scatter-add into out
//   shared experts: same two launches with SEL = all tokens, weight 1
//
// Every launch reads the routing result on the device (tile prefixes written by
// the scan kernel), so the layer never synchronises with the host and is CUDA-
// graph capturable.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "internal.h"

namespace smy {

namespace {
size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct LayerWs {
  int32_t *ids, *counts, *offsets, *sel, *prefix;
  float *w, *gw;
  void* route_ws;
  size_t route_ws_bytes;
  uint16_t* inter;
  float *fallback_g, *fallback_u;
  size_t total;
};

LayerWs carve(const smy_moe_config* c, int64_t T, bool fallback, uint8_t* base) {
  LayerWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t* p = base ? base + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  // shared experts are compacted and run as extra groups (k + ns entries per token)
  const int ns = c->num_shared > 0 ? c->num_shared : 0;
  const int64_t Tk = T * (c->top_k + ns);
  const int E = c->num_experts + ns;
  w.ids = reinterpret_cast<int32_t*>(take(Tk * 4));
  w.w = reinterpret_cast<float*>(take(Tk * 4));
  w.counts = reinterpret_cast<int32_t*>(take(E * 4));
  w.offsets = reinterpret_cast<int32_t*>(take((E + 1) * 4));
  w.sel = reinterpret_cast<int32_t*>(take(Tk * 4));
  w.gw = reinterpret_cast<float*>(take(Tk * 4));
  w.prefix = reinterpret_cast<int32_t*>(take(2 * (E + 1) * 4));
  w.route_ws_bytes = route_ws_bytes(T, E);
  w.route_ws = take(w.route_ws_bytes);
  const int64_t inter_rows = Tk > T ? Tk : T;  // shared experts reuse it with T rows
  w.inter = reinterpret_cast<uint16_t*>(take((size_t)inter_rows * c->ffn * 2));
  if (fallback) {
    w.fallback_g = reinterpret_cast<float*>(take((size_t)inter_rows * c->ffn * 4));
    w.fallback_u = reinterpret_cast<float*>(take((size_t)inter_rows * c->ffn * 4));
  }
  w.total = off;
  return w;
}

__global__ void silu_mul_kernel(const float* g, const float* u, int64_t n, uint16_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gv = g[i];
    out[i] = __bfloat16_as_ushort(__float2bfloat16_rn(gv / (1.f + expf(-gv)) * u[i]));
  }
}
}  // namespace

smy_status silu_mul_launch(const float* g, const float* u, int64_t rows, int64_t cols, uint16_t* out,
                           cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n <= 0) return SMY_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  silu_mul_kernel<<<blocks, 256, 0, s>>>(g, u, n, out);
  count_launch();
  return cuda_status(cudaGetLastError());
}

static bool gate_up_fused(const Geometry& g) { return !(g.ms >= 16); }

// m-tile pairing of the interleaved (1,2,V) gate/up on the CTA pair (0 = off): two
// m-tiles per SEL-gathered token stage at NT = 112 -- four lane-masked MMAs per window
// instead of two at NT = 224, half the token bytes per MMA (Qwen2 gate/up 0.635 ->
// 0.598 ms, Mixtral neutral, DeepSeek -2 %; SMY_DEBUG=1048576 turns it off)
static int gu_mtp_half(bool ilv, int cl_gu, const Geometry& ggu, int nt_gu) {
  if (!ilv || cl_gu != 2 || ggu.ms != 2 || nt_gu != SMY_NT_WIDE || ggu.m_tiles < 3 || (debug_flags() & 1048576))
    return 0;
  return (ggu.m_tiles + 1) / 2;
}

// m-tile pairing of an N = M down launch (0 = off): wide token tiles on the CTA pair
static int down_mtp_half(const Geometry& gdn, int64_t tpg, int64_t tpg_hi) {
  if (gdn.rep != 1 || gdn.m_tiles < 3 || (debug_flags() & 131072)) return 0;
  const int half = (gdn.m_tiles + 1) / 2;
  if (gdn.ms == 1)
    return ssmm_pick_nt(2, 1, 1, tpg_hi) == 224 && ssmm_pair_cluster(224, 2, 1, 1, half, tpg, 0) == 2 ? half : 0;
  // (1,2,V) down with NT = 112, two m-tiles per token stage: measured slower (Mixtral down
  // 0.337 -> 0.378 ms, Qwen2 0.350 -> 0.374; DeepSeek -1.7 %) -- opt-in, SMY_DEBUG=2097152
  if (gdn.ms == 2 && (debug_flags() & 2097152))
    return ssmm_pick_nt(1, 2, 1, tpg_hi) == SMY_NT_WIDE && ssmm_pair_cluster(112, 2, 2, 1, half, tpg, 0) == 2 ? half
                                                                                                              : 0;
  return 0;
}
static int down_mtp_nt(const Geometry& gdn) { return gdn.ms == 1 ? 224 : 112; }

static bool interleaved(const smy_moe_config* c) { return c->gate_up == SMY_GU_INTERLEAVED; }

smy_status moe_workspace_bytes(const smy_moe_config* c, int64_t T, size_t* bytes) {
  smy_wdesc d{c->ffn, c->hidden, c->fmt};
  Geometry g;
  smy_status st = geometry(&d, &g);
  if (st != SMY_OK) return st;
  *bytes = carve(c, T, !interleaved(c) && !gate_up_fused(g), nullptr).total;
  // bf16 layer output: the fp32 accumulation buffer after the layer's own regions
  if (c->out_dtype == SMY_BF16) *bytes += align_up((size_t)T * c->hidden * 4, 256);
  return SMY_OK;
}

namespace {
__global__ void f32_to_bf16_kernel(const float4* __restrict__ in, int64_t n4, uint2* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = in[i];
    const __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    out[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
  }
}
}  // namespace

// grouped SSMM over `groups` weights; tile prefix already on the device
static smy_status grouped(const smy_weight* const* w0, const smy_weight* const* w1, int groups, const Geometry& g,
                          int m_out, int nt, int nw, const uint16_t* x, int64_t ldx, int64_t x_rows,
                          const int32_t* sel_in, const int32_t* offsets, const int32_t* prefix, int max_tiles,
                          int epi, void* out, int64_t ldo, int out_bf16, const int32_t* sel_out,
                          const float* scale, int64_t k_cols, int stream_w, int k_splits, int cl,
                          cudaStream_t s, const PeerRows* peers = nullptr, float* zero_ptr = nullptr,
                          int64_t zero_elems = 0, const int32_t* rows_out = nullptr, int mtp_half = 0,
                          int pdl = 0) {
  SsmmArgs a;
  memset(&a, 0, sizeof(a));
  a.rows_out = rows_out;
  a.pdl = pdl;
  a.zero_ptr = zero_ptr;
  a.zero_elems = zero_elems;
  if (peers != nullptr) {
    a.row_map = peers->row_map;
    for (int p = 0; p < peers->world; ++p) {
      a.x_peers[p] = peers->x_peers[p];
      a.out_peers[p] = peers->out_peers[p];
    }
  }
  for (int e = 0; e < groups; ++e) {
    a.img0[e] = static_cast<const uint8_t*>(w0[e]->image);
    a.img1[e] = w1 ? static_cast<const uint8_t*>(w1[e]->image) : nullptr;
  }
  a.num_groups = groups;
  // (N, 2N, 32) weights: the in-smem row expansion (single-CTA, one weight per launch)
  a.xp = (nw == 1 && cl == 0 && mtp_half == 0 && xp_on(w0[0]->d.fmt)) ? 1 : 0;
  a.R = (int)g.R;
  a.m_out = m_out;
  a.n_fmt = g.ms == 1 ? 1 : w0[0]->d.fmt.n;
  a.m_fmt = g.ms == 1 ? 1 : w0[0]->d.fmt.m;
  a.m_tiles = g.m_tiles;
  a.k_stages = g.k_stages;
  a.planes = g.planes;
  a.block = g.block;
  a.x = x;
  a.ldx = ldx;
  a.x_rows = x_rows;
  a.sel_in = sel_in;
  a.offsets = offsets;
  a.tile_prefix = prefix;
  a.n_sel = 0;
  a.epi = epi;
  a.out_bf16 = out_bf16;
  a.out = out;
  a.ldo = ldo;
  a.sel_out = sel_out;
  a.scale = scale;
  a.max_tiles = max_tiles * k_splits;
  a.weights_stream = stream_w;
  a.k_splits = k_splits;
  if (mtp_half > 0) {  // m-tile pairing: "weight" 1 = the same weight's m-tiles [half, 2 half)
    for (int e = 0; e < groups; ++e) a.img1[e] = a.img0[e] + (size_t)mtp_half * g.k_stages * g.block;
    a.m_tiles = mtp_half;
    a.mtp_half = mtp_half;
  }
  smy_status st = make_x_tmap(&a.tmap_x, x, k_cols, x_rows, ldx, cl ? nt / 2 : nt);
  if (st != SMY_OK) return st;
  return cl ? ssmm_launch_pair(a, nt, nw, g.ms, cl, s) : ssmm_launch(a, nt, nw, g.ms, g.rep, s);
}

// ---- ablation variants (the paper's breakdown, and
// the compressed-output-layout figure).  NOT the product path: the layer
// runs them only between smy_moe_set_variant(v != 0) and smy_moe_set_variant(0), on
// the calling thread, with caller-provided scratch.
//   SMY_VARIANT_PERMUTE ("+W"): the input permutation materialised -- xp = x[SEL]
//     (expert-major copy), gate/up on xp as contiguous rows (2D TMA, no gather),
//     down into compact fp32 rows y, then the un-permute out[sel[i]] += gw[i] y[i]
//   SMY_VARIANT_DENSE_INTER (no compressed output layout): the intermediate is an
//     [E x T x f] token-position layout, zero-filled every call (the zero rows are
//     the redundant transfers P:374 removes); gate/up stores row e*T + sel[i], the
//     down launch gathers those rows back through SEL
namespace {
struct Variant {
  int v = 0;
  uint8_t* scratch = nullptr;
  size_t bytes = 0;
};
thread_local Variant t_variant;

__global__ void permute_rows_kernel(const uint16_t* __restrict__ x, int64_t d, const int32_t* __restrict__ sel,
                                    const int32_t* __restrict__ offsets, int E, uint16_t* __restrict__ xp) {
  const int64_t n = offsets[E], v8 = d / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * v8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / v8, c = i % v8;
    reinterpret_cast<uint4*>(xp + r * d)[c] = reinterpret_cast<const uint4*>(x + (int64_t)sel[r] * d)[c];
  }
}
__global__ void unpermute_rows_kernel(const float* __restrict__ y, int64_t d, const int32_t* __restrict__ sel,
                                      const float* __restrict__ gw, const int32_t* __restrict__ offsets, int E,
                                      float* __restrict__ out) {
  const int64_t n = offsets[E], v4 = d / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * v4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / v4, c = i % v4;
    const float4 a = reinterpret_cast<const float4*>(y + r * d)[c];
    const float g = gw[r];
    atomicAdd(reinterpret_cast<float4*>(out + (int64_t)sel[r] * d) + c, make_float4(g * a.x, g * a.y, g * a.z, g * a.w));
  }
}
__global__ void dense_rows_kernel(const int32_t* __restrict__ sel, const int32_t* __restrict__ offsets, int E,
                                  int64_t T, int32_t* __restrict__ rows) {
  for (int e = blockIdx.x; e < E; e += gridDim.x)
    for (int i = offsets[e] + threadIdx.x; i < offsets[e + 1]; i += blockDim.x) rows[i] = (int32_t)(e * T + sel[i]);
}
size_t variant_bytes(const smy_moe_config* c, int64_t T, int v) {
  const int ns = c->num_shared > 0 ? c->num_shared : 0;
  const int64_t Tk = T * (c->top_k + ns);
  if (v == SMY_VARIANT_PERMUTE) return align_up((size_t)Tk * c->hidden * 2, 256) + align_up((size_t)Tk * c->hidden * 4, 256);
  if (v == SMY_VARIANT_DENSE_INTER)
    return align_up((size_t)(c->num_experts + ns) * T * c->ffn * 2, 256) + align_up((size_t)Tk * 4, 256);
  return 0;
}
}  // namespace

smy_status moe_variant_bytes(const smy_moe_config* c, int64_t T, int v, size_t* bytes) {
  if (v < 0 || v > SMY_VARIANT_DENSE_INTER) return SMY_E_CONFIG;
  *bytes = variant_bytes(c, T, v);
  return SMY_OK;
}
smy_status moe_set_variant(int v, void* scratch, size_t bytes) {
  if (v < 0 || v > SMY_VARIANT_DENSE_INTER) return SMY_E_CONFIG;
  if (v != 0 && scratch == nullptr) return SMY_E_NULL;
  t_variant.v = v;
  t_variant.scratch = static_cast<uint8_t*>(scratch);
  t_variant.bytes = bytes;
  return SMY_OK;
}

// The expert computation over T rows of x.  Routing either comes from router
// logits (top-k on device) or is given as keys[T x k] (expert ids, -1 = none)
// with weights vals[T x k] -- the expert-parallel receive side.
smy_status moe_core(const smy_moe_config* c, const smy_weight* experts, const smy_weight* shared, const void* x,
                    const float* logits, const int32_t* keys, const float* vals, int64_t T, float* out,
                    void* workspace, size_t ws_bytes, cudaStream_t s, const PeerRows* peers) {
  const int d = c->hidden, f = c->ffn;
  // shared experts (weight 1, every token -- reading R15): with router logits
  // they are appended to every token's routing entries (route_launch), so the two
  // grouped launches run them as groups E_r .. E_r + ns - 1 (SEL = all tokens)
  const int nsh = (shared != nullptr && keys == nullptr && c->num_shared > 0) ? c->num_shared : 0;
  const int Er = c->num_experts, kr = c->top_k;
  const int E = Er + nsh, k = kr + nsh;
  // interleaved: experts[3e] is the [2f x d] gate/up weight (reading R20), experts[3e+1] unused
  const bool ilv = interleaved(c);
  smy_wdesc dgu{ilv ? 2 * f : f, d, c->fmt}, ddn{d, f, c->fmt};
  Geometry ggu, gdn;
  smy_status st;
  if ((st = geometry(&dgu, &ggu)) != SMY_OK) return st;
  if ((st = geometry(&ddn, &gdn)) != SMY_OK) return st;
  if (E > kMaxGroups) return SMY_E_CONFIG;
  const bool fused = ilv || gate_up_fused(ggu);
  const int nw_gu = ilv ? 1 : fused ? 2 : 1;
  LayerWs w = carve(c, T, !fused, static_cast<uint8_t*>(workspace));
  if (w.total > ws_bytes) return SMY_E_WORKSPACE;

  const int64_t tpg = Er ? (T * kr + Er - 1) / Er : 0;  // routed tokens per expert
  // tile width: the mean tokens per expert + 3 sigma of the (binomial) spread, so a
  // decode-sized expert rarely needs a second n-tile (which would re-stream its weights
  // through the SMs); ragged tiles issue MMAs of their own width
  const int64_t tpg_hi = tpg + (int64_t)(3.0 * sqrt((double)tpg) + 0.999);
  // (N, 2N, 32) formats, N > 1: one-weight launches run the in-smem row expansion
  const int xp_gu = nw_gu == 1 && xp_on(c->fmt) ? 1 : 0, xp_dn = xp_on(c->fmt) ? 1 : 0;
  int nt_gu = ssmm_pick_nt(nw_gu, ggu.ms, ggu.rep, tpg_hi, xp_gu);
  int nt_dn = ssmm_pick_nt(1, gdn.ms, gdn.rep, tpg_hi, xp_dn);
  const int64_t act = E < T * k ? E : T * k;
  const Variant var = t_variant;
  if (var.v != 0) {  // ablation variants: the single-GPU interleaved layer with router logits
    if (!ilv || keys != nullptr || peers != nullptr) return SMY_E_CONFIG;
    if (variant_bytes(c, T, var.v) > var.bytes) return SMY_E_WORKSPACE;
  }
  const smy_weight* wg[kMaxGroups];
  const smy_weight* wu[kMaxGroups];
  const smy_weight* wd[kMaxGroups];
  for (int e = 0; e < E; ++e) {
    const smy_weight* t3 = e < Er ? &experts[3 * e] : &shared[3 * (e - Er)];
    wg[e] = &t3[0];
    wu[e] = &t3[1];
    wd[e] = &t3[2];
  }
  const size_t img_gu = (size_t)ggu.m_tiles * ggu.k_stages * ggu.block;
  const size_t img_dn = (size_t)gdn.m_tiles * gdn.k_stages * gdn.block;
  const bool pair_gu_ok = ssmm_pair_images_ok(wg, nw_gu == 2 ? wu : nullptr, E, img_gu);
  const bool pair_dn_ok = ssmm_pair_images_ok(wd, nullptr, E, img_dn);
  const int cl_gu = fused && pair_gu_ok ? ssmm_pair_cluster(nt_gu, nw_gu, ggu.ms, ggu.rep, ggu.m_tiles, tpg, 1) : 0;
  const int mtp_gu = var.v == 0 ? gu_mtp_half(ilv, cl_gu, ggu, nt_gu) : 0;
  if (mtp_gu) nt_gu = SMY_MTP_NT;
  // N = M down weights with wide tiles: m-tile pairing on the CTA pair (the weight's
  // second half of m-tiles as the launch's second weight, samoyeds_ssmm): every token
  // stage of the intermediate feeds two accumulators
  const int mtp_dn = pair_dn_ok && var.v == 0 ? down_mtp_half(gdn, tpg, tpg_hi) : 0;
  if (mtp_dn) nt_dn = down_mtp_nt(gdn);
  const int mtiles_dn = mtp_dn ? mtp_dn : gdn.m_tiles;  // m-tiles per weight of the launch
  const int cl_dn =
      mtp_dn ? 2 : pair_dn_ok ? ssmm_pair_cluster(nt_dn, 1, gdn.ms, gdn.rep, gdn.m_tiles, tpg, 0) : 0;
  // expected down tiles -> K split (the scatter-add epilogue makes partial sums free);
  // the permute variant's down writes compact fp32 rows: no K split
  const int ks_dn = var.v == SMY_VARIANT_PERMUTE
                        ? 1
                        : ssmm_pick_ksplit((int64_t)mtiles_dn * act * ((tpg + nt_dn - 1) / (nt_dn > 0 ? nt_dn : 1)),
                                           gdn.k_stages);
  const int mtiles_gu = mtp_gu ? mtp_gu : ggu.m_tiles;
  const int mt_gu = cl_gu ? (mtiles_gu + 1) / 2 : mtiles_gu;
  const int mt_dn = cl_dn ? (mtiles_dn + 1) / 2 : mtiles_dn;
  // the routing scan counts tiles per expert in units of the launch's token span
  const int nts[2] = {nt_gu, nt_dn};
  const int mts[2] = {mt_gu, mt_dn * ks_dn};
  int32_t* prefix_gu = w.prefix;
  int32_t* prefix_dn = w.prefix + (E + 1);

  record_phase(0, s);
  if (keys == nullptr)
    st = route_launch(logits, T, Er, kr, c->gating, w.ids, w.w, w.counts, w.offsets, w.sel, w.gw, w.route_ws,
                      w.route_ws_bytes, nts, mts, 2, w.prefix, s, nsh);
  else
    st = compact_launch(keys, vals, T, E, k, w.counts, w.offsets, w.sel, w.gw, w.route_ws, w.route_ws_bytes, nts,
                        mts, 2, w.prefix, s);
  if (st != SMY_OK) return st;
  record_phase(1, s);
  // the output is zeroed by the gate/up launch (SsmmArgs::zero_ptr); in peer mode every
  // rank zeroed its own output before the exchange
  float* zero_out = peers == nullptr && T > 0 ? out : nullptr;
  record_phase(2, s);
  if (T == 0) {
    for (int i = 3; i < 6; ++i) record_phase(i, s);
    return SMY_OK;
  }

  const int64_t Tk = T * k;
  const int max_gu = mt_gu * (E + (int)((Tk + nts[0] - 1) / nts[0]));
  const int max_dn = mt_dn * (E + (int)((Tk + nts[1] - 1) / nts[1]));
  const uint16_t* xb = static_cast<const uint16_t*>(x);

  // gate/up: H = Wg x[SEL], U = Wu x[SEL], inter = bf16(silu(H) * U)
  uint16_t* xp = nullptr;       // SMY_VARIANT_PERMUTE: x[SEL], then y (fp32) after it
  float* yp = nullptr;
  uint16_t* inter_dense = nullptr;  // SMY_VARIANT_DENSE_INTER: [E x T x f], then the row map
  int32_t* rows_dense = nullptr;
  const int vblocks = 148 * 8;
  if (var.v == SMY_VARIANT_PERMUTE) {
    xp = reinterpret_cast<uint16_t*>(var.scratch);
    yp = reinterpret_cast<float*>(var.scratch + align_up((size_t)Tk * d * 2, 256));
    permute_rows_kernel<<<vblocks, 256, 0, s>>>(xb, d, w.sel, w.offsets, E, xp);
    count_launch();
    st = grouped(wg, nullptr, E, ggu, f, nt_gu, 1, xp, d, Tk, nullptr, w.offsets, prefix_gu, max_gu, kEpiSiluMulIlv,
                 w.inter, f, 1, nullptr, nullptr, d, tpg <= nt_gu, 1, cl_gu, s, nullptr, zero_out, T * d);
  } else if (var.v == SMY_VARIANT_DENSE_INTER) {
    inter_dense = reinterpret_cast<uint16_t*>(var.scratch);
    rows_dense = reinterpret_cast<int32_t*>(var.scratch + align_up((size_t)E * T * f * 2, 256));
    cudaMemsetAsync(inter_dense, 0, (size_t)E * T * f * 2, s);
    dense_rows_kernel<<<E, 256, 0, s>>>(w.sel, w.offsets, E, T, rows_dense);
    count_launch();
    st = grouped(wg, nullptr, E, ggu, f, nt_gu, 1, xb, d, T, w.sel, w.offsets, prefix_gu, max_gu, kEpiSiluMulIlv,
                 inter_dense, f, 1, nullptr, nullptr, d, tpg <= nt_gu, 1, cl_gu, s, nullptr, zero_out, T * d,
                 rows_dense);
  } else if (ilv) {
    st = grouped(wg, nullptr, E, ggu, f, nt_gu, mtp_gu ? 2 : 1, xb, peers ? peers->ldx : d, T, w.sel, w.offsets,
                 prefix_gu, max_gu, kEpiSiluMulIlv, w.inter, f, 1, nullptr, nullptr, d, tpg <= nt_gu, 1, cl_gu, s,
                 peers, zero_out, T * d, nullptr, mtp_gu);
  } else if (fused) {
    st = grouped(wg, wu, E, ggu, f, nt_gu, 2, xb, peers ? peers->ldx : d, T, w.sel, w.offsets, prefix_gu, max_gu,
                 kEpiSiluMul, w.inter, f, 1, nullptr, nullptr, d, tpg <= nt_gu, 1, cl_gu, s, peers, zero_out, T * d);
  } else {
    st = grouped(wg, nullptr, E, ggu, f, nt_gu, 1, xb, peers ? peers->ldx : d, T, w.sel, w.offsets, prefix_gu,
                 max_gu, kEpiCompact, w.fallback_g, f, 0, nullptr, nullptr, d, tpg <= nt_gu, 1, 0, s, peers, zero_out,
                 T * d);
    if (st == SMY_OK)
      st = grouped(wu, nullptr, E, ggu, f, nt_gu, 1, xb, peers ? peers->ldx : d, T, w.sel, w.offsets, prefix_gu,
                   max_gu, kEpiCompact, w.fallback_u, f, 0, nullptr, nullptr, d, tpg <= nt_gu, 1, 0, s, peers);
    if (st == SMY_OK) st = silu_mul_launch(w.fallback_g, w.fallback_u, Tk, f, w.inter, s);
  }
  if (st != SMY_OK) return st;
  record_phase(3, s);
  // down: out[sel[t]] += gw[t] * Wd inter[t]
  if (var.v == SMY_VARIANT_PERMUTE) {
    st = grouped(wd, nullptr, E, gdn, d, nt_dn, 1, w.inter, f, Tk, nullptr, w.offsets, prefix_dn, max_dn, kEpiCompact,
                 yp, d, 0, nullptr, nullptr, f, tpg <= nt_dn, 1, cl_dn, s);
    if (st == SMY_OK) {
      unpermute_rows_kernel<<<vblocks, 256, 0, s>>>(yp, d, w.sel, w.gw, w.offsets, E, out);
      count_launch();
      st = cuda_status(cudaGetLastError());
    }
  } else if (var.v == SMY_VARIANT_DENSE_INTER) {
    st = grouped(wd, nullptr, E, gdn, d, nt_dn, 1, inter_dense, f, (int64_t)E * T, rows_dense, w.offsets, prefix_dn,
                 max_dn, kEpiScatter, out, d, 0, w.sel, w.gw, f, tpg <= nt_dn, ks_dn, cl_dn, s);
  } else {
    st = grouped(wd, nullptr, E, gdn, d, nt_dn, mtp_dn ? 2 : 1, w.inter, f, Tk, nullptr, w.offsets, prefix_dn, max_dn,
                 kEpiScatter, out, peers ? peers->ldo : d, 0, w.sel, w.gw, f, tpg <= nt_dn, ks_dn, cl_dn, s, peers,
                 nullptr, 0, nullptr, mtp_dn, peers == nullptr && !(debug_flags() & 4194304));
  }
  if (st != SMY_OK) return st;
  record_phase(4, s);

  // shared experts: every token, weight 1 (reading R15)
  // (the expert-parallel receive side, whose routing arrives as keys, runs them here)
  for (int i = 0; shared && nsh == 0 && i < c->num_shared; ++i) {
    const smy_weight* sg[1] = {&shared[3 * i + 0]};
    const smy_weight* su[1] = {&shared[3 * i + 1]};
    const smy_weight* sd[1] = {&shared[3 * i + 2]};
    const int nts_gu = ssmm_pick_nt(nw_gu, ggu.ms, ggu.rep, T, xp_gu);
    const int nts_dn = ssmm_pick_nt(1, gdn.ms, gdn.rep, T, xp_dn);
    auto single = [&](const smy_weight* const* a0, const smy_weight* const* a1, const Geometry& g, int m_out, int nt,
                      int nw, const uint16_t* xx, int64_t ldx, int epi, void* o, int64_t ldo, int ob) {
      SsmmArgs a;
      memset(&a, 0, sizeof(a));
      a.img0[0] = static_cast<const uint8_t*>(a0[0]->image);
      a.img1[0] = a1 ? static_cast<const uint8_t*>(a1[0]->image) : nullptr;
      a.num_groups = 1;
      a.xp = nw == 1 && xp_on(c->fmt) ? 1 : 0;
      a.R = (int)g.R;
      a.m_out = m_out;
      a.n_fmt = g.ms == 1 ? 1 : c->fmt.n;
      a.m_fmt = g.ms == 1 ? 1 : c->fmt.m;
      a.m_tiles = g.m_tiles;
      a.k_stages = g.k_stages;
      a.planes = g.planes;
      a.block = g.block;
      a.x = xx;
      a.ldx = ldx;
      a.x_rows = T;
      a.n_sel = (int)T;
      a.epi = epi;
      a.out_bf16 = ob;
      a.out = o;
      a.ldo = ldo;
      a.max_tiles = g.m_tiles * (int)((T + nt - 1) / nt);
      a.weights_stream = T <= nt;
      a.k_splits = epi == kEpiScatter ? ssmm_pick_ksplit(a.max_tiles, g.k_stages) : 1;
      a.max_tiles *= a.k_splits;
      smy_status st2 = make_x_tmap(&a.tmap_x, xx, ldx, T, ldx, nt);
      if (st2 != SMY_OK) return st2;
      return ssmm_launch(a, nt, nw, g.ms, g.rep, s);
    };
    if (ilv) {
      st = single(sg, nullptr, ggu, f, nts_gu, 1, xb, d, kEpiSiluMulIlv, w.inter, f, 1);
    } else if (fused) {
      st = single(sg, su, ggu, f, nts_gu, 2, xb, d, kEpiSiluMul, w.inter, f, 1);
    } else {
      st = single(sg, nullptr, ggu, f, nts_gu, 1, xb, d, kEpiCompact, w.fallback_g, f, 0);
      if (st == SMY_OK) st = single(su, nullptr, ggu, f, nts_gu, 1, xb, d, kEpiCompact, w.fallback_u, f, 0);
      if (st == SMY_OK) st = silu_mul_launch(w.fallback_g, w.fallback_u, T, f, w.inter, s);
    }
    if (st != SMY_OK) return st;
    st = single(sd, nullptr, gdn, d, nts_dn, 1, w.inter, f, kEpiScatter, out, d, 0);
    if (st != SMY_OK) return st;
  }
  record_phase(5, s);
  return SMY_OK;
}

// The SSMM kernels a single-GPU layer call over T tokens launches (the same
// tile-width / CTA-pair decisions as moe_core, weight images in one block as
// prepare_experts lays them out): names as the profiler prints them.
smy_status moe_kernel_names(const smy_moe_config* c, int64_t T, char* gu, char* dn, int len) {
  const bool ilv = interleaved(c);
  smy_wdesc dgu{ilv ? 2 * c->ffn : c->ffn, c->hidden, c->fmt}, ddn{c->hidden, c->ffn, c->fmt};
  Geometry ggu, gdn;
  smy_status st;
  if ((st = geometry(&dgu, &ggu)) != SMY_OK) return st;
  if ((st = geometry(&ddn, &gdn)) != SMY_OK) return st;
  const bool fused = ilv || gate_up_fused(ggu);
  const int nw_gu = ilv ? 1 : fused ? 2 : 1;
  const int Er = c->num_experts, kr = c->top_k;
  const int64_t tpg = Er ? (T * kr + Er - 1) / Er : 0;
  const int64_t tpg_hi = tpg + (int64_t)(3.0 * sqrt((double)tpg) + 0.999);
  const int xp_gu = nw_gu == 1 && xp_on(c->fmt) ? 1 : 0, xp_dn = xp_on(c->fmt) ? 1 : 0;
  const int nt_gu = ssmm_pick_nt(nw_gu, ggu.ms, ggu.rep, tpg_hi, xp_gu);
  const int nt_dn = ssmm_pick_nt(1, gdn.ms, gdn.rep, tpg_hi, xp_dn);
  const int cl_gu = fused ? ssmm_pair_cluster(nt_gu, nw_gu, ggu.ms, ggu.rep, ggu.m_tiles, tpg, 1) : 0;
  const int mtp_dn = down_mtp_half(gdn, tpg, tpg_hi);
  const int cl_dn = mtp_dn ? 2 : ssmm_pair_cluster(nt_dn, 1, gdn.ms, gdn.rep, gdn.m_tiles, tpg, 0);
  // the SEL-gather pair launch of the widest (1,2,V) tile runs split rings (ssmm.cu)
  const int split_gu =
      cl_gu && ((ggu.ms == 2 && nw_gu == 1 && (nt_gu == SMY_NT_WIDE || nt_gu == 128) && !(debug_flags() & 16384)) ||
                (ggu.ms == 1 && nw_gu == 2 && nt_gu == 224));
  const int mtp_gu = gu_mtp_half(ilv, cl_gu, ggu, nt_gu);
  if (mtp_gu)
    snprintf(gu, len, "ssmm_pair_kernel<%d, 2, 2, 1>", SMY_MTP_NT);
  else if (cl_gu)
    snprintf(gu, len, "ssmm_pair_kernel<%d, %d, %d, %d>", nt_gu, nw_gu, ggu.ms, split_gu);
  else if (xp_gu)
    snprintf(gu, len, "ssmm_kernel<%d, 1, 2, 1, 1>", nt_gu);
  else
    snprintf(gu, len, "ssmm_kernel<%d, %d, %d, %d>", nt_gu, nw_gu, ggu.ms, ggu.rep);
  if (mtp_dn && gdn.ms == 1)
    snprintf(dn, len, "ssmm_pair_kernel<224, 2, 1, 1>");
  else if (mtp_dn)
    snprintf(dn, len, "ssmm_pair_kernel<112, 2, 2, 0>");
  else if (cl_dn)
    snprintf(dn, len, "ssmm_pair_kernel<%d, %d, %d, %d>", nt_dn, 1, gdn.ms, 0);
  else if (xp_dn)
    snprintf(dn, len, "ssmm_kernel<%d, 1, 2, 1, 1>", nt_dn);
  else
    snprintf(dn, len, "ssmm_kernel<%d, %d, %d, %d>", nt_dn, 1, gdn.ms, gdn.rep);
  return SMY_OK;
}

smy_status moe_view(const smy_moe_config* c, int64_t T, void* workspace, size_t ws_bytes, smy_moe_view* v) {
  smy_wdesc dgu{interleaved(c) ? 2 * c->ffn : c->ffn, c->hidden, c->fmt};
  Geometry ggu;
  smy_status st = geometry(&dgu, &ggu);
  if (st != SMY_OK) return st;
  const bool fused = interleaved(c) || gate_up_fused(ggu);
  LayerWs w = carve(c, T, !fused, static_cast<uint8_t*>(workspace));
  if (w.total > ws_bytes) return SMY_E_WORKSPACE;
  const int ns = c->num_shared > 0 ? c->num_shared : 0;
  v->counts = w.counts;
  v->offsets = w.offsets;
  v->sel = w.sel;
  v->gw = w.gw;
  v->inter = w.inter;
  v->inter_rows = T * (c->top_k + ns) > T ? T * (c->top_k + ns) : T;
  v->groups = c->num_experts + ns;
  return SMY_OK;
}

smy_status moe_layer(const smy_moe_config* c, const smy_weight* experts, const smy_weight* shared, const void* x,
                     const float* logits, int64_t T, void* out, void* workspace, size_t ws_bytes, cudaStream_t s) {
  if (c->out_dtype != SMY_BF16)
    return moe_core(c, experts, shared, x, logits, nullptr, nullptr, T, static_cast<float*>(out), workspace, ws_bytes,
                    s);
  // bf16 output: accumulate in fp32 at the end of the workspace, round once
  smy_moe_config cf = *c;
  cf.out_dtype = SMY_F32;
  size_t core = 0;
  smy_status st = moe_workspace_bytes(&cf, T, &core);
  if (st != SMY_OK) return st;
  core = align_up(core, 256);
  const size_t acc_bytes = (size_t)T * c->hidden * 4;
  if (core + acc_bytes > ws_bytes) return SMY_E_WORKSPACE;
  float* acc = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + core);
  st = moe_core(&cf, experts, shared, x, logits, nullptr, nullptr, T, acc, workspace, core, s);
  if (st != SMY_OK || T == 0) return st;
  const int64_t n4 = T * c->hidden / 4;
  int blocks = (int)((n4 + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  f32_to_bf16_kernel<<<blocks, 256, 0, s>>>(reinterpret_cast<const float4*>(acc), n4, static_cast<uint2*>(out));
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
