// C ABI entry points (include/samoyeds.h): host-side validation + dispatch.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <string>

#include "internal.h"

namespace smy {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};
static thread_local cudaEvent_t g_phase[6];
static thread_local bool g_phase_on = false;

int debug_flags() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SMY_DEBUG");
    v = e ? atoi(e) : 0;
  }
  return v;
}

static unsigned long long* g_prof = nullptr;
static int g_prof_ctas = 0;
unsigned long long* debug_prof_buffer(int ctas) {
  if (ctas > g_prof_ctas) {
    if (g_prof) cudaFree(g_prof);
    cudaMalloc(&g_prof, sizeof(unsigned long long) * 32 * ctas);
    cudaMemset(g_prof, 0, sizeof(unsigned long long) * 32 * ctas);
    g_prof_ctas = ctas;
  }
  return g_prof;
}

void count_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
void record_phase(int i, cudaStream_t s) {
  if (!g_phase_on || i < 0 || i >= 6) return;
  // inside a stream capture the record must become an event-record NODE of the
  // graph (external), so every replay timestamps it
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(g_phase[i], s, cudaEventRecordExternal);
  else
    cudaEventRecord(g_phase[i], s);
}

void set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }

smy_status cuda_status(cudaError_t e) {
  if (e != cudaSuccess) cudaGetLastError();
  if (e == cudaSuccess) return SMY_OK;
  g_last_error = cudaGetErrorString(e);
  return SMY_E_CUDA;
}

smy_status check_arch() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return SMY_E_CUDA;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    cached = (major == 10 && minor == 0) ? 1 : 0;
  }
  if (!cached) {
    set_last_error("samoyeds requires an sm_100 (B200) device");
    return SMY_E_ARCH;
  }
  return SMY_OK;
}

static bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

smy_status geometry(const smy_wdesc* d, Geometry* g) {
  if (!d || !g) return SMY_E_NULL;
  const smy_format f = d->fmt;
  if (f.n < 1 || f.n > f.m || f.v <= 0 || f.v % 4) {
    set_last_error("format: need 1 <= N <= M and V a multiple of 4");
    return SMY_E_CONFIG;
  }
  if (!(f.m == 1 || f.m == 2 || f.m == 4 || f.m == 8 || f.m == 16) || !is_pow2(f.n)) {
    set_last_error("format: GPU path supports M in {1,2,4,8,16}, N a power of two");
    return SMY_E_CONFIG;
  }
  if (!(f.v % 32 == 0 || (f.v == 16 && f.n == 1 && f.m == 2))) {
    set_last_error("format: V must be a multiple of 32, or V=16 with (N,M)=(1,2)");
    return SMY_E_CONFIG;
  }
  if (d->rows <= 0 || d->cols <= 0 || d->rows % f.m || d->cols % f.v || d->cols % 128) {
    set_last_error("shape: need rows % M == 0, cols % V == 0 and cols % 128 == 0");
    return SMY_E_SHAPE;
  }
  g->R = d->rows * f.n / f.m;
  g->rep = f.v == 16 ? 2 : 1;
  g->m_tiles = (int)((g->R + kTileM - 1) / kTileM);
  g->k_stages = (int)(d->cols * g->rep / kStageVK);
  g->ms = (f.n == f.m) ? 1 : f.m;
  g->planes = g->ms == 1 ? 0 : (f.m == 2 ? 1 : f.m == 4 ? 2 : f.m == 8 ? 3 : 4);
  g->block = (kABytes + kEBytes + 64 * g->planes + 255) / 256 * 256;
  return SMY_OK;
}

smy_status synth_launch(uint64_t seed, int dist, float scale, int lo, int hi, int64_t idx0, int64_t n, void* out,
                        int out_bf16, cudaStream_t s);
smy_status moe_workspace_bytes(const smy_moe_config* c, int64_t T, size_t* bytes);
smy_status moe_layer(const smy_moe_config* c, const smy_weight* experts, const smy_weight* shared, const void* x,
                     const float* logits, int64_t T, void* out, void* workspace, size_t ws_bytes, cudaStream_t s);
smy_status moe_view(const smy_moe_config* c, int64_t T, void* workspace, size_t ws_bytes, smy_moe_view* v);
smy_status moe_kernel_names(const smy_moe_config* c, int64_t T, char* gu, char* dn, int len);

}  // namespace smy

using namespace smy;

static smy_status check_experts(const smy_moe_config* cfg, const smy_weight* experts, int n) {
  if (cfg->gate_up != SMY_GU_SEPARATE && cfg->gate_up != SMY_GU_INTERLEAVED) return SMY_E_CONFIG;
  const bool ilv = cfg->gate_up == SMY_GU_INTERLEAVED;
  if (ilv && !ilv_format(cfg->fmt)) {
    set_last_error("SMY_GU_INTERLEAVED needs format (1,2,V), (N,2N,V) or N == M, with V % 32 == 0");
    return SMY_E_CONFIG;
  }
  for (int e = 0; e < n; ++e)
    for (int i = 0; i < 3; ++i) {
      if (ilv && i == 1) continue;  // unused slot
      const smy_weight& w = experts[3 * e + i];
      const int64_t rows = i < 2 ? (ilv ? 2 * (int64_t)cfg->ffn : cfg->ffn) : cfg->hidden;
      const int64_t cols = i < 2 ? cfg->hidden : cfg->ffn;
      if (!w.image) return SMY_E_NULL;
      if (w.d.rows != rows || w.d.cols != cols || memcmp(&w.d.fmt, &cfg->fmt, sizeof(smy_format)) != 0)
        return SMY_E_SHAPE;
    }
  return SMY_OK;
}

extern "C" {

const char* smy_status_str(int s) {
  switch (s) {
    case SMY_OK: return "SMY_OK";
    case SMY_E_NULL: return "SMY_E_NULL";
    case SMY_E_SHAPE: return "SMY_E_SHAPE";
    case SMY_E_CONFIG: return "SMY_E_CONFIG";
    case SMY_E_PATTERN: return "SMY_E_PATTERN";
    case SMY_E_SELECTION: return "SMY_E_SELECTION";
    case SMY_E_CORRUPT: return "SMY_E_CORRUPT";
    case SMY_E_WORKSPACE: return "SMY_E_WORKSPACE";
    case SMY_E_ARCH: return "SMY_E_ARCH";
    case SMY_E_CUDA: return "SMY_E_CUDA";
    case SMY_E_NCCL: return "SMY_E_NCCL";
    default: return "SMY_E_UNKNOWN";
  }
}

int smy_version(void) { return 1; }

const char* smy_last_error(void) { return g_last_error.c_str(); }

smy_status smy_weight_layout(const smy_wdesc* d, smy_wlayout* out) {
  if (!d || !out) return SMY_E_NULL;
  Geometry g;
  smy_status st = geometry(d, &g);
  if (st != SMY_OK) return st;
  out->values = (size_t)g.R * (d->cols / 2) * 2;
  out->codes = (size_t)g.R * (d->cols / 8);
  out->indices = (size_t)g.R * (d->cols / d->fmt.v);
  out->image = (size_t)g.m_tiles * g.k_stages * g.block;
  out->comp_rows = (int32_t)g.R;
  out->m_tiles = g.m_tiles;
  out->k_stages = g.k_stages;
  out->planes = g.planes;
  out->rep = g.rep;
  out->block = g.block;
  return SMY_OK;
}

smy_status samoyeds_compress(const smy_wdesc* desc, const void* w_bf16, int64_t ldw, int flags, smy_weight* out,
                             int32_t* d_status, void* stream) {
  if (!desc || !w_bf16 || !out || !out->values || !out->codes || !out->indices || !out->image) return SMY_E_NULL;
  Geometry g;
  smy_status st = geometry(desc, &g);
  if (st != SMY_OK) return st;
  if (ldw < desc->cols) return SMY_E_SHAPE;
  if ((flags & (SMY_PRUNE_MAGNITUDE | SMY_ASSUME_PRUNED)) == (SMY_PRUNE_MAGNITUDE | SMY_ASSUME_PRUNED))
    return SMY_E_CONFIG;
  if ((st = check_arch()) != SMY_OK) return st;
  out->d = *desc;
  return compress_launch(desc, g, static_cast<const uint16_t*>(w_bf16), ldw, flags, out, d_status,
                         static_cast<cudaStream_t>(stream));
}

smy_status samoyeds_decompress(const smy_weight* w, void* w_bf16, int64_t ldw, int32_t* d_status, void* stream) {
  if (!w || !w_bf16 || !w->values || !w->codes || !w->indices) return SMY_E_NULL;
  Geometry g;
  smy_status st = geometry(&w->d, &g);
  if (st != SMY_OK) return st;
  if (ldw < w->d.cols) return SMY_E_SHAPE;
  if ((st = check_arch()) != SMY_OK) return st;
  return decompress_launch(w, static_cast<uint16_t*>(w_bf16), ldw, d_status, static_cast<cudaStream_t>(stream));
}

smy_status samoyeds_validate_sel(const int32_t* sel, int32_t n_sel, int64_t x_rows, int32_t* d_status, void* stream) {
  if ((n_sel > 0 && !sel) || !d_status) return SMY_E_NULL;
  if (n_sel < 0 || x_rows < 0) return SMY_E_SHAPE;
  smy_status st;
  if ((st = check_arch()) != SMY_OK) return st;
  return sel_check_launch(sel, n_sel, x_rows, d_status, static_cast<cudaStream_t>(stream));
}

smy_status samoyeds_interleave_gate_up(const smy_weight* gate, const smy_weight* up, smy_weight* gu, void* stream) {
  if (!gate || !up || !gu) return SMY_E_NULL;
  if (!gate->values || !gate->codes || !gate->indices || !up->values || !up->codes || !up->indices || !gu->values ||
      !gu->codes || !gu->indices || !gu->image)
    return SMY_E_NULL;
  if (memcmp(&gate->d, &up->d, sizeof(smy_wdesc)) != 0 || gate->d.rows % 32) return SMY_E_SHAPE;
  // the kernel moves blocks of 16 compressed rows (reading R20): R = rows*N/M % 16 == 0
  if ((gate->d.rows * gate->d.fmt.n / gate->d.fmt.m) % 16) {
    set_last_error("interleave_gate_up needs rows * N / M % 16 == 0 (blocks of 16 compressed rows)");
    return SMY_E_SHAPE;
  }
  smy_wdesc d = gate->d;
  d.rows *= 2;
  Geometry g;
  smy_status st = geometry(&d, &g);
  if (st != SMY_OK) return st;
  if ((st = check_arch()) != SMY_OK) return st;
  gu->d = d;
  return interleave_launch(gate, up, d, g, gu, static_cast<cudaStream_t>(stream));
}

smy_status samoyeds_ssmm(const smy_weight* w, const smy_weight* w2, const void* x_bf16, int64_t ldx, int64_t x_rows,
                         const int32_t* sel, int32_t n_sel, const float* scale, int epi, void* out, int64_t ldo,
                         int out_dtype, void* stream) {
  if (!w || !w->image || (n_sel > 0 && (!sel || !x_bf16 || !out))) return SMY_E_NULL;
  Geometry g;
  smy_status st = geometry(&w->d, &g);
  if (st != SMY_OK) return st;
  if (n_sel < 0) return SMY_E_SELECTION;
  if (ldx < w->d.cols || ldx % 8 || x_rows < 0) return SMY_E_SHAPE;
  if (epi == SMY_EPI_SILU_MUL_COMPACT) {
    if (!w2 || !w2->image) return SMY_E_NULL;
    if (memcmp(&w2->d, &w->d, sizeof(smy_wdesc)) != 0) return SMY_E_SHAPE;
    if (out_dtype != SMY_BF16) return SMY_E_CONFIG;
    if (g.ms >= 16) {
      set_last_error("SILU_MUL fusion unsupported for M=16 (use two COMPACT calls)");
      return SMY_E_CONFIG;
    }
  } else if (epi == SMY_EPI_SILU_MUL_INTERLEAVED) {
    if (out_dtype != SMY_BF16) return SMY_E_CONFIG;
    if (!ilv_format(w->d.fmt)) {
      set_last_error("SILU_MUL_INTERLEAVED needs format (1,2,V), (N,2N,V) or N == M, with V % 32 == 0");
      return SMY_E_CONFIG;
    }
    if (w->d.rows % 64) return SMY_E_SHAPE;
  } else if (epi == SMY_EPI_SCATTER_ADD) {
    if (out_dtype != SMY_F32) return SMY_E_CONFIG;
  } else if (epi != SMY_EPI_COMPACT) {
    return SMY_E_CONFIG;
  }
  if (out_dtype != SMY_F32 && out_dtype != SMY_BF16) return SMY_E_CONFIG;
  const int64_t out_cols = epi == SMY_EPI_SILU_MUL_INTERLEAVED ? w->d.rows / 2 : w->d.rows;
  if (ldo < out_cols || (ldo % 2)) return SMY_E_SHAPE;
  // the scatter epilogue reduces 16 B (4 fp32 outputs) per lane pair
  const bool v4_ok = ldo % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && w->d.rows % 4 == 0;
  if (epi == SMY_EPI_SCATTER_ADD && !v4_ok) {
    set_last_error("SCATTER_ADD needs ldo % 4 == 0, a 16-byte aligned out and rows % 4 == 0");
    return SMY_E_SHAPE;
  }
  if ((st = check_arch()) != SMY_OK) return st;
  if (n_sel == 0) return SMY_OK;
  if (debug_flags() & kDebugValidate) {  // debug builds of a caller: check SEL, synchronously
    int32_t* d_st = nullptr;
    int32_t h_st = SMY_OK;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    if (cudaMallocAsync(reinterpret_cast<void**>(&d_st), 4, cs) != cudaSuccess) return cuda_status(cudaGetLastError());
    cudaMemsetAsync(d_st, 0, 4, cs);
    st = sel_check_launch(sel, n_sel, x_rows, d_st, cs);
    cudaMemcpyAsync(&h_st, d_st, 4, cudaMemcpyDeviceToHost, cs);
    cudaFreeAsync(d_st, cs);
    cudaError_t ce = cudaStreamSynchronize(cs);
    if (st != SMY_OK) return st;
    if (ce != cudaSuccess) return cuda_status(ce);
    if (h_st != SMY_OK) {
      set_last_error("sel: entries must be strictly increasing and in [0, x_rows)");
      return SMY_E_SELECTION;
    }
  }
  const int nw = epi == SMY_EPI_SILU_MUL_COMPACT ? 2 : 1;
  const int xp = nw == 1 && xp_on(w->d.fmt) ? 1 : 0;  // (N, 2N, 32): in-smem row expansion
  const int nt = ssmm_pick_nt(nw, g.ms, g.rep, n_sel, xp);
  SsmmArgs a;
  memset(&a, 0, sizeof(a));
  a.xp = xp;
  a.img0[0] = static_cast<const uint8_t*>(w->image);
  a.img1[0] = nw == 2 ? static_cast<const uint8_t*>(w2->image) : nullptr;
  a.num_groups = 1;
  a.R = (int)g.R;
  a.m_out = (int)w->d.rows;
  a.n_fmt = g.ms == 1 ? 1 : w->d.fmt.n;
  a.m_fmt = g.ms == 1 ? 1 : w->d.fmt.m;
  a.m_tiles = g.m_tiles;
  a.k_stages = g.k_stages;
  a.planes = g.planes;
  a.block = g.block;
  a.x = static_cast<const uint16_t*>(x_bf16);
  a.ldx = ldx;
  a.x_rows = x_rows;
  a.sel_in = sel;
  a.offsets = nullptr;
  a.tile_prefix = nullptr;
  a.n_sel = n_sel;
  a.epi = epi == SMY_EPI_COMPACT               ? kEpiCompact
          : epi == SMY_EPI_SILU_MUL_COMPACT    ? kEpiSiluMul
          : epi == SMY_EPI_SILU_MUL_INTERLEAVED ? kEpiSiluMulIlv
                                               : kEpiScatter;
  a.out_bf16 = out_dtype == SMY_BF16;
  a.out = out;
  a.ldo = ldo;
  a.sel_out = sel;
  a.scale = scale;
  a.weights_stream = n_sel <= nt;
  // Too few tiles to fill the GPU with an fp32 COMPACT output (small M, long K): zero the
  // output and run it as a scatter-add into rows 0..n_sel-1 -- K is then split over the
  // SMs (split-K / stream-K tail) and the partial sums add.
  {
    const int64_t tiles = (int64_t)g.m_tiles * ((n_sel + nt - 1) / nt);
    if (a.epi == kEpiCompact && !a.out_bf16 && tiles < 74 && g.k_stages >= 16 && v4_ok) {
      cudaError_t ce = cudaMemset2DAsync(out, (size_t)ldo * 4, 0, (size_t)w->d.rows * 4, (size_t)n_sel,
                                         static_cast<cudaStream_t>(stream));
      if (ce != cudaSuccess) return cuda_status(ce);
      a.epi = kEpiScatter;
      a.sel_out = nullptr;  // destination row = compact row
      a.scale = nullptr;
    }
  }
  // N = M weight, > 128 tokens: m-tile pairing on the CTA pair -- the weight's second half
  // of m-tiles runs as a second "weight" of the same launch, so every SEL-gathered token
  // stage feeds two accumulators (half the gather bytes per MMA of the one-slot kernel)
  if (nw == 1 && g.ms == 1 && g.rep == 1 && g.m_tiles >= 2 && !(debug_flags() & 131072)) {
    const int nt2 = ssmm_pick_nt(2, 1, 1, n_sel);
    const int half = (g.m_tiles + 1) / 2;
    const smy_weight* w0a[1] = {w};
    const size_t img = (size_t)g.m_tiles * g.k_stages * g.block;
    if (nt2 == 224 && ssmm_pair_images_ok(w0a, nullptr, 1, img) &&
        ssmm_pair_cluster(nt2, 2, 1, 1, half, n_sel, 1) == 2) {
      a.img1[0] = a.img0[0] + (size_t)half * g.k_stages * g.block;
      a.m_tiles = half;
      a.mtp_half = half;
      a.max_tiles = ((half + 1) / 2) * ((n_sel + nt2 - 1) / nt2);
      a.k_splits = 1;
      if ((st = make_x_tmap(&a.tmap_x, x_bf16, w->d.cols, x_rows, ldx, nt2 / 2)) != SMY_OK) return st;
      return ssmm_launch_pair(a, nt2, 2, 1, 2, static_cast<cudaStream_t>(stream));
    }
  }
  // >= 64 tokens of a (1,2,V) weight: CTA-pair tiles (M = 256, cta_group::2), as in the layer
  const smy_weight* w0a[1] = {w};
  const smy_weight* w1a[1] = {nw == 2 ? w2 : nullptr};
  const size_t img = (size_t)g.m_tiles * g.k_stages * g.block;
  const int cl = ssmm_pair_images_ok(w0a, nw == 2 ? w1a : nullptr, 1, img)
                     ? ssmm_pair_cluster(nt, nw, g.ms, g.rep, g.m_tiles, n_sel, 1)
                     : 0;
  if (cl) {
    a.max_tiles = ((g.m_tiles + 1) / 2) * ((n_sel + nt - 1) / nt);
    a.k_splits = 1;  // scatter-add balance comes from the stream-K tail
    if ((st = make_x_tmap(&a.tmap_x, x_bf16, w->d.cols, x_rows, ldx, nt / 2)) != SMY_OK) return st;
    return ssmm_launch_pair(a, nt, nw, g.ms, cl, static_cast<cudaStream_t>(stream));
  }
  a.max_tiles = g.m_tiles * ((n_sel + nt - 1) / nt);
  a.k_splits = a.epi == kEpiScatter ? ssmm_pick_ksplit(a.max_tiles, g.k_stages) : 1;
  a.max_tiles *= a.k_splits;
  if ((st = make_x_tmap(&a.tmap_x, x_bf16, w->d.cols, x_rows, ldx, nt)) != SMY_OK) return st;
  return ssmm_launch(a, nt, nw, g.ms, g.rep, static_cast<cudaStream_t>(stream));
}

smy_status smy_route_workspace_bytes(int64_t T, int32_t E, size_t* bytes) {
  if (!bytes) return SMY_E_NULL;
  if (T < 0 || E < 1) return SMY_E_SHAPE;
  *bytes = route_ws_bytes(T, E);
  return SMY_OK;
}

smy_status samoyeds_route(const float* logits, int64_t T, int32_t E, int32_t k, int gating, int32_t* ids, float* w,
                          int32_t* counts, int32_t* offsets, int32_t* sel, float* gw, void* workspace,
                          size_t ws_bytes, void* stream) {
  if (!counts || !offsets || !workspace) return SMY_E_NULL;
  if (T > 0 && (!logits || !ids || !w || !sel || !gw)) return SMY_E_NULL;
  if (T < 0 || E < 1 || k < 1 || k > E) return SMY_E_SHAPE;
  if (gating != SMY_GATE_RENORM_TOPK && gating != SMY_GATE_SOFTMAX_ALL) return SMY_E_CONFIG;
  smy_status st;
  if ((st = check_arch()) != SMY_OK) return st;
  return route_launch(logits, T, E, k, gating, ids, w, counts, offsets, sel, gw, workspace, ws_bytes, nullptr,
                      nullptr, 0, nullptr, static_cast<cudaStream_t>(stream));
}

smy_status smy_moe_workspace_bytes(const smy_moe_config* cfg, int64_t max_tokens, size_t* bytes) {
  if (!cfg || !bytes) return SMY_E_NULL;
  if (max_tokens < 0) return SMY_E_SHAPE;
  return moe_workspace_bytes(cfg, max_tokens, bytes);
}

smy_status samoyeds_moe_layer(const smy_moe_config* cfg, const smy_weight* experts, const smy_weight* shared,
                              const void* x_bf16, const float* logits, int64_t T, void* out, void* workspace,
                              size_t ws_bytes, smy_ep_comm* comm, void* stream) {
  if (!cfg || !experts || !out || !workspace) return SMY_E_NULL;
  if (T > 0 && (!x_bf16 || !logits)) return SMY_E_NULL;
  if (cfg->num_experts < 1 || cfg->top_k < 1 || cfg->top_k > cfg->num_experts || cfg->top_k > 8 ||
      cfg->num_experts > kMaxGroups || cfg->num_shared < 0 || (cfg->num_shared > 0 && !shared))
    return SMY_E_CONFIG;
  // shared experts run as extra groups with extra routing entries per token
  if (cfg->num_experts + cfg->num_shared > kMaxGroups || cfg->top_k + cfg->num_shared > 16) return SMY_E_CONFIG;
  {
    const int base = cfg->gating & ~SMY_GATE_SHARED_SIGMOID;
    if (base != SMY_GATE_RENORM_TOPK && base != SMY_GATE_SOFTMAX_ALL) return SMY_E_CONFIG;
    if ((cfg->gating & SMY_GATE_SHARED_SIGMOID) && (cfg->num_shared < 1 || comm != nullptr)) return SMY_E_CONFIG;
  }
  if (cfg->out_dtype != SMY_F32 && cfg->out_dtype != SMY_BF16) return SMY_E_CONFIG;
  if (cfg->out_dtype == SMY_BF16 && comm != nullptr) return SMY_E_CONFIG;
  if (cfg->hidden % 128 || cfg->ffn % 128) return SMY_E_SHAPE;
  if (reinterpret_cast<uintptr_t>(out) & 15) return SMY_E_SHAPE;  // 16-B scatter reductions
  smy_status st;
  if (comm != nullptr) {  // expert parallelism: experts = this rank's E / world (NCCL transport)
    const int W = ep_comm_world(comm);
    if (cfg->num_experts % W || cfg->num_shared != 0) return SMY_E_CONFIG;
    smy_moe_config lc = *cfg;
    lc.num_experts = cfg->num_experts / W;
    if ((st = check_experts(&lc, experts, lc.num_experts)) != SMY_OK) return st;
    if ((st = check_arch()) != SMY_OK) return st;
    return ep_layer(cfg, experts, x_bf16, logits, T, static_cast<float*>(out), workspace, ws_bytes, comm,
                    static_cast<cudaStream_t>(stream));
  }
  if ((st = check_experts(cfg, experts, cfg->num_experts)) != SMY_OK) return st;
  if (cfg->num_shared > 0 && (st = check_experts(cfg, shared, cfg->num_shared)) != SMY_OK) return st;
  if ((st = check_arch()) != SMY_OK) return st;
  return moe_layer(cfg, experts, shared, x_bf16, logits, T, out, workspace, ws_bytes,
                   static_cast<cudaStream_t>(stream));
}


smy_status smy_moe_kernel_names(const smy_moe_config* cfg, int64_t T, char* gate_up, char* down, int32_t len) {
  if (!cfg || !gate_up || !down) return SMY_E_NULL;
  if (T < 0 || len < 48) return SMY_E_SHAPE;
  if (cfg->num_experts < 1 || cfg->top_k < 1) return SMY_E_CONFIG;
  return moe_kernel_names(cfg, T, gate_up, down, len);
}

smy_status smy_moe_workspace_view(const smy_moe_config* cfg, int64_t T, void* workspace, size_t ws_bytes,
                                  smy_moe_view* view) {
  if (!cfg || !workspace || !view) return SMY_E_NULL;
  if (T < 0) return SMY_E_SHAPE;
  if (cfg->num_experts < 1 || cfg->top_k < 1 || cfg->num_shared < 0) return SMY_E_CONFIG;
  return moe_view(cfg, T, workspace, ws_bytes, view);
}

smy_status smy_ep_plan_workspace_bytes(int64_t T, int32_t k, int32_t world, size_t* bytes) {
  if (!bytes) return SMY_E_NULL;
  if (T < 0 || k < 1 || k > 8 || world < 1 || world > 256) return SMY_E_SHAPE;
  *bytes = ep_plan_ws_bytes(T, world, k);
  return SMY_OK;
}

smy_status samoyeds_ep_plan(const int32_t* ids, const float* w, int64_t T, int32_t k, int32_t num_experts,
                            int32_t world, int32_t* send_counts, int32_t* send_offsets, int32_t* send_sel,
                            int32_t* tag_ids, float* tag_w, void* workspace, size_t ws_bytes, void* stream) {
  if (!send_counts || !send_offsets || !workspace) return SMY_E_NULL;
  if (T > 0 && (!ids || !w || !send_sel || !tag_ids || !tag_w)) return SMY_E_NULL;
  if (T < 0 || k < 1 || k > 8 || world < 1 || world > 256 || num_experts % world) return SMY_E_SHAPE;
  smy_status st;
  if ((st = check_arch()) != SMY_OK) return st;
  return ep_plan_launch(ids, w, T, k, num_experts, world, send_counts, send_offsets, send_sel, tag_ids, tag_w,
                        workspace, ws_bytes, static_cast<cudaStream_t>(stream));
}

smy_status samoyeds_ep_pack(const void* x_bf16, int64_t ldx, int64_t hidden, const int32_t* send_offsets,
                            int32_t world, const int32_t* send_sel, int64_t max_rows, void* x_send, void* stream) {
  if (max_rows > 0 && (!x_bf16 || !send_offsets || !send_sel || !x_send)) return SMY_E_NULL;
  if (hidden % 8 || ldx < hidden || ldx % 8 || world < 1) return SMY_E_SHAPE;
  smy_status st;
  if ((st = check_arch()) != SMY_OK) return st;
  return ep_pack_launch(static_cast<const uint16_t*>(x_bf16), ldx, hidden, send_offsets, world, send_sel, max_rows,
                        static_cast<uint16_t*>(x_send), static_cast<cudaStream_t>(stream));
}

smy_status samoyeds_moe_experts(const smy_moe_config* cfg, const smy_weight* experts, const void* x_bf16,
                                int64_t rows, const int32_t* keys, const float* vals, float* out, void* workspace,
                                size_t ws_bytes, void* stream) {
  if (!cfg || !experts || !out || !workspace) return SMY_E_NULL;
  if (rows > 0 && (!x_bf16 || !keys || !vals)) return SMY_E_NULL;
  if (cfg->num_experts < 1 || cfg->top_k < 1 || cfg->top_k > 8 || cfg->num_experts > kMaxGroups ||
      cfg->num_shared != 0 || cfg->out_dtype != SMY_F32)
    return SMY_E_CONFIG;
  if (cfg->hidden % 128 || cfg->ffn % 128 || rows < 0 || (reinterpret_cast<uintptr_t>(out) & 15)) return SMY_E_SHAPE;
  smy_status st;
  if ((st = check_experts(cfg, experts, cfg->num_experts)) != SMY_OK) return st;
  if ((st = check_arch()) != SMY_OK) return st;
  return moe_core(cfg, experts, nullptr, x_bf16, nullptr, keys, vals, rows, out, workspace, ws_bytes,
                  static_cast<cudaStream_t>(stream));
}

smy_status smy_ep_unique_id(void* id128) {
  if (!id128) return SMY_E_NULL;
  return ep_unique_id(id128);
}

smy_status smy_ep_comm_create(const void* id128, int32_t rank, int32_t world, smy_ep_comm** comm) {
  if (!id128 || !comm) return SMY_E_NULL;
  if (world < 1 || world > 256 || rank < 0 || rank >= world) return SMY_E_SHAPE;
  return ep_comm_create(id128, rank, world, comm);
}

smy_status smy_ep_comm_destroy(smy_ep_comm* comm) { return ep_comm_destroy(comm); }

smy_status smy_moe_ep_workspace_bytes(const smy_moe_config* cfg, int64_t max_tokens, int32_t world, size_t* bytes) {
  if (!cfg || !bytes) return SMY_E_NULL;
  if (max_tokens < 0 || world < 1 || cfg->num_experts % world) return SMY_E_SHAPE;
  return ep_workspace_bytes(cfg, max_tokens, world, bytes);
}

smy_status samoyeds_ep_row_ids(const int32_t* send_sel, const int32_t* send_offsets, int32_t world, int32_t rank,
                               int64_t max_rows, int32_t* row_ids, void* stream) {
  if (max_rows > 0 && (!send_sel || !send_offsets || !row_ids)) return SMY_E_NULL;
  if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world || max_rows >= (1 << 24)) return SMY_E_SHAPE;
  smy_status st;
  if ((st = check_arch()) != SMY_OK) return st;
  return ep_row_ids_launch(send_sel, send_offsets, world, rank, max_rows, row_ids, static_cast<cudaStream_t>(stream));
}

smy_status samoyeds_moe_experts_peer(const smy_moe_config* cfg, const smy_weight* experts, int32_t world,
                                     const void* const* x_peers, int64_t ldx, float* const* out_peers, int64_t ldo,
                                     int64_t rows, const int32_t* row_map, const int32_t* keys, const float* vals,
                                     void* workspace, size_t ws_bytes, void* stream) {
  if (!cfg || !experts || !x_peers || !out_peers || !workspace) return SMY_E_NULL;
  if (rows > 0 && (!row_map || !keys || !vals)) return SMY_E_NULL;
  if (world < 1 || world > kMaxPeers) return SMY_E_SHAPE;
  for (int p = 0; p < world; ++p)
    if (!x_peers[p] || !out_peers[p]) return SMY_E_NULL;
  if (cfg->num_experts < 1 || cfg->top_k < 1 || cfg->top_k > 8 || cfg->num_experts > kMaxGroups ||
      cfg->num_shared != 0 || cfg->out_dtype != SMY_F32)
    return SMY_E_CONFIG;
  if (cfg->hidden % 128 || cfg->ffn % 128 || rows < 0 || ldx < cfg->hidden || ldx % 8 || ldo < cfg->hidden ||
      ldo % 4)
    return SMY_E_SHAPE;
  smy_status st;
  if ((st = check_experts(cfg, experts, cfg->num_experts)) != SMY_OK) return st;
  if ((st = check_arch()) != SMY_OK) return st;
  PeerRows pr;
  memset(&pr, 0, sizeof(pr));
  pr.world = world;
  pr.row_map = row_map;
  for (int p = 0; p < world; ++p) {
    pr.x_peers[p] = static_cast<const uint16_t*>(x_peers[p]);
    pr.out_peers[p] = out_peers[p];
  }
  pr.ldx = ldx;
  pr.ldo = ldo;
  return moe_core(cfg, experts, nullptr, x_peers[0], nullptr, keys, vals, rows, out_peers[0], workspace, ws_bytes,
                  static_cast<cudaStream_t>(stream), &pr);
}

smy_status samoyeds_ep_combine(const float* back, int64_t hidden, const int32_t* send_offsets, int32_t world,
                               const int32_t* send_sel, int64_t max_rows, float* out, void* stream) {
  if (max_rows > 0 && (!back || !send_offsets || !send_sel || !out)) return SMY_E_NULL;
  if (hidden % 2 || world < 1) return SMY_E_SHAPE;
  smy_status st;
  if ((st = check_arch()) != SMY_OK) return st;
  return ep_combine_launch(back, hidden, send_offsets, world, send_sel, max_rows, out,
                           static_cast<cudaStream_t>(stream));
}

smy_status smy_moe_set_phase_events(void** events, int n) {
  if (events == nullptr) {
    g_phase_on = false;
    return SMY_OK;
  }
  if (n < 6) return SMY_E_SHAPE;
  for (int i = 0; i < 6; ++i) g_phase[i] = static_cast<cudaEvent_t>(events[i]);
  g_phase_on = true;
  return SMY_OK;
}

uint64_t smy_launch_count(void) { return g_launches.load(); }

smy_status smy_moe_variant_scratch_bytes(const smy_moe_config* cfg, int64_t T, int32_t variant, size_t* bytes) {
  if (!cfg || !bytes) return SMY_E_NULL;
  if (T < 0) return SMY_E_SHAPE;
  return moe_variant_bytes(cfg, T, variant, bytes);
}

smy_status smy_moe_set_variant(int32_t variant, void* scratch, size_t bytes) {
  return moe_set_variant(variant, scratch, bytes);
}

// SMY_DEBUG & 128: accumulated per-role cycle counters of the last pair-kernel launches
int smy_debug_prof(unsigned long long* host, int ctas) {
  if (!g_prof || ctas > g_prof_ctas) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_prof, sizeof(unsigned long long) * 32 * ctas, cudaMemcpyDeviceToHost);
  cudaMemset(g_prof, 0, sizeof(unsigned long long) * 32 * g_prof_ctas);
  return ctas;
}

smy_status smy_synth_fill(uint64_t seed, int dist, float scale, int lo, int hi, int64_t idx0, int64_t n, void* out,
                          int out_bf16, void* stream) {
  if (!out && n > 0) return SMY_E_NULL;
  if (dist < 0 || dist > 2 || (dist == 2 && hi < lo)) return SMY_E_CONFIG;
  smy_status st;
  if ((st = check_arch()) != SMY_OK) return st;
  return synth_launch(seed, dist, scale, lo, hi, idx0, n, out, out_bf16, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
