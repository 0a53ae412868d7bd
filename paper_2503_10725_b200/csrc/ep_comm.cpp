// smy_ep_comm: the library-owned NCCL communicator of expert parallelism, and the
// whole EP layer call behind samoyeds_moe_layer(..., comm, ...) (SURVEY.md §8(b):
// "the library ... owns only smy_ep_comm"; §8(e): one exchange step each way).
//
// NCCL is loaded with dlopen at smy_ep_comm_create time (libnccl.so.2: the copy a
// PyTorch process already has loaded, else the system one), so only EP users need
// it and the library has no link-time NCCL dependency.
//
//   route (all E) -> ep_plan -> ep_pack -> [send counts: group of ncclSend/Recv]
//   -> D2H of the [W] receive counts -> [rows + tags: ncclSend/Recv per peer]
//   -> moe_core over the received rows (keys path) -> [fp32 partial rows back]
//   -> ep_combine (red.add into the owner's output)
#include <dlfcn.h>

#include <cstring>
#include <vector>

#include "internal.h"

namespace smy {

namespace {
// the subset of nccl.h this file uses (ABI-stable since NCCL 2.0)
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclInt8 = 0, ncclInt32 = 2, ncclFloat32 = 7 } ncclDataType_t;
typedef int ncclResult_t;

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl* nccl() {
  static Nccl n;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      n.h = h;
      n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
      n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
      n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
      n.Send = reinterpret_cast<decltype(n.Send)>(dlsym(h, "ncclSend"));
      n.Recv = reinterpret_cast<decltype(n.Recv)>(dlsym(h, "ncclRecv"));
      n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(dlsym(h, "ncclGroupStart"));
      n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
      n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
    }
  }
  if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.CommDestroy || !n.Send || !n.Recv || !n.GroupStart ||
      !n.GroupEnd)
    return nullptr;
  return &n;
}

smy_status nccl_status(ncclResult_t r) {
  if (r == 0) return SMY_OK;
  Nccl* n = nccl();
  set_last_error(n && n->GetErrorString ? n->GetErrorString(r) : "NCCL error");
  return SMY_E_NCCL;
}

size_t up(size_t x) { return (x + 255) / 256 * 256; }

// workspace of one EP layer call: every rank may receive at most T rows from each peer
struct EpWs {
  int32_t *ids, *cnt_send, *off_send, *sel, *tag_ids, *cnt_recv, *r_counts, *r_offsets, *r_sel;
  float *w, *tag_w, *back, *part, *r_gw;
  uint16_t *x_send, *x_recv;
  int32_t* keys_recv;
  float* vals_recv;
  void *plan_ws, *core_ws;
  size_t plan_ws_bytes, core_ws_bytes, total;
};

EpWs carve_ep(const smy_moe_config* c, int64_t T, int world, uint8_t* base, size_t core_bytes) {
  EpWs w{};
  size_t off = 0;
  auto take = [&](size_t b) {
    uint8_t* p = base ? base + off : nullptr;
    off = up(off + b);
    return p;
  };
  const int64_t k = c->top_k, d = c->hidden;
  const int64_t S = T * k;                    // send rows (<= T per destination, <= T*k in all)
  const int64_t R = T * world;                // receive rows
  const int E = c->num_experts;
  w.ids = reinterpret_cast<int32_t*>(take(T * k * 4));
  w.w = reinterpret_cast<float*>(take(T * k * 4));
  w.r_counts = reinterpret_cast<int32_t*>(take(E * 4));        // routing's own per-expert compaction
  w.r_offsets = reinterpret_cast<int32_t*>(take((E + 1) * 4));
  w.r_sel = reinterpret_cast<int32_t*>(take(T * k * 4));
  w.r_gw = reinterpret_cast<float*>(take(T * k * 4));
  w.cnt_send = reinterpret_cast<int32_t*>(take(world * 4));
  w.off_send = reinterpret_cast<int32_t*>(take((world + 1) * 4));
  w.cnt_recv = reinterpret_cast<int32_t*>(take(world * 4));
  w.sel = reinterpret_cast<int32_t*>(take(S * 4));
  w.tag_ids = reinterpret_cast<int32_t*>(take(S * k * 4));
  w.tag_w = reinterpret_cast<float*>(take(S * k * 4));
  w.x_send = reinterpret_cast<uint16_t*>(take(S * d * 2));
  w.x_recv = reinterpret_cast<uint16_t*>(take(R * d * 2));
  w.keys_recv = reinterpret_cast<int32_t*>(take(R * k * 4));
  w.vals_recv = reinterpret_cast<float*>(take(R * k * 4));
  w.part = reinterpret_cast<float*>(take(R * d * 4));
  w.back = reinterpret_cast<float*>(take(S * d * 4));
  w.plan_ws_bytes = ep_plan_ws_bytes(T, world, (int)k);
  if (route_ws_bytes(T, E) > w.plan_ws_bytes) w.plan_ws_bytes = route_ws_bytes(T, E);
  w.plan_ws = take(w.plan_ws_bytes);
  w.core_ws_bytes = core_bytes;
  w.core_ws = take(core_bytes);
  w.total = off;
  return w;
}
}  // namespace

}  // namespace smy

struct smy_ep_comm {
  smy::ncclComm_t comm;
  int rank, world;
};

namespace smy {

smy_status ep_unique_id(void* out128) {
  Nccl* n = nccl();
  if (!n) {
    set_last_error("libnccl.so.2 not found");
    return SMY_E_NCCL;
  }
  ncclUniqueId id;
  smy_status st = nccl_status(n->GetUniqueId(&id));
  if (st == SMY_OK) memcpy(out128, &id, sizeof(id));
  return st;
}

smy_status ep_comm_create(const void* id128, int rank, int world, smy_ep_comm** out) {
  Nccl* n = nccl();
  if (!n) {
    set_last_error("libnccl.so.2 not found");
    return SMY_E_NCCL;
  }
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  ncclComm_t c = nullptr;
  smy_status st = nccl_status(n->CommInitRank(&c, world, id, rank));
  if (st != SMY_OK) return st;
  *out = new smy_ep_comm{c, rank, world};
  return SMY_OK;
}

smy_status ep_comm_destroy(smy_ep_comm* c) {
  if (!c) return SMY_OK;
  Nccl* n = nccl();
  smy_status st = n ? nccl_status(n->CommDestroy(c->comm)) : SMY_E_NCCL;
  delete c;
  return st;
}

int ep_comm_world(const smy_ep_comm* c) { return c->world; }

smy_status ep_workspace_bytes(const smy_moe_config* c, int64_t T, int world, size_t* bytes) {
  smy_moe_config lc = *c;
  lc.num_experts = c->num_experts / world;
  size_t core = 0;
  smy_status st = moe_workspace_bytes(&lc, T * world, &core);
  if (st != SMY_OK) return st;
  *bytes = carve_ep(c, T, world, nullptr, core).total;
  return SMY_OK;
}

// the largest max_tokens whose EP workspace fits in ws_bytes (the byte count is
// monotone in T): receive buffers are sized by it, not by the call's T, because a
// peer may send up to ITS T rows
static int64_t ep_capacity(const smy_moe_config* c, int world, size_t ws_bytes) {
  int64_t lo = 0, hi = (int64_t)1 << 24;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) / 2;
    size_t b = 0;
    if (ep_workspace_bytes(c, mid, world, &b) == SMY_OK && b <= ws_bytes) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

smy_status ep_layer(const smy_moe_config* c, const smy_weight* experts, const void* x, const float* logits, int64_t T,
                    float* out, void* workspace, size_t ws_bytes, smy_ep_comm* comm, cudaStream_t s) {
  Nccl* n = nccl();
  if (!n) return SMY_E_NCCL;
  const int W = comm->world, E = c->num_experts, k = c->top_k;
  const int64_t d = c->hidden;
  if (E % W) return SMY_E_CONFIG;
  smy_moe_config lc = *c;
  lc.num_experts = E / W;
  // every rank sizes its workspace for the same max_tokens (include/samoyeds.h)
  const int64_t cap = ep_capacity(c, W, ws_bytes);
  size_t core = 0;
  smy_status st = moe_workspace_bytes(&lc, cap * W, &core);
  if (st != SMY_OK) return st;
  EpWs w = carve_ep(c, cap, W, static_cast<uint8_t*>(workspace), core);
  if (w.total > ws_bytes || w.total == 0) return SMY_E_WORKSPACE;

  // 1. route this rank's tokens over all E experts; plan one copy per destination
  //    rank.  A local failure is announced to every peer in the counts exchange
  //    (count -1) so that all ranks leave after it and none blocks in NCCL.
  smy_status local = T > cap ? SMY_E_WORKSPACE : SMY_OK;
  if (local == SMY_OK)
    local = route_launch(logits, T, E, k, c->gating, w.ids, w.w, w.r_counts, w.r_offsets, w.r_sel, w.r_gw,
                         w.plan_ws, w.plan_ws_bytes, nullptr, nullptr, 0, nullptr, s);
  if (local == SMY_OK)
    local = ep_plan_launch(w.ids, w.w, T, k, E, W, w.cnt_send, w.off_send, w.sel, w.tag_ids, w.tag_w, w.plan_ws,
                           w.plan_ws_bytes, s);
  if (local == SMY_OK)
    local = ep_pack_launch(static_cast<const uint16_t*>(x), d, d, w.off_send, W, w.sel, T * k, w.x_send, s);
  if (local != SMY_OK) {
    cudaGetLastError();
    if (cudaMemsetAsync(w.cnt_send, 0xFF, W * 4, s) != cudaSuccess) return cuda_status(cudaGetLastError());
  }

  // 2. counts: one int per peer each way, then the host needs them for the split sizes
  n->GroupStart();
  for (int q = 0; q < W; ++q) {
    n->Send(w.cnt_send + q, 1, ncclInt32, q, comm->comm, s);
    n->Recv(w.cnt_recv + q, 1, ncclInt32, q, comm->comm, s);
  }
  if ((st = nccl_status(n->GroupEnd())) != SMY_OK) return st;
  std::vector<int32_t> cs(W), cr(W);
  cudaMemcpyAsync(cs.data(), w.cnt_send, W * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(cr.data(), w.cnt_recv, W * 4, cudaMemcpyDeviceToHost, s);
  cudaError_t ce = cudaStreamSynchronize(s);
  if (ce != cudaSuccess) return cuda_status(ce);
  if (local != SMY_OK) return local;
  for (int q = 0; q < W; ++q)
    if (cr[q] < 0) {
      set_last_error("expert parallelism: a peer rank failed before the dispatch (T > its workspace, or a launch)");
      return SMY_E_WORKSPACE;
    }
  std::vector<int64_t> os(W + 1, 0), orr(W + 1, 0);
  for (int q = 0; q < W; ++q) {
    os[q + 1] = os[q] + cs[q];
    orr[q + 1] = orr[q] + cr[q];
  }
  const int64_t R = orr[W];
  if (R > cap * W) {  // only with mismatched max_tokens across ranks (a caller contract violation)
    set_last_error("expert parallelism: received rows exceed the workspace (ranks sized for different max_tokens)");
    return SMY_E_WORKSPACE;
  }

  // 3. dispatch: token rows + tags (local expert ids, gate weights)
  n->GroupStart();
  for (int q = 0; q < W; ++q) {
    if (cs[q]) {
      n->Send(w.x_send + os[q] * d, (size_t)cs[q] * d * 2, ncclInt8, q, comm->comm, s);
      n->Send(w.tag_ids + os[q] * k, (size_t)cs[q] * k, ncclInt32, q, comm->comm, s);
      n->Send(w.tag_w + os[q] * k, (size_t)cs[q] * k, ncclFloat32, q, comm->comm, s);
    }
    if (cr[q]) {
      n->Recv(w.x_recv + orr[q] * d, (size_t)cr[q] * d * 2, ncclInt8, q, comm->comm, s);
      n->Recv(w.keys_recv + orr[q] * k, (size_t)cr[q] * k, ncclInt32, q, comm->comm, s);
      n->Recv(w.vals_recv + orr[q] * k, (size_t)cr[q] * k, ncclFloat32, q, comm->comm, s);
    }
  }
  if ((st = nccl_status(n->GroupEnd())) != SMY_OK) return st;

  // 4. this rank's experts over the received rows -> fp32 partial rows (a failure
  //    here still posts the combine below: the peers are waiting for it)
  const smy_status core_st = moe_core(&lc, experts, nullptr, w.x_recv, nullptr, w.keys_recv, w.vals_recv, R, w.part,
                                      w.core_ws, w.core_ws_bytes, s);
  if (core_st != SMY_OK) cudaGetLastError();

  // 5. combine: partial rows back to their token's rank, summed into out
  n->GroupStart();
  for (int q = 0; q < W; ++q) {
    if (cr[q]) n->Send(w.part + orr[q] * d, (size_t)cr[q] * d, ncclFloat32, q, comm->comm, s);
    if (cs[q]) n->Recv(w.back + os[q] * d, (size_t)cs[q] * d, ncclFloat32, q, comm->comm, s);
  }
  if ((st = nccl_status(n->GroupEnd())) != SMY_OK) return st;
  if (core_st != SMY_OK) return core_st;
  ce = cudaMemsetAsync(out, 0, (size_t)T * d * 4, s);
  if (ce != cudaSuccess) return cuda_status(ce);
  return ep_combine_launch(w.back, d, w.off_send, W, w.sel, T * k, out, s);
}

}  // namespace smy
