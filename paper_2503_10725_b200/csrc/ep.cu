// Expert parallelism (EP) device kernels: dispatch plan, pack, combine.
//
// Rank r owns experts [r*E/P, (r+1)*E/P).  A token is sent ONCE to every rank
// that owns at least one of its top-k experts, with tags (local expert id,
// gate weight) for the experts it meets there; the receive buffer of a rank is
// ordered by (source rank, token id) -- deterministic (oracle/moe.py:
// ep_dispatch_plan).  The exchange itself (all_to_all_v over NCCL/NVLink) is
// done by the caller's process group between samoyeds_ep_pack and
// samoyeds_moe_experts, and back before samoyeds_ep_combine.
#include "internal.h"
#include "ptx.cuh"

namespace smy {

constexpr int kEpMaxK = 8;

// dkeys[t][j] = destination rank of ids[t][j] if it is its first occurrence in
// the token's list, else -1 (one copy per destination).
__global__ void ep_dest_keys_kernel(const int32_t* __restrict__ ids, int64_t T, int k, int e_local,
                                    int32_t* __restrict__ dkeys, float* __restrict__ ones) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  for (int j = 0; j < k; ++j) {
    const int d = ids[t * k + j] / e_local;
    bool first = true;
    for (int i = 0; i < j; ++i) first &= (ids[t * k + i] / e_local) != d;
    dkeys[t * k + j] = first ? d : -1;
    ones[t * k + j] = 1.f;
  }
}

__device__ __forceinline__ int dest_of(const int32_t* offsets, int world, int pos) {
  int d = 0;
  while (d + 1 < world && offsets[d + 1] <= pos) ++d;
  return d;
}

// For every send row: the tags (local expert ids ascending, weights), -1 padded.
__global__ void ep_tags_kernel(const int32_t* __restrict__ ids, const float* __restrict__ w, int k, int e_local,
                               const int32_t* __restrict__ offsets, int world, const int32_t* __restrict__ sel,
                               int64_t max_rows, int32_t* __restrict__ tag_ids, float* __restrict__ tag_w) {
  const int S = offsets[world];
  for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < S && pos < max_rows;
       pos += (int64_t)gridDim.x * blockDim.x) {
    const int d = dest_of(offsets, world, (int)pos);
    const int t = sel[pos];
    int li[kEpMaxK];
    float lw[kEpMaxK];
    int n = 0;
    for (int j = 0; j < k; ++j) {
      const int e = ids[(int64_t)t * k + j];
      if (e / e_local == d) {
        int p = n++;
        const int le = e - d * e_local;
        while (p > 0 && li[p - 1] > le) { li[p] = li[p - 1]; lw[p] = lw[p - 1]; --p; }
        li[p] = le;
        lw[p] = w[(int64_t)t * k + j];
      }
    }
    for (int j = 0; j < k; ++j) {
      tag_ids[pos * k + j] = j < n ? li[j] : -1;
      tag_w[pos * k + j] = j < n ? lw[j] : 0.f;
    }
  }
}

// x_send[pos] = x[sel[pos]] (bf16 rows, 16-byte vectors)
__global__ void ep_pack_kernel(const uint16_t* __restrict__ x, int64_t ldx, int64_t d,
                               const int32_t* __restrict__ offsets, int world, const int32_t* __restrict__ sel,
                               int64_t max_rows, uint16_t* __restrict__ xs) {
  const int S = offsets[world];
  const int64_t vec = d / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)S * vec && i < max_rows * vec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = i / vec, c = i % vec;
    const uint4 v = *reinterpret_cast<const uint4*>(x + (int64_t)sel[pos] * ldx + c * 8);
    *reinterpret_cast<uint4*>(xs + pos * d + c * 8) = v;
  }
}

// out[sel[pos]] += back[pos]  (fp32 rows; one token may come back from several ranks)
__global__ void ep_combine_kernel(const float* __restrict__ back, int64_t d, const int32_t* __restrict__ offsets,
                                  int world, const int32_t* __restrict__ sel, int64_t max_rows,
                                  float* __restrict__ out) {
  const int S = offsets[world];
  const int64_t vec = d / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (int64_t)S * vec && i < max_rows * vec;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = i / vec, c = i % vec;
    const float2 v = *reinterpret_cast<const float2*>(back + pos * d + c * 2);
    red_add_v2(out + (int64_t)sel[pos] * d + c * 2, v.x, v.y);
  }
}

size_t ep_plan_ws_bytes(int64_t T, int world, int k) {
  return route_ws_bytes(T, world) + 2 * (size_t)T * k * 4 + 1024;
}

// row_ids[i] = (rank << 24) | sel[i] for the send rows i < offsets[world]: the id under
// which the destination reads this token's row from, and adds its output into, this
// rank's peer-mapped buffers (expert parallelism over NVLink peer memory)
__global__ void ep_row_ids_kernel(const int32_t* __restrict__ sel, const int32_t* __restrict__ offsets, int world,
                                  int rank, int64_t max_rows, int32_t* __restrict__ row_ids) {
  const int64_t n = min((int64_t)offsets[world], max_rows);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    row_ids[i] = (rank << 24) | sel[i];
}

smy_status ep_row_ids_launch(const int32_t* sel, const int32_t* offsets, int world, int rank, int64_t max_rows,
                             int32_t* row_ids, cudaStream_t s) {
  if (max_rows <= 0) return SMY_OK;
  int blocks = (int)((max_rows + 255) / 256);
  if (blocks > 148 * 4) blocks = 148 * 4;
  ep_row_ids_kernel<<<blocks, 256, 0, s>>>(sel, offsets, world, rank, max_rows, row_ids);
  count_launch();
  return cuda_status(cudaGetLastError());
}

smy_status ep_plan_launch(const int32_t* ids, const float* w, int64_t T, int k, int E, int world, int32_t* counts,
                          int32_t* offsets, int32_t* sel, int32_t* tag_ids, float* tag_w, void* ws, size_t ws_bytes,
                          cudaStream_t s) {
  if (ws_bytes < ep_plan_ws_bytes(T, world, k)) return SMY_E_WORKSPACE;
  const int e_local = E / world;
  uint8_t* p = static_cast<uint8_t*>(ws);
  int32_t* dkeys = reinterpret_cast<int32_t*>(p);
  float* ones = reinterpret_cast<float*>(p + (size_t)T * k * 4);
  void* cws = p + 2 * (size_t)T * k * 4;
  const size_t cws_bytes = ws_bytes - 2 * (size_t)T * k * 4;
  if (T > 0) {
    ep_dest_keys_kernel<<<(unsigned)((T + 255) / 256), 256, 0, s>>>(ids, T, k, e_local, dkeys, ones);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e);
  smy_status st = compact_launch(dkeys, ones, T, world, k, counts, offsets, sel, ones /*unused vals out*/, cws,
                                 cws_bytes, nullptr, nullptr, 0, nullptr, s);
  if (st != SMY_OK || T == 0) return st;
  const int64_t rows = T * k;
  int blocks = (int)((rows + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  ep_tags_kernel<<<blocks, 256, 0, s>>>(ids, w, k, e_local, offsets, world, sel, rows, tag_ids, tag_w);
  count_launch();
  return cuda_status(cudaGetLastError());
}

smy_status ep_pack_launch(const uint16_t* x, int64_t ldx, int64_t d, const int32_t* offsets, int world,
                          const int32_t* sel, int64_t max_rows, uint16_t* xs, cudaStream_t s) {
  if (max_rows <= 0) return SMY_OK;
  int64_t n = max_rows * (d / 8);
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  ep_pack_kernel<<<blocks, 256, 0, s>>>(x, ldx, d, offsets, world, sel, max_rows, xs);
  count_launch();
  return cuda_status(cudaGetLastError());
}

smy_status ep_combine_launch(const float* back, int64_t d, const int32_t* offsets, int world, const int32_t* sel,
                             int64_t max_rows, float* out, cudaStream_t s) {
  if (max_rows <= 0) return SMY_OK;
  int64_t n = max_rows * (d / 2);
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  ep_combine_kernel<<<blocks, 256, 0, s>>>(back, d, offsets, world, sel, max_rows, out);
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
