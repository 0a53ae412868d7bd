// samoyeds_compress: (optional magnitude pruning) + encoding into the
// canonical data / indices / metadata (§4.1) and packing into the
// sm_100a device image (the B200 counterpart of §4.4's data packing).
#include <cuda_bf16.h>

#include "internal.h"

namespace smy {

__device__ __forceinline__ float bf16_abs_f32(uint16_t b) { return __uint_as_float((uint32_t)(b & 0x7FFF) << 16); }
__device__ __forceinline__ bool bf16_nz(uint16_t b) { return (b & 0x7FFF) != 0; }

// One thread per (row-group g, K-block j): select the N kept sub-rows and the
// 2-of-4 positions, write values / codes / indices.
__global__ void encode_kernel(const uint16_t* __restrict__ w, int64_t ldw, int64_t rows, int64_t cols, int N,
                              int M, int V, int prune, uint16_t* __restrict__ values, uint8_t* __restrict__ codes,
                              uint8_t* __restrict__ indices, int32_t* status) {
  const int64_t J = cols / V;
  const int64_t G = rows / M;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= G * J) return;
  const int64_t g = tid / J, j = tid % J;
  const uint16_t* blk = w + (g * M) * ldw + j * V;

  // --- choose the N sub-rows (ascending row order)
  int pick[16];
  if (prune) {
    float score[16];
    for (int r = 0; r < M; ++r) {
      float acc = 0.f;
      for (int c = 0; c < V; ++c) acc = __fadd_rn(acc, bf16_abs_f32(blk[r * ldw + c]));  // sequential fp32 (R4)
      score[r] = acc;
    }
    int n = 0;
    for (int r = 0; r < M; ++r) {
      int beaten = 0;
      for (int o = 0; o < M; ++o) beaten += (score[o] > score[r]) || (score[o] == score[r] && o < r);
      if (beaten < N) pick[n++] = r;
    }
  } else {
    bool nz[16];
    int cnt = 0;
    for (int r = 0; r < M; ++r) {
      bool any = false;
      for (int c = 0; c < V; ++c) any |= bf16_nz(blk[r * ldw + c]);
      nz[r] = any;
      cnt += any;
    }
    if (cnt > N && status) atomicExch(status, (int)SMY_E_PATTERN);
    // non-zero rows first, then the lowest unused rows (R5), then sort ascending
    int n = 0;
    for (int r = 0; r < M && n < N; ++r)
      if (nz[r]) pick[n++] = r;
    for (int r = 0; r < M && n < N; ++r)
      if (!nz[r]) pick[n++] = r;
    for (int a = 1; a < N; ++a)  // insertion sort
      for (int b = a; b > 0 && pick[b - 1] > pick[b]; --b) {
        int t = pick[b]; pick[b] = pick[b - 1]; pick[b - 1] = t;
      }
  }

  // --- per kept sub-row: 2 of every 4 elements
  for (int i = 0; i < N; ++i) {
    const int64_t rc = g * N + i;  // compressed row
    const uint16_t* src = blk + pick[i] * ldw;
    indices[rc * J + j] = (uint8_t)pick[i];
    uint16_t* vout = values + rc * (cols / 2) + j * (V / 2);
    uint8_t* cout = codes + rc * (cols / 8) + j * (V / 8);
    for (int q = 0; q < V / 4; q += 2) {
      uint8_t byte = 0;
      for (int h = 0; h < 2; ++h) {
        const uint16_t* e = src + 4 * (q + h);
        int p0, p1;
        if (prune) {  // two largest |w|, ties -> lower position
          int keep[2], nk = 0;
          for (int p = 0; p < 4; ++p) {
            int beaten = 0;
            const float ap = bf16_abs_f32(e[p]);
            for (int o = 0; o < 4; ++o) {
              const float ao = bf16_abs_f32(e[o]);
              beaten += (ao > ap) || (ao == ap && o < p);
            }
            if (beaten < 2) keep[nk++] = p;
          }
          p0 = keep[0]; p1 = keep[1];
        } else {  // the non-zeros, padded with the smallest unused positions (R6)
          int pos[4], np = 0, nzc = 0;
          for (int p = 0; p < 4; ++p) nzc += bf16_nz(e[p]);
          if (nzc > 2 && status) atomicExch(status, (int)SMY_E_PATTERN);
          for (int p = 0; p < 4 && np < 2; ++p)
            if (bf16_nz(e[p])) pos[np++] = p;
          for (int p = 0; p < 4 && np < 2; ++p)
            if (!bf16_nz(e[p])) pos[np++] = p;
          p0 = min(pos[0], pos[1]); p1 = max(pos[0], pos[1]);
        }
        vout[2 * (q + h)] = e[p0];
        vout[2 * (q + h) + 1] = e[p1];
        byte |= (uint8_t)((p0 | (p1 << 2)) << (4 * h));
      }
      cout[q / 2] = byte;
    }
  }
}

// One CTA (128 threads = 128 TMEM lanes) per (m_tile, k_stage) image block.
__global__ void pack_kernel(const uint16_t* __restrict__ values, const uint8_t* __restrict__ codes,
                            const uint8_t* __restrict__ indices, int64_t R, int64_t cols, int V, int rep, int P,
                            int k_stages, int block, uint8_t* __restrict__ image) {
  const int mt = blockIdx.x / k_stages, s = blockIdx.x % k_stages;
  const int l = threadIdx.x;
  const int64_t cr = (int64_t)mt * kTileM + l;
  const bool valid = cr < R;
  uint8_t* blk = image + (size_t)blockIdx.x * block;
  const int64_t vcols = cols / 2, ccols = cols / 8, icols = cols / V;

  // A: 8 chunks of 16 B per row, 128B swizzle
  for (int ch = 0; ch < 8; ++ch) {
    const int kb = ch >> 1, half = ch & 1;
    const int vb = s * 4 + kb;
    uint4 val = make_uint4(0, 0, 0, 0);
    if (valid) {
      const int j = vb / rep, h = vb % rep;
      if (rep == 1 || half == h)
        val = *reinterpret_cast<const uint4*>(values + cr * vcols + (int64_t)j * 16 + half * 8);
    }
    *reinterpret_cast<uint4*>(blk + (l >> 3) * 1024 + (l & 7) * 128 + ((ch ^ (l & 7)) << 4)) = val;
  }
  // E: lane-major TMEM image
  {
    const int r_lo = (l & 7) + 16 * (l >> 4), r_hi = r_lo + 8, k1 = (l >> 3) & 1;
    const int64_t c_lo = (int64_t)mt * kTileM + r_lo, c_hi = (int64_t)mt * kTileM + r_hi;
    uint32_t wd[4];
    for (int kb = 0; kb < 4; ++kb) {
      const int vb = s * 4 + kb;
      const int j = vb / rep, h = vb % rep;
      const bool live = rep == 1 || k1 == h;
      // 4-groups 8j+4k1 .. +3 of the row = codes bytes 4j+2k1, 4j+2k1+1 (nibble q at bits 4q)
      auto half16 = [&](int64_t crow) -> uint32_t {
        if (!live || crow >= R) return 0x4444u;
        const uint8_t* c = codes + crow * ccols + (int64_t)j * 4 + k1 * 2;
        return (uint32_t)c[0] | ((uint32_t)c[1] << 8);
      };
      wd[kb] = half16(c_lo) | (half16(c_hi) << 16);
    }
    *reinterpret_cast<uint4*>(blk + kABytes + 16 * l) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
  }
  // index bit-planes
  for (int kb = 0; kb < 4; ++kb) {
    const int vb = s * 4 + kb;
    const int vblock = rep == 1 ? (vb * 32) / V : vb;
    const int idx = valid ? indices[cr * icols + vblock] : 0;
    for (int b = 0; b < P; ++b) {
      const uint32_t word = __ballot_sync(0xffffffffu, (idx >> b) & 1);
      if ((l & 31) == 0) *reinterpret_cast<uint32_t*>(blk + kABytes + kEBytes + (kb * P + b) * 16 + (l >> 5) * 4) = word;
    }
  }
  // zero the tail pad
  for (int o = kABytes + kEBytes + 64 * P + 4 * l; o < block; o += 4 * kTileM)
    *reinterpret_cast<uint32_t*>(blk + o) = 0u;
}

// Interleaved gate/up (reading R20): gu compressed row r' of block b = r' / (2 cb)
// (cb = 16 compressed rows) comes from gate (first half of the
// block) or up (second half), row b * cb + r' % cb.  One CTA per gu row.
__global__ void interleave_rows_kernel(const uint8_t* __restrict__ gv, const uint8_t* __restrict__ gc,
                                       const uint8_t* __restrict__ gi, const uint8_t* __restrict__ uv,
                                       const uint8_t* __restrict__ uc, const uint8_t* __restrict__ ui, int64_t cb,
                                       int64_t vbytes, int64_t cbytes, int64_t ibytes, uint8_t* __restrict__ ov,
                                       uint8_t* __restrict__ oc, uint8_t* __restrict__ oi) {
  const int64_t r = blockIdx.x;
  const int64_t b = r / (2 * cb), within = r % (2 * cb);
  const bool from_up = within >= cb;
  const int64_t src = b * cb + (from_up ? within - cb : within);
  const uint4* sv = reinterpret_cast<const uint4*>((from_up ? uv : gv) + src * vbytes);
  const uint4* sc = reinterpret_cast<const uint4*>((from_up ? uc : gc) + src * cbytes);
  const uint8_t* si = (from_up ? ui : gi) + src * ibytes;
  uint4* dv = reinterpret_cast<uint4*>(ov + r * vbytes);
  uint4* dc = reinterpret_cast<uint4*>(oc + r * cbytes);
  for (int64_t i = threadIdx.x; i < vbytes / 16; i += blockDim.x) dv[i] = sv[i];
  for (int64_t i = threadIdx.x; i < cbytes / 16; i += blockDim.x) dc[i] = sc[i];
  for (int64_t i = threadIdx.x; i < ibytes; i += blockDim.x) oi[r * ibytes + i] = si[i];
}

// Decode (PAPER.md:237 inverse; oracle fmt.decode): every stored value of
// compressed row r, V-block j, 4-group q, slot s goes to
// W[g*M + idx[r][j], j*V + 4q + code]; everything else stays zero (memset first).
__global__ void decompress_kernel(const uint16_t* __restrict__ values, const uint8_t* __restrict__ codes,
                                  const uint8_t* __restrict__ indices, int64_t R, int64_t cols, int N, int M, int V,
                                  uint16_t* __restrict__ w, int64_t ldw) {
  const int64_t half = cols / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < R * half; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / half, c = i % half;
    const int64_t j = (2 * c) / V, q = (c % (V / 2)) / 2;
    const int code = (codes[r * (cols / 8) + c / 4] >> (2 * (c % 4))) & 3;
    const int sub = indices[r * (cols / V) + j];
    if (sub >= M) continue;  // corrupt index (reported by decode_check_kernel): no write outside the block
    const int64_t row = (r / N) * M + sub;
    w[row * ldw + j * V + 4 * q + code] = values[i];
  }
}

// The decoding invariants of the canonical arrays (reading R5/R6, S:43-44,
// S:80-88): per (row group g, K-block j) the N sub-row indices are < M and
// strictly increasing; per kept 4-group the two 2-bit codes are strictly
// increasing.  One thread per (g, j); any violation -> *status = SMY_E_CORRUPT.
__global__ void decode_check_kernel(const uint8_t* __restrict__ codes, const uint8_t* __restrict__ indices, int64_t G,
                                    int64_t cols, int N, int M, int V, int32_t* __restrict__ status) {
  const int64_t J = cols / V;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < G * J; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = i / J, j = i % J;
    bool bad = false;
    int prev = -1;
    for (int n = 0; n < N; ++n) {
      const int64_t r = g * N + n;
      const int sub = indices[r * J + j];
      bad |= sub >= M || sub <= prev;
      prev = sub;
      for (int q = 0; q < V / 4; ++q) {
        const int64_t c = j * (V / 2) + 2 * q;  // first of the two stored values of 4-group q
        const int c0 = (codes[r * (cols / 8) + c / 4] >> (2 * (c % 4))) & 3;
        const int c1 = (codes[r * (cols / 8) + (c + 1) / 4] >> (2 * ((c + 1) % 4))) & 3;
        bad |= c0 >= c1;
      }
    }
    if (bad) *status = SMY_E_CORRUPT;
  }
}

// SEL contract of samoyeds_ssmm: entries in [0, x_rows), strictly increasing.
__global__ void sel_check_kernel(const int32_t* __restrict__ sel, int32_t n, int64_t x_rows,
                                 int32_t* __restrict__ status) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t t = sel[i];
    if (t < 0 || t >= x_rows || (i > 0 && sel[i - 1] >= t)) *status = SMY_E_SELECTION;
  }
}

smy_status sel_check_launch(const int32_t* sel, int32_t n, int64_t x_rows, int32_t* d_status, cudaStream_t s) {
  if (n <= 0) return SMY_OK;
  int blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  sel_check_kernel<<<blocks, 256, 0, s>>>(sel, n, x_rows, d_status);
  count_launch();
  return cuda_status(cudaGetLastError());
}

smy_status decompress_launch(const smy_weight* src, uint16_t* w, int64_t ldw, int32_t* d_status, cudaStream_t s) {
  const smy_wdesc& d = src->d;
  cudaError_t e = cudaMemset2DAsync(w, (size_t)ldw * 2, 0, (size_t)d.cols * 2, (size_t)d.rows, s);
  if (e != cudaSuccess) return cuda_status(e);
  const int64_t R = d.rows * d.fmt.n / d.fmt.m;
  const int64_t n = R * (d.cols / 2);
  if (n == 0) return SMY_OK;
  if (d_status != nullptr) {
    const int64_t gj = (d.rows / d.fmt.m) * (d.cols / d.fmt.v);
    int cb = (int)((gj + 127) / 128);
    if (cb > 148 * 16) cb = 148 * 16;
    decode_check_kernel<<<cb, 128, 0, s>>>(static_cast<const uint8_t*>(src->codes),
                                           static_cast<const uint8_t*>(src->indices), d.rows / d.fmt.m, d.cols,
                                           d.fmt.n, d.fmt.m, d.fmt.v, d_status);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_status(e);
  }
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  decompress_kernel<<<blocks, 256, 0, s>>>(static_cast<const uint16_t*>(src->values),
                                           static_cast<const uint8_t*>(src->codes),
                                           static_cast<const uint8_t*>(src->indices), R, d.cols, d.fmt.n, d.fmt.m,
                                           d.fmt.v, w, ldw);
  count_launch();
  return cuda_status(cudaGetLastError());
}

smy_status interleave_launch(const smy_weight* gate, const smy_weight* up, const smy_wdesc& d, const Geometry& g,
                             smy_weight* gu, cudaStream_t s) {
  const int64_t cols = d.cols;
  if (cols % 128) return SMY_E_SHAPE;
  const int64_t cb = 16;  // compressed rows per interleave block (reading R20)
  interleave_rows_kernel<<<(unsigned)g.R, 128, 0, s>>>(
      static_cast<const uint8_t*>(gate->values), static_cast<const uint8_t*>(gate->codes),
      static_cast<const uint8_t*>(gate->indices), static_cast<const uint8_t*>(up->values),
      static_cast<const uint8_t*>(up->codes), static_cast<const uint8_t*>(up->indices), cb, cols, cols / 8,
      cols / d.fmt.v, static_cast<uint8_t*>(gu->values), static_cast<uint8_t*>(gu->codes),
      static_cast<uint8_t*>(gu->indices));
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e);
  pack_kernel<<<(unsigned)(g.m_tiles * g.k_stages), kTileM, 0, s>>>(
      static_cast<const uint16_t*>(gu->values), static_cast<const uint8_t*>(gu->codes),
      static_cast<const uint8_t*>(gu->indices), g.R, cols, d.fmt.v, g.rep, g.planes, g.k_stages, g.block,
      static_cast<uint8_t*>(gu->image));
  count_launch();
  return cuda_status(cudaGetLastError());
}

smy_status compress_launch(const smy_wdesc* d, const Geometry& g, const uint16_t* w, int64_t ldw, int flags,
                           smy_weight* out, int32_t* d_status, cudaStream_t s) {
  const int64_t G = d->rows / d->fmt.m, J = d->cols / d->fmt.v;
  const int64_t n = G * J;
  const int prune = (flags & SMY_PRUNE_MAGNITUDE) ? 1 : 0;
  encode_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(
      w, ldw, d->rows, d->cols, d->fmt.n, d->fmt.m, d->fmt.v, prune, static_cast<uint16_t*>(out->values),
      static_cast<uint8_t*>(out->codes), static_cast<uint8_t*>(out->indices), d_status);
  count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_status(e);
  pack_kernel<<<(unsigned)(g.m_tiles * g.k_stages), kTileM, 0, s>>>(
      static_cast<const uint16_t*>(out->values), static_cast<const uint8_t*>(out->codes),
      static_cast<const uint8_t*>(out->indices), g.R, d->cols, d->fmt.v, g.rep, g.planes, g.k_stages, g.block,
      static_cast<uint8_t*>(out->image));
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
