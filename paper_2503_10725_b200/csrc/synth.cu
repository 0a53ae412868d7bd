// Counter-based synthetic input generator: the CUDA twin of synth/__init__.py.
// Input preparation only (no Samoyeds arithmetic); pinned bit-exactly against
// the NumPy generator by tests/test_synth_gpu.py.
#include <cuda_bf16.h>

#include "internal.h"

namespace smy {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
__host__ __device__ inline uint64_t mix64_h(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_kernel(uint64_t key, uint64_t key2, int dist, float scale, int lo, int hi, int64_t idx0,
                             int64_t n, void* out, int out_bf16) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t idx = (uint64_t)(idx0 + i);
    const uint64_t h = mix64(key + (idx + 1) * kPhi);
    float v;
    if (dist == 0) {
      const int64_t m = (int64_t)(h >> 40);
      v = __fmul_rn((float)(2 * m - (1ll << 24)), scale);
    } else if (dist == 1) {
      const uint64_t h2 = mix64(key2 + (idx + 1) * kPhi);
      const int64_t s = (int64_t)(h >> 40) + (int64_t)((h >> 16) & 0xFFFFFF) + (int64_t)(h2 >> 40) +
                        (int64_t)((h2 >> 16) & 0xFFFFFF) - (1ll << 25);
      v = __fmul_rn(__ll2float_rn(s), scale);
    } else {
      const uint64_t span = (uint64_t)(hi - lo + 1);
      v = (float)((int64_t)((h >> 32) % span) + lo);
    }
    if (out_bf16)
      static_cast<uint16_t*>(out)[i] = __bfloat16_as_ushort(__float2bfloat16_rn(v));
    else
      static_cast<float*>(out)[i] = v;
  }
}

smy_status synth_launch(uint64_t seed, int dist, float scale, int lo, int hi, int64_t idx0, int64_t n, void* out,
                        int out_bf16, cudaStream_t s) {
  const uint64_t key = mix64_h(seed * kPhi + kPhi);
  const uint64_t key2 = mix64_h((seed ^ 0x5DEECE66Dull) * kPhi + kPhi);
  if (n <= 0) return SMY_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  synth_kernel<<<blocks, 256, 0, s>>>(key, key2, dist, scale, lo, hi, idx0, n, out, out_bf16);
  count_launch();
  return cuda_status(cudaGetLastError());
}

}  // namespace smy
