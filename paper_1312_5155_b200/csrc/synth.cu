// synth.cu -- device twin of synth/__init__.py (input generator only; see include/rs_synth.h).
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/rs_synth.h"

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(uint8_t *base, uint64_t n_stripes, uint64_t ss, uint64_t bs, uint64_t B, int k,
                            uint64_t seed, uint64_t stripe0, int aligned8) {
  const uint64_t words = (B + 7) / 8;
  const uint64_t total = n_stripes * (uint64_t)k * words;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t q = i % words, sj = i / words;
    const uint64_t j = sj % (uint64_t)k, s = sj / (uint64_t)k;
    const uint64_t v = splitmix64((seed << 48) | ((stripe0 + s) << 32) | (j << 24) | q);
    uint8_t *p = base + s * ss + j * bs + q * 8;
    if (aligned8 && q * 8 + 8 <= B) {
      *reinterpret_cast<uint64_t *>(p) = v;
    } else {
      for (uint64_t b = 0; b < 8 && q * 8 + b < B; ++b) p[b] = (uint8_t)(v >> (8 * b));
    }
  }
}

}  // namespace

extern "C" int rs_synth_fill(void *stripes, size_t n_stripes, size_t stripe_stride, size_t block_stride,
                             size_t block_bytes, int k, uint32_t seed, uint32_t stripe0, void *stream) {
  if (seed >= (1u << 16) || (uint64_t)stripe0 + n_stripes > (1ull << 16) || k < 1 || k > 254 ||
      block_bytes > (1ull << 27) || (!stripes && n_stripes))
    return -1;
  if (n_stripes == 0 || block_bytes == 0) return 0;
  const uintptr_t b = reinterpret_cast<uintptr_t>(stripes);
  const int aligned8 = (b % 8 == 0 && stripe_stride % 8 == 0 && block_stride % 8 == 0) ? 1 : 0;
  fill_kernel<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<uint8_t *>(stripes), n_stripes, stripe_stride, block_stride, block_bytes, k, seed, stripe0,
      aligned8);
  return (int)cudaGetLastError();
}
