// Streaming ceiling of the codec's access mix on sm_100a (measurement only, not the product).
//
// The roofline peak in MEASURED_PEAKS.json is a 1:1 copy (torch b.copy_(a)).  The codec kernels
// read (n - t) blocks and write t (decode) or read k and write m (encode) per stripe, with 256-bit
// loads / stores over the [S][n][B] batch layout.  This kernel moves exactly those bytes with the
// same access instructions and the same launch shape (one launch per stripe, 128-thread CTAs,
// one or two 32-byte units per thread per block, or one grid-stride launch over every stripe) and
// does no GF arithmetic (each output = XOR of the inputs and its index), so its rate is the
// HBM ceiling for that read:write mix and layout.  DESIGN.md §6 quotes the codec kernels against it.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_mix stream_mix.cu
//   ./stream_mix                 # JSON lines: one per (mix, launch shape)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) {                                                               \
      fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                            \
    }                                                                                      \
  } while (0)

__device__ __forceinline__ void ldg_v8(const void *p, uint32_t *r) {
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void stg_v8(void *p, const uint32_t *r) {
  asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// Block b of stripe s starts at base + s*stripe_stride + b*B.  Blocks [0, R) are read, blocks
// [R, R + W) written.  A "unit" is 32 bytes of every block (the w8 codec's unit; the w16 codec's
// unit is two of them).  Unit u of the launch covers stripe s0 + u / units_per_stripe.
template <int R, int W, int UPT>
__global__ void __launch_bounds__(128) mix_kernel(uint8_t *base, uint64_t stripe_stride, uint64_t B,
                                                  uint64_t units_per_stripe, uint64_t s0, uint64_t n_units,
                                                  uint32_t *sink) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t * UPT < n_units; t += stride) {
#pragma unroll
    for (int q = 0; q < UPT; ++q) {
      // unit index: the UPT units of one thread are blockDim.x units apart (coalesced per warp)
      const uint64_t u = (t / blockDim.x) * blockDim.x * UPT + q * blockDim.x + (t % blockDim.x);
      if (u >= n_units) break;
      const uint64_t s = s0 + u / units_per_stripe, c = (u % units_per_stripe) * 32;
      uint8_t *sp = base + s * stripe_stride + c;
      uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int b = 0; b < R; ++b) {
        uint32_t x[8];
        ldg_v8(sp + b * B, x);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] ^= x[i];
      }
      if (W == 0) {
        uint32_t v = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) v ^= acc[i];
        if (v == 0x9E3779B9u) sink[0] = v;  // keeps the loads alive; practically never taken
      }
#pragma unroll
      for (int w = 0; w < W; ++w) {
        uint32_t y[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) y[i] = acc[i] ^ (uint32_t)w;
        stg_v8(sp + (R + w) * B, y);
      }
    }
  }
}

struct Shape {
  const char *name;
  int per_stripe;   // 1: one launch per stripe (the codec's decode chain shape); 0: one launch
  int upt;          // units per thread
  int ctas_per_sm;  // one launch: 0 = a grid covering every unit once, else a persistent grid
};

template <int R, int W>
static int run_mix(const char *tag, uint8_t *base, int S, int n, uint64_t B, int sm_count, uint32_t *sink) {
  const uint64_t stripe_stride = (uint64_t)n * B, ups = B / 32;
  const Shape shapes[] = {{"per_stripe_upt1", 1, 1, 0},          {"per_stripe_upt2", 1, 2, 0},
                          {"one_launch_full_grid_upt1", 0, 1, 0}, {"one_launch_full_grid_upt2", 0, 2, 0},
                          {"one_launch_persistent4", 0, 2, 4},    {"one_launch_persistent8", 0, 2, 8},
                          {"one_launch_persistent16", 0, 2, 16}};
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  for (const Shape &sh : shapes) {
    auto launch = [&]() {
      if (sh.per_stripe) {
        const uint64_t threads = (ups + sh.upt - 1) / sh.upt;
        const unsigned grid = (unsigned)((threads + 127) / 128);
        for (int s = 0; s < S; ++s) {
          if (sh.upt == 1)
            mix_kernel<R, W, 1><<<grid, 128>>>(base, stripe_stride, B, ups, s, ups, sink);
          else
            mix_kernel<R, W, 2><<<grid, 128>>>(base, stripe_stride, B, ups, s, ups, sink);
        }
      } else {
        const uint64_t threads = (ups * S + sh.upt - 1) / sh.upt;
        const unsigned grid = sh.ctas_per_sm ? (unsigned)(sm_count * sh.ctas_per_sm) : (unsigned)((threads + 127) / 128);
        if (sh.upt == 1)
          mix_kernel<R, W, 1><<<grid, 128>>>(base, stripe_stride, B, ups, 0, ups * S, sink);
        else
          mix_kernel<R, W, 2><<<grid, 128>>>(base, stripe_stride, B, ups, 0, ups * S, sink);
      }
    };
    for (int i = 0; i < 3; ++i) launch();
    CK(cudaDeviceSynchronize());
    std::vector<float> ms;
    for (int i = 0; i < 10; ++i) {
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float t = 0;
      CK(cudaEventElapsedTime(&t, e0, e1));
      ms.push_back(t);
    }
    CK(cudaGetLastError());
    std::sort(ms.begin(), ms.end());
    const double bytes = (double)S * (R + W) * (double)B;
    printf("{\"mix\": \"%s\", \"read_blocks\": %d, \"write_blocks\": %d, \"stripes\": %d, \"block_bytes\": %llu, "
           "\"shape\": \"%s\", \"bytes\": %.0f, \"best_ms\": %.4f, \"median_ms\": %.4f, \"best_gbs\": %.1f, "
           "\"median_gbs\": %.1f}\n",
           tag, R, W, S, (unsigned long long)B, sh.name, bytes, ms[0], ms[ms.size() / 2], bytes / ms[0] / 1e6,
           bytes / ms[ms.size() / 2] / 1e6);
    fflush(stdout);
  }
  CK(cudaEventDestroy(e0));
  CK(cudaEventDestroy(e1));
  return 0;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // the largest batch below: C4, 256 stripes x 16 blocks x 8 MiB = 32 GiB
  const uint64_t bytes = 256ull * 16 * (8ull << 20);
  uint8_t *base = nullptr;
  uint32_t *sink = nullptr;
  CK(cudaMalloc(&base, bytes));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(base, 0x5A, bytes));
  int rc = 0;
  // C5 shape: RS(10,4) w8, 51 stripes x 16 MiB (encode reads 10 / writes 4; decode reads 10 / writes 4)
  rc |= run_mix<10, 4>("C5_10r4w", base, 51, 14, 16ull << 20, sms, sink);
  // C3 shape: RS(10,4), 512 x 4 MiB would be 28 GiB; same mix
  rc |= run_mix<10, 4>("C3_10r4w", base, 512, 14, 4ull << 20, sms, sink);
  // C4 shape: RS(12,4) w16, 256 x 8 MiB (encode 12 / 4; decode 12 / 4)
  rc |= run_mix<12, 4>("C4_12r4w", base, 256, 16, 8ull << 20, sms, sink);
  // reference points: 1:1 (the copy peak's mix), read-only, write-only
  rc |= run_mix<1, 1>("copy_1r1w", base, 256, 2, 32ull << 20, sms, sink);
  rc |= run_mix<14, 0>("read_only_14r", base, 51, 14, 16ull << 20, sms, sink);
  rc |= run_mix<0, 14>("write_only_14w", base, 51, 14, 16ull << 20, sms, sink);
  CK(cudaFree(base));
  CK(cudaFree(sink));
  return rc;
}
