// Pipe-rate microbenchmark for sm_100a: integer ALU ops (LOP3/SHF/PRMT), FMA-pipe
// integer ops (IMAD shl / IMAD.HI), LDS bandwidth, and HBM streaming (LDG.128/256).
// Used once to size the GF inner loop. Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 12;  // independent chains per thread

__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
__device__ __forceinline__ uint32_t shfr(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("shf.r.clamp.b32 %0, %1, %2, 5;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t imadshl(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("mad.lo.u32 %0, %1, 16, %2;" : "=r"(r) : "r"(a), "r"(b)); return r;
}
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
  uint32_t r; asm volatile("mul.hi.u32 %0, %1, 268435456;" : "=r"(r) : "r"(a)); return r ^ 0 * b;
}

// right shift by S as the high word of a 32x32->64 product with a multiplier ptxas cannot see
// (a kernel argument): IMAD.WIDE.U32 on the FMA pipe instead of SHF.R on the ALU pipe
__device__ __forceinline__ uint32_t mulwide_hi(uint32_t a, uint32_t mul) {
  uint64_t r; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(mul)); return (uint32_t)(r >> 32);
}
__device__ __forceinline__ uint32_t mulhi_reg(uint32_t a, uint32_t mul) {
  uint32_t r; asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(mul)); return r;
}

template <int OP>
__global__ void pipe_kernel(uint32_t *out, long long *cyc, uint32_t seed, uint32_t mul) {
  uint32_t x[CH], y = seed ^ threadIdx.x, z = seed * 3u + blockIdx.x;
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = seed + c * 77u + threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) x[c] = lop3(x[c], y, z);
      if (OP == 1) x[c] = shfr(x[c], y);
      if (OP == 2) x[c] = prmt(x[c], y);
      if (OP == 3) x[c] = imadshl(x[c], y);
      if (OP == 4) x[c] = mulhi(x[c], y);
      if (OP == 5) { x[c] = (c & 1) ? imadshl(x[c], y) : lop3(x[c], y, z); }  // half FMA, half ALU
      if (OP == 6) { x[c] = lop3(x[c], y, z); x[c] = imadshl(x[c], z); }       // 1:1 dependent
      if (OP == 8) x[c] = mulwide_hi(x[c], mul);
      if (OP == 9) x[c] = mulhi_reg(x[c], mul);
      if (OP == 10) { x[c] = (c & 1) ? mulwide_hi(x[c], mul) : lop3(x[c], y, z); }  // 1:1 indep
      if (OP == 11) { x[c] = (c % 3 == 2) ? mulwide_hi(x[c], mul) : lop3(x[c], y, z); }  // 2 ALU : 1
      if (OP == 12) { x[c] = (c % 3 == 2) ? mulhi(x[c], y) : lop3(x[c], y, z); }  // 2 ALU : 1 IMAD.HI
      if (OP == 13) { x[c] = (c & 3) == 3 ? mulwide_hi(x[c], mul) : ((c & 3) == 2 ? imadshl(x[c], y) : lop3(x[c], y, z)); }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void lds_kernel(uint32_t *out, long long *cyc) {
  __shared__ uint32_t tab[32 * 32];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = i * 2654435761u;
  __syncthreads();
  uint32_t idx = threadIdx.x & 31, acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint32_t v = tab[(idx + c * 32) & 1023];
      acc ^= v; idx = (idx + (v & 32)) & 1023;  // lane stays in its own bank
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void copy128(const uint4 *__restrict__ a, uint4 *__restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 3 * st < n; i += 4 * st) {
    uint4 v0, v1, v2, v3;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v0.x), "=r"(v0.y), "=r"(v0.z), "=r"(v0.w) : "l"(a + i));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v1.x), "=r"(v1.y), "=r"(v1.z), "=r"(v1.w) : "l"(a + i + st));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v2.x), "=r"(v2.y), "=r"(v2.z), "=r"(v2.w) : "l"(a + i + 2 * st));
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v3.x), "=r"(v3.y), "=r"(v3.z), "=r"(v3.w) : "l"(a + i + 3 * st));
    b[i] = v0; b[i + st] = v1; b[i + 2 * st] = v2; b[i + 3 * st] = v3;
  }
  for (; i < n; i += st) b[i] = a[i];
}

__global__ void read256(const uint4 *__restrict__ a, uint32_t *out, size_t n2) {  // n2 = #32B units
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (; i < n2; i += st) {
    uint32_t r[8];
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(a + 2 * i));
#pragma unroll
    for (int c = 0; c < 8; ++c) acc ^= r[c];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("gpu %s sms %d l2 %d clk_khz %d smem/sm %zu\n", p.name, p.multiProcessorCount, p.l2CacheSize, clk, p.sharedMemPerMultiprocessor);
  const int SM = p.multiProcessorCount, TPB = 1024;
  uint32_t *out; long long *cyc; CK(cudaMalloc(&out, SM * 4 * TPB * 4)); CK(cudaMalloc(&cyc, SM * 4 * 8));
  long long hc[1024];
  const char *names[] = {"lop3", "shf", "prmt", "imad.shl", "mul.hi", "lop3+imad(1:1 indep)", "lop3->imad dep", "lds",
                         "mul.wide hi (reg)", "mul.hi (reg)", "lop3+mul.wide(1:1)", "lop3+mul.wide(2:1)",
                         "lop3+mul.hi(2:1)", "lop3:shl:mulwide 2:1:1"};
  auto run = [&](int op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: pipe_kernel<0><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 1: pipe_kernel<1><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 2: pipe_kernel<2><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 3: pipe_kernel<3><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 4: pipe_kernel<4><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 5: pipe_kernel<5><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 6: pipe_kernel<6><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 7: lds_kernel<<<SM, TPB>>>(out, cyc); break;
        case 8: pipe_kernel<8><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 9: pipe_kernel<9><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 10: pipe_kernel<10><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 11: pipe_kernel<11><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 12: pipe_kernel<12><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
        case 13: pipe_kernel<13><<<SM, TPB>>>(out, cyc, 7, 1u << 28); break;
      }
    }
    cudaDeviceSynchronize();
    cudaMemcpy(hc, cyc, SM * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < SM; ++i) mx = hc[i] > mx ? hc[i] : mx;
    double ops = (double)TPB * ITERS * CH * (op == 6 ? 2 : 1);
    printf("%-24s %.1f thread-ops/clk/SM (max block cycles %.0f)\n", op == 7 ? "lds.32" : names[op], ops / mx, mx);
  };
  for (int op = 0; op <= 13; ++op) run(op);

  // HBM streaming
  size_t bytes = (size_t)4 << 30; void *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 1, bytes); cudaMemset(b, 0, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int g : {SM * 2, SM * 4, SM * 8, SM * 16}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); copy128<<<g, 512>>>((const uint4 *)a, (uint4 *)b, bytes / 16); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("copy128 grid %d x512: %.1f GB/s (r+w)\n", g, 2.0 * bytes / best / 1e6);
  }
  for (int g : {SM * 4, SM * 8, SM * 16}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); read256<<<g, 512>>>((const uint4 *)a, out, bytes / 32); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("read256 grid %d x512: %.1f GB/s (read)\n", g, 1.0 * bytes / best / 1e6);
  }
  {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
    }
    printf("cudaMemcpy d2d: %.1f GB/s (r+w)\n", 2.0 * bytes / best / 1e6);
  }
  CK(cudaGetLastError());
  return 0;
}
