// polyrs_ablation.cu -- the paper's optimisation study on the GPU.
//
// A per-column, table-driven implementation of the two-step polynomial decode exactly as
// the paper describes HDFS-RAID's code, with each of the paper's optimisations switchable:
//   Opt1: the alpha powers alpha^{j*pos} are precomputed once (a table) instead of
//                 being recomputed iteratively for every vector of survivors;
//   Opt2: Step 1 skips the erased positions instead of multiplying their zeros;
//   Opt3: the Vandermonde matrix V_E is inverted once and each vector is
//                 multiplied by V_E^{-1}, instead of a Gaussian elimination per vector;
//   Opt4: region-level multiply-XOR -- on the GPU every thread already works on
//                 its own column with coalesced accesses across the warp, so Opt4 has no
//                 separate switch here.
// Encoding uses the same procedure with the m parity positions as the erasures (the
// symmetric use).  GF(2^8) only (the paper's field), log/exp tables in
// shared memory ("tables are pre-computed and maintained in memory").
//
// This is a baseline for measurement, not the product path: the bit-sliced kernels
// (rs_kernels.cu, jit.cpp) compute the same bytes.
#include <cstdint>

#include "rs_kernels.cuh"

namespace rsb {

namespace {

constexpr int kAblMaxN = 32, kAblMaxT = 8;

struct __align__(16) AblArgs {
  Layout L;
  uint64_t n_stripes, block_bytes;
  int k, m, t;
  int pos_e[kAblMaxT];   // polynomial positions of the erased blocks
  int blk_e[kAblMaxT];   // their API indices
  uint32_t erased_mask;  // API indices
  const uint8_t *consts; // device: exp[512], log[256] (as uint8 + high bit), apow[t][n], vinv[t][t]
};

__device__ __forceinline__ uint32_t gmul(const uint8_t *ex, const uint8_t *lg, uint32_t a, uint32_t b) {
  return (a && b) ? ex[(uint32_t)lg[a] + (uint32_t)lg[b]] : 0u;
}

template <int OPT>
__global__ void __launch_bounds__(256) polyrs_kernel(const AblArgs a) {
  constexpr bool O1 = OPT & 1, O2 = OPT & 2, O3 = OPT & 4;
  __shared__ uint8_t ex[512], lg[256], apow[kAblMaxT * kAblMaxN], vinv[kAblMaxT * kAblMaxT];
  const int n = a.k + a.m, t = a.t;
  for (int i = threadIdx.x; i < 512; i += blockDim.x) ex[i] = a.consts[i];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) lg[i] = a.consts[512 + i];
  for (int i = threadIdx.x; i < t * n; i += blockDim.x) apow[i] = a.consts[768 + i];
  for (int i = threadIdx.x; i < t * t; i += blockDim.x) vinv[i] = a.consts[768 + kAblMaxT * kAblMaxN + i];
  __syncthreads();

  const uint64_t total = a.n_stripes * a.block_bytes;
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
       g += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = g / a.block_bytes, col = g % a.block_bytes;
    // the codeword in polynomial-position order (pos 0..m-1 parity, m..n-1 data)
    uint8_t c[kAblMaxN];
    for (int p = 0; p < n; ++p) {
      const int b = p < a.m ? a.k + p : p - a.m;
      c[p] = ((a.erased_mask >> b) & 1u) ? 0 : a.L.block(s, b)[col];
    }
    // Step 1: D_j = sum over positions of c_p alpha^{j p}
    uint8_t D[kAblMaxT];
    for (int j = 0; j < t; ++j) {
      uint32_t acc = 0;
      if (O1) {
        for (int p = 0; p < n; ++p) {
          if (O2 && ((a.erased_mask >> (p < a.m ? a.k + p : p - a.m)) & 1u)) continue;
          acc ^= gmul(ex, lg, c[p], apow[j * n + p]);
        }
      } else {
        uint32_t aj = 1;  // alpha^j, recomputed for this vector
        for (int i = 0; i < j; ++i) aj = gmul(ex, lg, aj, 2u);
        uint32_t pw = 1;  // alpha^{j p}, advanced iteratively
        for (int p = 0; p < n; ++p) {
          const bool er = (a.erased_mask >> (p < a.m ? a.k + p : p - a.m)) & 1u;
          if (!(O2 && er)) acc ^= gmul(ex, lg, c[p], pw);
          pw = gmul(ex, lg, pw, aj);
        }
      }
      D[j] = (uint8_t)acc;
    }
    // Step 2: solve V_E y = D
    uint8_t y[kAblMaxT];
    if (O3) {
      for (int e = 0; e < t; ++e) {
        uint32_t acc = 0;
        for (int j = 0; j < t; ++j) acc ^= gmul(ex, lg, vinv[e * t + j], D[j]);
        y[e] = (uint8_t)acc;
      }
    } else {
      // Gauss-Jordan on [V | D] for this vector, V rebuilt here (from the Opt1 table if on)
      uint8_t A[kAblMaxT][kAblMaxT + 1];
      for (int j = 0; j < t; ++j) {
        for (int e = 0; e < t; ++e) {
          uint32_t v;
          if (O1) {
            v = apow[j * n + a.pos_e[e]];
          } else {
            uint32_t x = 1, xe = 1;
            for (int i = 0; i < a.pos_e[e]; ++i) xe = gmul(ex, lg, xe, 2u);  // alpha^{pos_e}
            for (int i = 0; i < j; ++i) x = gmul(ex, lg, x, xe);
            v = x;
          }
          A[j][e] = (uint8_t)v;
        }
        A[j][t] = D[j];
      }
      for (int col2 = 0; col2 < t; ++col2) {
        int piv = col2;
        while (piv < t && A[piv][col2] == 0) ++piv;
        if (piv == t) break;  // singular: cannot happen for distinct positions (G11)
        if (piv != col2)
          for (int x = 0; x <= t; ++x) {
            const uint8_t tmp = A[piv][x];
            A[piv][x] = A[col2][x];
            A[col2][x] = tmp;
          }
        const uint32_t inv = ex[255 - lg[A[col2][col2]]];
        for (int x = 0; x <= t; ++x) A[col2][x] = (uint8_t)gmul(ex, lg, A[col2][x], inv);
        for (int r = 0; r < t; ++r) {
          const uint32_t f = r == col2 ? 0u : A[r][col2];
          if (!f) continue;
          for (int x = 0; x <= t; ++x) A[r][x] ^= (uint8_t)gmul(ex, lg, f, A[col2][x]);
        }
      }
      for (int e = 0; e < t; ++e) y[e] = A[e][t];
    }
    for (int e = 0; e < t; ++e) a.L.block(s, a.blk_e[e])[col] = y[e];
  }
}

}  // namespace

// consts: exp[512] (exp[i] = alpha^(i mod 255)), log[256] (log[0] unused), apow[t][n]
// (alpha^{j * pos}, position order), vinv[t][t]; layout documented in AblArgs.
cudaError_t launch_polyrs_ablation(const Layout &L, uint64_t n_stripes, uint64_t block_bytes, int k, int m,
                                   const int *erased, int t, const uint8_t *dev_consts, int opt_mask,
                                   int sm_count, cudaStream_t st) {
  if (k + m > kAblMaxN || t > kAblMaxT || t < 1) return cudaErrorInvalidValue;
  AblArgs a{};
  a.L = L;
  a.n_stripes = n_stripes;
  a.block_bytes = block_bytes;
  a.k = k;
  a.m = m;
  a.t = t;
  for (int e = 0; e < t; ++e) {
    a.blk_e[e] = erased[e];
    a.pos_e[e] = erased[e] < k ? m + erased[e] : erased[e] - k;
    a.erased_mask |= 1u << erased[e];
  }
  a.consts = dev_consts;
  const uint64_t total = n_stripes * block_bytes;
  uint64_t grid = (total + 255) / 256;
  grid = grid < (uint64_t)sm_count * 16 ? grid : (uint64_t)sm_count * 16;
  if (grid == 0) return cudaSuccess;
  count_launch();
  switch (opt_mask & 7) {
    case 0: polyrs_kernel<0><<<(unsigned)grid, 256, 0, st>>>(a); break;
    case 1: polyrs_kernel<1><<<(unsigned)grid, 256, 0, st>>>(a); break;
    case 2: polyrs_kernel<2><<<(unsigned)grid, 256, 0, st>>>(a); break;
    case 3: polyrs_kernel<3><<<(unsigned)grid, 256, 0, st>>>(a); break;
    case 4: polyrs_kernel<4><<<(unsigned)grid, 256, 0, st>>>(a); break;
    case 5: polyrs_kernel<5><<<(unsigned)grid, 256, 0, st>>>(a); break;
    case 6: polyrs_kernel<6><<<(unsigned)grid, 256, 0, st>>>(a); break;
    default: polyrs_kernel<7><<<(unsigned)grid, 256, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace rsb
