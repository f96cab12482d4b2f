// rs_kernels.cuh -- types shared by the host planner (plan.cpp) and the sm_100a
// kernels (rs_kernels.cu).  See DESIGN.md "Kernels" for the data layout in HBM.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace rsb {

constexpr int kMaxN = 255;
constexpr int kMaxM = 32;

// Where block b of stripe s lives.  Strided mode: base + s*stripe_stride +
// b*block_stride.  Pointer mode (ptrs != nullptr): ptrs[s*n + b] (device array).
struct Layout {
  uint8_t *base;
  uint64_t stripe_stride, block_stride;
  const uint64_t *ptrs;
  int n;
  __host__ __device__ __forceinline__ uint8_t *block(uint64_t s, int b) const {
    return ptrs ? reinterpret_cast<uint8_t *>(ptrs[s * (uint64_t)n + b])
                : base + s * stripe_stride + (uint64_t)b * block_stride;
  }
};

// ---- generic split-nibble kernel ------------------------------------------
// out_blk[r] = sum_s M[r][s] * in_blk[s] per column, M given as packed nibble
// tables.  w=8: for output group g (4 outputs per 32-bit word) and input s,
//   tab32[(g*n_in + s)*32 + h*16 + v] = pack_r( M[4g+r][s] * (v << 4h) ),  h in {0,1}.
// w=16: tab64[(g*n_in + s)*64 + h*16 + v] = pack_r( M[4g+r][s] * (v << 4h) ) as
//   4 x 16-bit lanes, h in {0..3}.
struct GenericPat {
  int32_t n_in, n_out;
  uint32_t table_off;  // in bytes from GenericArgs::tables
  uint32_t pad;
  uint8_t in_blk[kMaxN + 1];
  uint8_t out_blk[kMaxM];
};

struct GenericArgs {
  Layout L;
  const GenericPat *pats;   // device
  const int32_t *pat_idx;   // device, per stripe (-1 = skip); nullptr = every stripe uses pats[0]
  const uint8_t *tables;    // device
  uint64_t n_stripes;
  uint64_t col_begin, col_end;  // byte range inside each block to process
  uint64_t chunk_bytes;         // bytes of that range per CTA (multiple of 16*blockDim)
  uint32_t ctas_per_group;      // CTAs per (stripe, output group)
  uint32_t n_groups;            // output groups of 4 (max over patterns)
  uint32_t vec_ok;              // all block addresses 16-byte aligned
  uint32_t smem_bytes;          // dynamic smem = table bytes per group
  unsigned *flags;              // non-null: verify mode (outputs are syndromes; flags[s] |= 1 if any != 0)
};

// ---- bit-sliced kernels (compile-time networks) ---------------------------
// One "unit" = 32 columns = 32*w/8 bytes of each block.
// Decode pattern record: W = V_E^{-1} * H_par[0:t,:] (t x m) as nibble tables
// over the m inputs Delta_i = received parity_i ^ encode(surviving data)_i
// (see DESIGN.md "Decode = encode + t x m solve").
//   w=8:  wtab32[i*32 + h*16 + v] = pack_e( W[e][i] * (v << 4h) ), 4 bytes
//   w=16: wtab64[i*64 + h*16 + v] = pack_e( W[e][i] * (v << 4h) ), 4 x 16 bit
struct SlicedPat {
  uint32_t erased_mask[8];  // bit b: API block b erased
  int32_t t;
  uint8_t out_blk[4];       // erased blocks, row order of W
  uint32_t table_off;       // bytes from SlicedArgs::tables
  uint32_t pad;
};

struct SlicedArgs {
  Layout L;
  const SlicedPat *pats;   // decode only
  const int32_t *pat_idx;  // decode only; per stripe, -1 = skip
  const uint8_t *tables;   // decode only
  uint64_t n_stripes;
  uint64_t units_per_stripe;
  uint32_t units_per_cta;
  uint32_t ctas_per_stripe;
};

// Launchers (rs_kernels.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_generic(int w, const GenericArgs &a, cudaStream_t st);
bool sliced_available(int k, int m, int w, uint32_t poly);
cudaError_t launch_sliced(int k, int m, int w, uint32_t poly, bool decode, const SlicedArgs &a,
                          cudaStream_t st);
// The paper's optimisation study (polyrs_ablation.cu): per-column two-step decode with
// Opt1/Opt2/Opt3 selected by opt_mask bits 0/1/2; GF(2^8), k+m <= 32, 1 <= t <= 8.
cudaError_t launch_polyrs_ablation(const Layout &L, uint64_t n_stripes, uint64_t block_bytes, int k, int m,
                                   const int *erased, int t, const uint8_t *dev_consts, int opt_mask,
                                   int sm_count, cudaStream_t st);
uint64_t launches_total();
void count_launch();

}  // namespace rsb
