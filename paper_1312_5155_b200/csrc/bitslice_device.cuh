// bitslice_device.cuh -- device helpers shared by the compiled kernels (rs_kernels.cu)
// and the per-pattern kernels generated at run time (jit.cpp, NVRTC).  Self-contained:
// NVRTC compiles it without any system header.
#pragma once
#ifdef __CUDACC_RTC__
typedef unsigned char uint8_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#else
#include <cstdint>
#endif

namespace rsb {

// ---------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldg_v4(const void *p) {
  uint4 r;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg_v4(void *p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// 256-bit accesses need PTX ISA 8.8 (CUDA 12.9); an older NVRTC gets RS_NO_V8 and two v4s.
#ifdef RS_NO_V8
__device__ __forceinline__ void ldg_v8(const void *p, uint32_t *r) {
  const uint4 a = ldg_v4(p), b = ldg_v4(static_cast<const uint8_t *>(p) + 16);
  r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
}
__device__ __forceinline__ void stg_v8(void *p, const uint32_t *r) {
  stg_v4(p, make_uint4(r[0], r[1], r[2], r[3]));
  stg_v4(static_cast<uint8_t *>(p) + 16, make_uint4(r[4], r[5], r[6], r[7]));
}
#else
__device__ __forceinline__ void ldg_v8(const void *p, uint32_t *r) {
  asm("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "l"(p));
}
__device__ __forceinline__ void stg_v8(void *p, const uint32_t *r) {
  asm volatile("st.global.L1::no_allocate.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                  "r"(r[7])
               : "memory");
}
#endif

// ---------------------------------------------------------------------------
// bit-plane transposes (delta swaps; each is an involution, so the same
// routine goes bytes -> planes and planes -> bytes)
// ---------------------------------------------------------------------------
// Shifts run on the FMA pipe (IMAD.SHL / IMAD.HI): on B200 the ALU pipe
// (LOP3/SHF/PRMT, 64 lanes/clk/SM) is the scarce one, the FMA pipe is mostly idle
// (profiles/r01_microbench_pipes.log: IMAD 128/clk/SM, mul.hi 32/clk/SM).
template <int S>
__device__ __forceinline__ uint32_t shl_fma(uint32_t v) {
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, 0;" : "=r"(r) : "r"(v), "n"(1u << S));
  return r;
}
template <int S>
__device__ __forceinline__ uint32_t shr_fma(uint32_t v) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(v), "n"(1u << (32 - S)));
  return r;
}
// MASK ? a : b in ONE LOP3 (ptxas otherwise splits a&M | b&~M into two).
template <uint32_t MASK>
__device__ __forceinline__ uint32_t bitsel(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(r) : "r"(a), "r"(b), "n"(MASK));
  return r;
}

// Swap in-word bit S-position (mask ~M) of a with word-index bit of c.
template <int S, uint32_t MASK>
__device__ __forceinline__ void delta_swap(uint32_t &a, uint32_t &c) {
  const uint32_t na = bitsel<MASK>(a, shl_fma<S>(c));
  const uint32_t nc = bitsel<MASK>(shr_fma<S>(a), c);
  a = na;
  c = nc;
}

// 8 words (32 columns of bytes; word i = columns 4i..4i+3) <-> 8 planes
// (plane b = bit b of the 32 columns; column 4i+r at plane bit 8r+i).
__device__ __forceinline__ void transpose8(uint32_t *x) {
#pragma unroll
  for (int i = 0; i < 4; ++i) delta_swap<4, 0x0F0F0F0Fu>(x[i], x[i + 4]);
#pragma unroll
  for (int i = 0; i < 8; i += 4) {
    delta_swap<2, 0x33333333u>(x[i], x[i + 2]);
    delta_swap<2, 0x33333333u>(x[i + 1], x[i + 3]);
  }
#pragma unroll
  for (int i = 0; i < 8; i += 2) delta_swap<1, 0x55555555u>(x[i], x[i + 1]);
}

// The same swap with plain shifts: ptxas puts the left shift on the FMA pipe (IMAD.SHL) and the
// right one on the ALU pipe (SHF.R) instead of the quarter-rate IMAD.HI.  The w16 kernels
// (ALU-heavier, power-capped) run faster this way -- C4 encode 91-92% vs 88-90% of the copy
// peak -- while the w8 decode chains lose 1-4% (profiles/r01r_shift_pipes.log).
template <int S, uint32_t MASK>
__device__ __forceinline__ void delta_swap_shf(uint32_t &a, uint32_t &c) {
  const uint32_t na = bitsel<MASK>(a, c << S);
  const uint32_t nc = bitsel<MASK>(a >> S, c);
  a = na;
  c = nc;
}

// 16 words (32 columns of LE uint16; word i = columns 2i, 2i+1) <-> 16 planes
// (plane b = bit b; column 2i+r at plane bit 16r+i).  The byte stage uses PRMT.
__device__ __forceinline__ void transpose16(uint32_t *x) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t a = x[i], c = x[i + 8];
    x[i] = __byte_perm(a, c, 0x6240);
    x[i + 8] = __byte_perm(a, c, 0x7351);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if ((i & 4) == 0) delta_swap_shf<4, 0x0F0F0F0Fu>(x[i], x[i + 4]);
#pragma unroll
  for (int i = 0; i < 16; ++i)
    if ((i & 2) == 0) delta_swap_shf<2, 0x33333333u>(x[i], x[i + 2]);
#pragma unroll
  for (int i = 0; i < 16; i += 2) delta_swap_shf<1, 0x55555555u>(x[i], x[i + 1]);
}

template <int W>
__device__ __forceinline__ void transposeW(uint32_t *x) {
  if (W == 8) transpose8(x);
  else transpose16(x);
}

// ---------------------------------------------------------------------------
// Horner steps on bit-planes (syndrome form): S <- S * alpha^J (+ c).
// Multiplication by the constant alpha^J is GF(2)-linear: plane o of the product is
// the XOR of the planes b with bit o of alpha^J * 2^b set.  The matrix is evaluated
// at compile time from (W, POLY); after unrolling only the XORs remain (alpha^J is
// sparse for small J: 3 extra XORs per power for 0x11D and 0x1100B).
// ---------------------------------------------------------------------------
template <int W, uint32_t POLY>
struct GFc {
  __host__ __device__ static constexpr uint32_t mul(uint32_t a, uint32_t b) {
    uint32_t r = 0;
    for (int i = 0; i < W; ++i) {
      if ((b >> i) & 1u) r ^= a;
      a <<= 1;
      if ((a >> W) & 1u) a ^= POLY;
    }
    return r;
  }
  __host__ __device__ static constexpr uint32_t alpha_pow(int e) {
    uint32_t r = 1;
    for (int i = 0; i < e; ++i) r = mul(r, 2u);
    return r;
  }
  // bit o of alpha^J * 2^b
  __host__ __device__ static constexpr bool bit(int J, int b, int o) { return (mul(alpha_pow(J), 1u << b) >> o) & 1u; }
};

template <int W, uint32_t POLY, int J, bool ADD>
__device__ __forceinline__ void horner_step(uint32_t *s, const uint32_t *c) {
  uint32_t o[W];
#pragma unroll
  for (int i = 0; i < W; ++i) o[i] = s[i];
#pragma unroll
  for (int ob = 0; ob < W; ++ob) {
    uint32_t acc = ADD ? c[ob] : 0u;
#pragma unroll
    for (int b = 0; b < W; ++b)
      if (GFc<W, POLY>::bit(J, b, ob)) acc ^= o[b];
    s[ob] = acc;
  }
}

// A unit is 32 columns: 32 bytes of a block (w = 8) or 64 (w = 16, two 32-byte halves).  The
// w = 16 halves are `h2` bytes apart: 32 (contiguous) or, for a full warp, 1024 -- lane l then
// owns bytes [32 l, 32 l + 32) and [1024 + 32 l, ...) of the warp's 2 KiB, so that each 256-bit
// load / store instruction of the warp covers 1 KiB contiguously (whole 128-byte lines) instead
// of every other 32-byte sector of 2 KiB (unit_offset() below).
template <int W>
__device__ __forceinline__ void load_unit(const uint8_t *p, uint32_t *x, uint32_t h2 = 32) {
  ldg_v8(p, x);
  if (W == 16) ldg_v8(p + h2, x + 8);
}
// y ^= the raw bytes of a unit (an input added unchanged to one output, after transpose back)
template <int W>
__device__ __forceinline__ void xor_unit(uint32_t *y, const uint8_t *p, uint32_t h2 = 32) {
  uint32_t r[W];
  load_unit<W>(p, r, h2);
#pragma unroll
  for (int q = 0; q < W; ++q) y[q] ^= r[q];
}
template <int W>
__device__ __forceinline__ void store_unit(uint8_t *p, const uint32_t *x, uint32_t h2 = 32) {
  stg_v8(p, x);
  if (W == 16) stg_v8(p + h2, x + 8);
}
// Byte offset of unit u in its block and the distance h2 of its second half (w = 16).  Units
// of a warp are consecutive and start at a multiple of 32 (CTA ranges are multiples of 128);
// a warp whose 32 units all lie below u_end uses the 1 KiB-interleaved halves, a partial one
// (the end of a stripe) the contiguous layout.  Every block of a stripe uses the same map,
// so column c's symbols still sit at the same offset in each block.
// Measured (profiles/r02f_w16_layout_ab.log, C4): the compiled w16 encoder runs 1% faster
// interleaved, the per-pattern JIT decoders 0-1.2% faster contiguous -- so the compiled
// kernels interleave (IL = true) and the generated ones do not.  (Any kernel may map columns
// to threads its own way: columns are independent codewords.)
template <int W, bool IL = true>
__device__ __forceinline__ uint64_t unit_offset(uint64_t u, uint64_t u_end, uint32_t &h2) {
  if (W != 16 || !IL) {
    h2 = 32;
    return u * (uint64_t)(4 * W);
  }
  const uint64_t lane = u & 31ull;
  const bool full = (u - lane) + 32ull <= u_end;
  h2 = full ? 1024u : 32u;
  return full ? u * 64ull - lane * 32ull : u * 64ull;
}

}  // namespace rsb
