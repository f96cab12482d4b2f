// rs_kernels.cu -- sm_100a kernels of the polynomial Reed-Solomon hot path.
//
// What they compute (PAPER.md, arXiv 1312.5155):
//   encode: parity p(x) = d(x) x^m mod g(x), g = prod_{i<m}(x + alpha^i)
//           (Eq. 1-2), per column of each stripe;
//   decode: the erased symbols of each column from the survivors (two-step
//           decode).
//
// Compiled kernel families (the per-pattern decoders are generated at
// run time by jit.cpp):
//   * sliced_kernel<K,M,W,POLY,DECODE>: each thread owns 32 columns; it loads
//     32*W/8 bytes of each block with 256-bit loads, transposes them into W
//     bit-planes (three/four delta swaps) and transposes the results back.
//     w8 encode: the compile-time GF(2) network RsNet (parity map of g, in
//     bit-matrix form; CSE for 3-input gates).  w16 encode: the syndrome
//     form -- Horner over the data blocks with step alpha^j, then the
//     network RsQNet = Vp^{-1} diag(alpha^{jm}) (the decoder used to encode).
//     DECODE (the table fallback): re-encode the surviving data (erased data
//     zeroed), XOR the received parity to get Delta, and solve the t erased
//     symbols with the runtime t x m matrix W = V_E^{-1} H_par[0:t,:] through
//     split-nibble tables in shared memory.
//   * generic_kernel<W, VERIFY>: out_r = sum_s M[r][s] in_s with runtime split-nibble
//     tables (any k, m, any erasure pattern, any alignment, ragged tails); VERIFY
//     ORs the outputs (syndromes) into a per-stripe flag instead of storing them.
// Every HBM byte of a stripe is read once or written once: (k+m)*B per pass.
#include <atomic>
#include <cstdio>

#include "bitslice_device.cuh"
#include "rs_kernels.cuh"
#include "rs_networks.cuh"

namespace rsb {

#ifndef RS_W16_HUNROLL
#define RS_W16_HUNROLL 3  // Horner over the data blocks unrolled by 3 (0: fully; C4 encode 86% -> 88.5%:
                          // a 40 KB fully unrolled loop body stalls on instruction fetch)
#endif

static std::atomic<uint64_t> g_launches{0};
uint64_t launches_total() { return g_launches.load(); }
void count_launch() { g_launches.fetch_add(1); }

// Addresses of the blocks of one stripe, computed per access: strided (base + b *
// block_stride) or pointer mode (the stripe's row of the pointer array).  Two types, so
// that the choice is made once per kernel, not per load (a branch between the loads of an
// unrolled loop body keeps ptxas from hoisting them: C4 encode 0.93 -> 0.78 of the copy peak).
struct StridedBlocks {
  uint8_t *base;
  uint64_t block_stride;
  __device__ __forceinline__ uint8_t *operator[](int b) const { return base + (uint64_t)b * block_stride; }
};
struct PointerBlocks {
  const uint64_t *ptrs;
  __device__ __forceinline__ uint8_t *operator[](int b) const { return reinterpret_cast<uint8_t *>(ptrs[b]); }
};

// The same from an array of the stripe's K+M block pointers (held in registers when every
// index is a compile-time constant, as in the w8 networks).
template <int N>
struct BlockArray {
  uint8_t *p[N];
  __device__ __forceinline__ uint8_t *operator[](int b) const { return p[b]; }
};

// Load + transpose the data blocks of CSE group G and run its sub-network
// (group 0 assigns y, later groups accumulate).  Erased data blocks (decode)
// are not read: their planes are zero.
template <int K, int M, int W, uint32_t POLY, bool DECODE, int G, class BLK>
__device__ __forceinline__ void net_groups(const BLK &blk, uint64_t off, uint32_t h2, uint32_t emask,
                                           uint32_t (&y)[M * W]) {
  using Grp = RsNetGroup<K, M, W, POLY, G>;
  constexpr int J0 = Grp::kFirstBlock, NB = Grp::kBlocks;
  uint32_t x[NB * W];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    if (DECODE && ((emask >> (J0 + j)) & 1u)) {
#pragma unroll
      for (int q = 0; q < W; ++q) x[j * W + q] = 0;
    } else {
      load_unit<W>(blk[J0 + j] + off, &x[j * W], h2);
    }
  }
#pragma unroll
  for (int j = 0; j < NB; ++j) transposeW<W>(&x[j * W]);
  Grp::run(x, y);
  if constexpr (G + 1 < RsNet<K, M, W, POLY>::kGroups)
    net_groups<K, M, W, POLY, DECODE, G + 1>(blk, off, h2, emask, y);
}

// Syndrome-form encoder (w = 16 instances, RsQNet): H_j = Horner over the data
// blocks from the highest position x^{m+k-1} down to x^m with step alpha^j
// (P:237-241), one block in registers at a time, then y = Q H (Q = Vp^{-1}
// diag(alpha^{jm}), the symmetric use of the decoder).  Erased data blocks
// (decode) are not read: their planes are zero.
template <int K, int M, int W, uint32_t POLY, bool DECODE, int J>
__device__ __forceinline__ void horner_all(uint32_t (&h)[M * W], const uint32_t (&c)[W]) {
  horner_step<W, POLY, J, true>(&h[J * W], c);
  if constexpr (J + 1 < M) horner_all<K, M, W, POLY, DECODE, J + 1>(h, c);
}

constexpr int kHornerUnroll = RS_W16_HUNROLL > 0 ? RS_W16_HUNROLL : 1;

template <int K, int M, int W, uint32_t POLY, bool DECODE, class BLK>
__device__ __forceinline__ void horner_encode(const BLK &blk, uint64_t off, uint32_t h2, uint32_t emask,
                                              uint32_t (&y)[M * W]) {
  uint32_t h[M * W];
  {
    uint32_t c[W];
    if (DECODE && ((emask >> (K - 1)) & 1u)) {
#pragma unroll
      for (int q = 0; q < W; ++q) c[q] = 0;
    } else {
      load_unit<W>(blk[K - 1] + off, c, h2);
      transposeW<W>(c);
    }
#pragma unroll
    for (int i = 0; i < M * W; ++i) h[i] = c[i % W];
  }
#if RS_W16_HUNROLL
#pragma unroll kHornerUnroll
#else
#pragma unroll
#endif
  for (int jb = K - 2; jb >= 0; --jb) {
    uint32_t c[W];
    if (DECODE && ((emask >> jb) & 1u)) {
#pragma unroll
      for (int q = 0; q < W; ++q) c[q] = 0;
    } else {
      load_unit<W>(blk[jb] + off, c, h2);
      transposeW<W>(c);
    }
    horner_all<K, M, W, POLY, DECODE, 0>(h, c);
  }
  RsQNet<K, M, W, POLY>::run(h, y);
}

// Syndromes of the received word (w = 16 table decode, SURVEY App. B design C): S_j =
// sum_p c_p alpha^{j p} over ALL n positions, Horner from the top (x^{n-1} = data K-1) down
// to x^0 (parity 0) with step alpha^j (Step 1); erased positions (CTA-uniform
// bits of emask) are not read and enter as zero.  j < M.
template <int K, int M, int W, uint32_t POLY, class BLK>
__device__ __forceinline__ void horner_syndromes(const BLK &blk, uint64_t off, uint32_t h2, uint32_t emask,
                                                 uint32_t (&h)[M * W]) {
  {
    uint32_t c[W];
    if ((emask >> (K - 1)) & 1u) {
#pragma unroll
      for (int q = 0; q < W; ++q) c[q] = 0;
    } else {
      load_unit<W>(blk[K - 1] + off, c, h2);
      transposeW<W>(c);
    }
#pragma unroll
    for (int i = 0; i < M * W; ++i) h[i] = c[i % W];
  }
#pragma unroll kHornerUnroll
  for (int p = K + M - 2; p >= 0; --p) {  // position p: data p - M (p >= M), else parity p
    const int b = p >= M ? p - M : K + p;
    uint32_t c[W];
    if ((emask >> b) & 1u) {
#pragma unroll
      for (int q = 0; q < W; ++q) c[q] = 0;
    } else {
      load_unit<W>(blk[b] + off, c, h2);
      transposeW<W>(c);
    }
    horner_all<K, M, W, POLY, true, 0>(h, c);
  }
}

template <int K, int M, int W, uint32_t POLY, bool DECODE, class BLK>
__device__ __forceinline__ void encode_planes(const BLK &blk, uint64_t off, uint32_t h2, uint32_t emask,
                                              uint32_t (&y)[M * W]) {
  if constexpr (RsQNet<K, M, W, POLY>::kHorner) horner_encode<K, M, W, POLY, DECODE>(blk, off, h2, emask, y);
  else net_groups<K, M, W, POLY, DECODE, 0>(blk, off, h2, emask, y);
}

// ---------------------------------------------------------------------------
// bit-sliced kernel
// ---------------------------------------------------------------------------
// Resident CTAs per SM (x 128 threads): the kernels hide HBM latency with warps, so
// occupancy matters more than registers.  Measured on B200 (profiles/r01b_occupancy_sweep.log):
// w8 at 4 CTAs/SM (<=128 regs, a few spilled bytes) reaches the copy roofline on RS(10,4)
// encode; w16 spills at 4 and runs best at 3.
#ifndef RS_W16_MINB
#define RS_W16_MINB 3
#endif
template <int W>
constexpr int sliced_min_blocks() { return W == 8 ? 4 : RS_W16_MINB; }

template <int K, int M, int W, uint32_t POLY, bool DECODE>
__global__ void __launch_bounds__(128, sliced_min_blocks<W>()) sliced_kernel(const SlicedArgs a) {
  // register spills (the w8 networks run at the 128-register cap) go to shared memory rather
  // than local memory, whose lines reached DRAM (profiles/r02n_smem_spilling_ab.log)
  asm volatile(".pragma \"enable_smem_spilling\";");
  constexpr int TAB_WORDS = M * (W / 4) * 16 * (W / 8);  // W-step tables, 32-bit words
  __shared__ __align__(16) uint32_t wtab[DECODE ? TAB_WORDS : 1];

  const uint64_t s = blockIdx.x / a.ctas_per_stripe;
  const uint32_t c = blockIdx.x % a.ctas_per_stripe;
  if (s >= a.n_stripes) return;

  uint32_t emask = 0;
  int t = 0;
  uint8_t outb[4] = {0, 0, 0, 0};
  if (DECODE) {
    const int pi = a.pat_idx[s];
    if (pi < 0) return;
    const SlicedPat &P = a.pats[pi];
    emask = P.erased_mask[0];
    t = P.t;
#pragma unroll
    for (int e = 0; e < 4; ++e) outb[e] = P.out_blk[e];
    const uint4 *src = reinterpret_cast<const uint4 *>(a.tables + P.table_off);
    for (int i = threadIdx.x; i < TAB_WORDS / 4; i += blockDim.x) reinterpret_cast<uint4 *>(wtab)[i] = src[i];
    __syncthreads();
  }

  // Block addresses.  w16: computed per access (an IMAD on the FMA pipe) -- the Horner loop
  // indexes the blocks at run time, and an array of K+M pointers then lives in local memory
  // (128 B of stack stores per thread that reached DRAM: ~6% of C4's write traffic).  w8:
  // every index is a compile-time constant, the array stays in registers (computing the
  // addresses instead needs more temporaries: 32 -> 140 B of spills for RS(10,4)).
  const auto units = [&](const auto &blk) {
    const uint64_t u0 = (uint64_t)c * a.units_per_cta;
    const uint64_t u1 = min(u0 + a.units_per_cta, a.units_per_stripe);
    for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x) {
      uint32_t h2;
      const uint64_t off = unit_offset<W>(u, u1, h2);
      uint32_t y[M * W];
      // w = 16 decode: the m syndromes of the received word (design C); otherwise the encoder
      constexpr bool kSyn = DECODE && RsQNet<K, M, W, POLY>::kHorner;
      if constexpr (kSyn) horner_syndromes<K, M, W, POLY>(blk, off, h2, emask, y);
      else encode_planes<K, M, W, POLY, DECODE>(blk, off, h2, emask, y);
  #pragma unroll
      for (int i = 0; i < M; ++i) transposeW<W>(&y[i * W]);

      if (!DECODE) {
  #pragma unroll
        for (int i = 0; i < M; ++i) store_unit<W>(blk[K + i] + off, &y[i * W], h2);
        continue;
      }

      if constexpr (!kSyn) {
        // Delta_i = received parity_i ^ encode(surviving data)_i (erased parity: received = 0)
  #pragma unroll
        for (int i = 0; i < M; ++i) {
          if (!((emask >> (K + i)) & 1u)) {
            uint32_t r[W];
            load_unit<W>(blk[K + i] + off, r, h2);
  #pragma unroll
            for (int q = 0; q < W; ++q) y[i * W + q] ^= r[q];
          }
        }
      }

      if (W == 8) {
        // y_e = sum_i W[e][i] Delta_i, four erasures packed per 32-bit table word.
        uint32_t acc[32];
  #pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = 0;
  #pragma unroll
        for (int i = 0; i < M; ++i) {
          const char *Tl = reinterpret_cast<const char *>(&wtab[i * 32]);
          const char *Th = reinterpret_cast<const char *>(&wtab[i * 32 + 16]);
  #pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t v = y[i * W + q];
            const uint32_t lo = shl_fma<2>(v) & 0x3C3C3C3Cu;  // low nibbles * 4 (byte offsets)
            const uint32_t hi = shr_fma<2>(v) & 0x3C3C3C3Cu;  // high nibbles * 4
  #pragma unroll
            for (int r = 0; r < 4; ++r) {
              const uint32_t il = __byte_perm(lo, 0, 0x4440 + r), ih = __byte_perm(hi, 0, 0x4440 + r);
              acc[4 * q + r] ^= *reinterpret_cast<const uint32_t *>(Tl + il) ^
                                *reinterpret_cast<const uint32_t *>(Th + ih);
            }
          }
        }
        // 4x4 byte transposes: acc[4q+r] byte e -> output e, word q, byte r
        uint32_t o[4][8];
  #pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t t0 = __byte_perm(acc[4 * q], acc[4 * q + 1], 0x5140);
          const uint32_t t1 = __byte_perm(acc[4 * q], acc[4 * q + 1], 0x7362);
          const uint32_t t2 = __byte_perm(acc[4 * q + 2], acc[4 * q + 3], 0x5140);
          const uint32_t t3 = __byte_perm(acc[4 * q + 2], acc[4 * q + 3], 0x7362);
          o[0][q] = __byte_perm(t0, t2, 0x5410);
          o[1][q] = __byte_perm(t0, t2, 0x7632);
          o[2][q] = __byte_perm(t1, t3, 0x5410);
          o[3][q] = __byte_perm(t1, t3, 0x7632);
        }
  #pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < t) store_unit<W>(a.L.block(s, outb[e]) + off, o[e], h2);
      } else {
        // w = 16: entries are 4 x 16-bit lanes (uint2), four nibbles per symbol.
        uint2 acc[32];
  #pragma unroll
        for (int q = 0; q < 32; ++q) acc[q] = make_uint2(0, 0);
  #pragma unroll
        for (int i = 0; i < M; ++i) {
          const char *T0 = reinterpret_cast<const char *>(&wtab[i * 128]);
  #pragma unroll
          for (int q = 0; q < 16; ++q) {
            const uint32_t v = y[i * W + q];
            const uint32_t lo = shl_fma<3>(v) & 0x78787878u;  // nibbles 0,2 of both symbols * 8
            const uint32_t hi = shr_fma<1>(v) & 0x78787878u;  // nibbles 1,3 * 8
  #pragma unroll
            for (int r = 0; r < 2; ++r) {  // symbol r of the word = column 2q+r
              const uint32_t n0 = __byte_perm(lo, 0, 0x4440 + 2 * r), n2 = __byte_perm(lo, 0, 0x4441 + 2 * r);
              const uint32_t n1 = __byte_perm(hi, 0, 0x4440 + 2 * r), n3 = __byte_perm(hi, 0, 0x4441 + 2 * r);
              const uint2 e0 = *reinterpret_cast<const uint2 *>(T0 + 0 * 128 + n0);
              const uint2 e1 = *reinterpret_cast<const uint2 *>(T0 + 1 * 128 + n1);
              const uint2 e2 = *reinterpret_cast<const uint2 *>(T0 + 2 * 128 + n2);
              const uint2 e3 = *reinterpret_cast<const uint2 *>(T0 + 3 * 128 + n3);
              acc[2 * q + r].x ^= e0.x ^ e1.x ^ e2.x ^ e3.x;
              acc[2 * q + r].y ^= e0.y ^ e1.y ^ e2.y ^ e3.y;
            }
          }
        }
        uint32_t o[16];
  #pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (e < t) {
  #pragma unroll
            for (int q = 0; q < 16; ++q) {
              const uint32_t a0 = (e < 2) ? acc[2 * q].x : acc[2 * q].y;
              const uint32_t a1 = (e < 2) ? acc[2 * q + 1].x : acc[2 * q + 1].y;
              o[q] = __byte_perm(a0, a1, (e & 1) ? 0x7632 : 0x5410);
            }
            store_unit<W>(a.L.block(s, outb[e]) + off, o, h2);
          }
        }
      }
    }
  };
  if constexpr (W == 16) {
    if (a.L.ptrs) units(PointerBlocks{a.L.ptrs + s * (uint64_t)a.L.n});
    else units(StridedBlocks{a.L.base + s * a.L.stripe_stride, a.L.block_stride});
  } else {
    BlockArray<K + M> arr;
#pragma unroll
    for (int i = 0; i < K + M; ++i) arr.p[i] = a.L.block(s, i);
    units(arr);
  }
}

// ---------------------------------------------------------------------------
// generic split-nibble kernel
// ---------------------------------------------------------------------------
// VERIFY: the outputs are syndromes; nothing is stored, a non-zero one sets a.flags[s].
template <int W, bool VERIFY>
__global__ void __launch_bounds__(256) generic_kernel(const GenericArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint8_t in_blk[kMaxN + 1];
  __shared__ uint8_t out_blk[4];

  const uint64_t per_stripe = (uint64_t)a.ctas_per_group * a.n_groups;
  const uint64_t s = blockIdx.x / per_stripe;
  const uint32_t rem = (uint32_t)(blockIdx.x % per_stripe);
  const uint32_t g = rem / a.ctas_per_group, c = rem % a.ctas_per_group;
  if (s >= a.n_stripes) return;
  const int pi = a.pat_idx ? a.pat_idx[s] : 0;
  if (pi < 0) return;
  const GenericPat &P = a.pats[pi];
  const int n_in = P.n_in, n_out = P.n_out;
  if ((int)g * 4 >= n_out) return;
  const int nr = min(4, n_out - 4 * (int)g);

  constexpr uint32_t TB = (W == 8) ? 128 : 512;  // table bytes per input
  const uint32_t tb = TB * (uint32_t)n_in;
  const uint4 *src = reinterpret_cast<const uint4 *>(a.tables + P.table_off + (uint64_t)g * tb);
  for (uint32_t i = threadIdx.x; i < tb / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = src[i];
  for (int i = threadIdx.x; i < n_in; i += blockDim.x) in_blk[i] = P.in_blk[i];
  if ((int)threadIdx.x < nr) out_blk[threadIdx.x] = P.out_blk[4 * g + threadIdx.x];
  __syncthreads();

  const uint64_t begin = a.col_begin + (uint64_t)c * a.chunk_bytes;
  const uint64_t end = min(begin + a.chunk_bytes, a.col_end);
  const uint32_t *T32 = reinterpret_cast<const uint32_t *>(smem);
  const uint2 *T64 = reinterpret_cast<const uint2 *>(smem);

  for (uint64_t off = begin + (uint64_t)threadIdx.x * 16; off < end; off += (uint64_t)blockDim.x * 16) {
    if (a.vec_ok && off + 16 <= end) {
      if (W == 8) {
        uint32_t acc[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) acc[q] = 0;
        for (int si = 0; si < n_in; ++si) {
          const uint4 v = ldg_v4(a.L.block(s, in_blk[si]) + off);
          const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
          const uint32_t *T = T32 + si * 32;
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const uint32_t byte = (wv[q] >> (8 * r)) & 0xFFu;
              acc[4 * q + r] ^= T[byte & 15u] ^ T[16 + (byte >> 4)];
            }
        }
        if (VERIFY) {
          uint32_t bad = 0;
#pragma unroll
          for (int q = 0; q < 16; ++q) bad |= acc[q];
          if (bad) atomicOr(&a.flags[s], 1u);
          continue;
        }
        for (int r = 0; r < nr; ++r) {
          uint32_t o[4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
            o[q] = ((acc[4 * q] >> (8 * r)) & 0xFFu) | (((acc[4 * q + 1] >> (8 * r)) & 0xFFu) << 8) |
                   (((acc[4 * q + 2] >> (8 * r)) & 0xFFu) << 16) | (((acc[4 * q + 3] >> (8 * r)) & 0xFFu) << 24);
          stg_v4(a.L.block(s, out_blk[r]) + off, make_uint4(o[0], o[1], o[2], o[3]));
        }
      } else {
        uint2 acc[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[q] = make_uint2(0, 0);
        for (int si = 0; si < n_in; ++si) {
          const uint4 v = ldg_v4(a.L.block(s, in_blk[si]) + off);
          const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
          const uint2 *T = T64 + si * 64;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const uint32_t sym = (wv[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
            const uint2 e0 = T[sym & 15u], e1 = T[16 + ((sym >> 4) & 15u)];
            const uint2 e2 = T[32 + ((sym >> 8) & 15u)], e3 = T[48 + (sym >> 12)];
            acc[q].x ^= e0.x ^ e1.x ^ e2.x ^ e3.x;
            acc[q].y ^= e0.y ^ e1.y ^ e2.y ^ e3.y;
          }
        }
        if (VERIFY) {
          uint32_t bad = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) bad |= acc[q].x | acc[q].y;
          if (bad) atomicOr(&a.flags[s], 1u);
          continue;
        }
        for (int r = 0; r < nr; ++r) {
          uint32_t o[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t a0 = r < 2 ? acc[2 * q].x : acc[2 * q].y;
            const uint32_t a1 = r < 2 ? acc[2 * q + 1].x : acc[2 * q + 1].y;
            o[q] = __byte_perm(a0, a1, (r & 1) ? 0x7632 : 0x5410);
          }
          stg_v4(a.L.block(s, out_blk[r]) + off, make_uint4(o[0], o[1], o[2], o[3]));
        }
      }
    } else {
      // scalar path: ragged tail or unaligned blocks
      const uint64_t lim = min(off + 16, end);
      for (uint64_t x = off; x < lim; x += W / 8) {
        if (W == 8) {
          uint32_t acc = 0;
          for (int si = 0; si < n_in; ++si) {
            const uint32_t byte = a.L.block(s, in_blk[si])[x];
            acc ^= T32[si * 32 + (byte & 15u)] ^ T32[si * 32 + 16 + (byte >> 4)];
          }
          if (VERIFY) {
            if (acc) atomicOr(&a.flags[s], 1u);
            continue;
          }
          for (int r = 0; r < nr; ++r) a.L.block(s, out_blk[r])[x] = (uint8_t)(acc >> (8 * r));
        } else {
          uint2 acc = make_uint2(0, 0);
          for (int si = 0; si < n_in; ++si) {
            const uint8_t *p = a.L.block(s, in_blk[si]) + x;
            const uint32_t sym = (uint32_t)p[0] | ((uint32_t)p[1] << 8);
            const uint2 *T = T64 + si * 64;
            const uint2 e0 = T[sym & 15u], e1 = T[16 + ((sym >> 4) & 15u)];
            const uint2 e2 = T[32 + ((sym >> 8) & 15u)], e3 = T[48 + (sym >> 12)];
            acc.x ^= e0.x ^ e1.x ^ e2.x ^ e3.x;
            acc.y ^= e0.y ^ e1.y ^ e2.y ^ e3.y;
          }
          if (VERIFY) {
            if (acc.x | acc.y) atomicOr(&a.flags[s], 1u);
            continue;
          }
          for (int r = 0; r < nr; ++r) {
            const uint32_t v = ((r < 2 ? acc.x : acc.y) >> (16 * (r & 1))) & 0xFFFFu;
            uint8_t *p = a.L.block(s, out_blk[r]) + x;
            p[0] = (uint8_t)(v & 0xFF);
            p[1] = (uint8_t)(v >> 8);
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_generic(int w, const GenericArgs &a, cudaStream_t st) {
  const uint64_t grid = a.n_stripes * a.n_groups * a.ctas_per_group;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
  count_launch();
  const bool verify = a.flags != nullptr;
  // The dynamic shared-memory opt-in is a per-device (per-context) function attribute:
  // set it once on every device the kernels launch on.
  static std::atomic<uint32_t> attr_done[64];
  int dev = 0;
  cudaGetDevice(&dev);
  const uint32_t bit = w == 8 ? 1u : 2u;
  if (dev >= 0 && dev < 64 && !(attr_done[dev].load() & bit)) {
    const int cap = kMaxN * (w == 8 ? 128 : 512);
    const bool ok = w == 8
        ? cudaFuncSetAttribute(generic_kernel<8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap) ==
                  cudaSuccess &&
              cudaFuncSetAttribute(generic_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap) ==
                  cudaSuccess
        : cudaFuncSetAttribute(generic_kernel<16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap) ==
                  cudaSuccess &&
              cudaFuncSetAttribute(generic_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap) ==
                  cudaSuccess;
    if (ok) attr_done[dev].fetch_or(bit);
    else cudaGetLastError();
  }
  if (w == 8) {
    if (verify) generic_kernel<8, true><<<(unsigned)grid, 256, a.smem_bytes, st>>>(a);
    else generic_kernel<8, false><<<(unsigned)grid, 256, a.smem_bytes, st>>>(a);
  } else {
    if (verify) generic_kernel<16, true><<<(unsigned)grid, 256, a.smem_bytes, st>>>(a);
    else generic_kernel<16, false><<<(unsigned)grid, 256, a.smem_bytes, st>>>(a);
  }
  return cudaGetLastError();
}

bool sliced_available(int k, int m, int w, uint32_t poly) {
#define RS_AVAIL(K, M, W, P) \
  if (k == K && m == M && w == W && poly == P) return true;
  RS_NET_INSTANCES(RS_AVAIL)
#undef RS_AVAIL
  return false;
}

cudaError_t launch_sliced(int k, int m, int w, uint32_t poly, bool decode, const SlicedArgs &a, cudaStream_t st) {
  const uint64_t grid = a.n_stripes * a.ctas_per_stripe;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
#define RS_LAUNCH(K, M, W, P)                                                  \
  if (k == K && m == M && w == W && poly == P) {                               \
    count_launch();                                                            \
    if (decode) sliced_kernel<K, M, W, P, true><<<(unsigned)grid, 128, 0, st>>>(a);  \
    else sliced_kernel<K, M, W, P, false><<<(unsigned)grid, 128, 0, st>>>(a);        \
    return cudaGetLastError();                                                 \
  }
  RS_NET_INSTANCES(RS_LAUNCH)
#undef RS_LAUNCH
  return cudaErrorNotSupported;
}

}  // namespace rsb
