// jit.hpp -- run-time specialised bit-sliced kernels (NVRTC, sm_100a).
//
// For a fixed GF matrix M (outputs x inputs) -- an erasure pattern's decode
// matrix R_E = V_E^{-1} A_E (P:244-303 with Opt1/Opt3 of P:319-323 taken to
// code generation), the parity map of a code without a compiled network, a
// diff-update / partial-encode / XOR "linear job", or the syndrome map of verify --
// this builds the GF(2) bit-matrix, reduces it with the same greedy CSE as
// gen_networks.py (pairs and triples, for 3-input LOP3 gates) and compiles a
// straight-line kernel: every HBM byte of the inputs read once, the outputs written
// once, no runtime tables.  w16 decoders/encoders use the syndrome (Horner) form.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gf.hpp"

namespace rsb {
namespace jit {

struct Spec {
  int w = 8;
  std::vector<int> in_blk;   // API block indices read, input order
  std::vector<int> out_blk;  // API block indices written
  std::vector<uint32_t> M;   // out x in GF(2^w) matrix, row-major
  int group_blocks = 0;      // inputs per CSE group (0 = all)
  int min_blocks = 4;        // __launch_bounds__ min CTAs/SM
  // Syndrome (Horner) form, used for w = 16: `seq` lists the API block at
  // each polynomial position from the highest down (-1 = erased: multiply only), T
  // syndromes S_j = sum_p c_p alpha^{j p'} are folded with step alpha^j, and the
  // outputs are M (out x T) applied to S.  in_blk is unused in this form.
  bool horner = false;
  uint32_t poly = 0;
  std::vector<int> seq;
  int T = 0;
  // verify: compute the outputs (syndromes) but, instead of storing them, flag the stripe
  // (Args::flags[s] |= 1) when any is non-zero
  bool verify = false;
};

struct Kernel {
  bool ok = false;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t fn = nullptr;
  int xors = 0;
  int w = 8;            // symbol width of the spec it was generated from (grid sizing)
  bool cached = false;  // loaded from the on-disk cubin cache
  double compile_ms = 0;
  std::string log;
};

// Argument block of every generated kernel (mirrors the struct in the source).
struct Args {
  uint8_t *base;
  uint64_t stripe_stride, block_stride;
  const uint64_t *ptrs;
  int n;
  int pad;
  const int32_t *stripes;  // selected stripe indices (nullptr = stripe_base .. stripe_base+n_sel-1)
  uint64_t n_sel, units_per_stripe;
  uint32_t units_per_cta, ctas_per_stripe;
  uint64_t stripe_base;
  unsigned *flags;  // verify kernels: per stripe, set to 1 if not a codeword
};

bool available(std::string *why = nullptr);
std::string source(const Field &F, const Spec &spec, int *xors);
Kernel compile(const std::string &src);
void release(Kernel &k);

}  // namespace jit
}  // namespace rsb
