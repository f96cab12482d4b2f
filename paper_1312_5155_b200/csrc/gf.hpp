// gf.hpp -- GF(2^w) table and constant builder (host side of the product path).
//
// Builds, from (w, prim_poly) with alpha = 2:
//   * exp/log tables and the primitivity check ord(alpha) = 2^w - 1;
//   * the generator polynomial g(x) = prod_{i<m} (x + alpha^i);
//   * the m x k parity map P: column j = x^{m+j} mod g(x), i.e. the
//     generator-matrix form of g, computed by the shift-register
//     recurrence col_{j+1} = x * col_j mod g (col_0 = g_0..g_{m-1});
//   * the per-erasure-pattern decode matrices of P:244-303 (Opt1/Opt3 of
//     alpha powers and V^{-1} computed once per pattern).
// Independent of oracle/: nothing here is shared with the CPU oracle.
#pragma once
#include <cstdint>
#include <vector>

namespace rsb {

struct Field {
  int w = 0;
  uint32_t poly = 0, q = 0;  // q = 2^w - 1
  std::vector<uint32_t> exp_;  // 2q entries
  std::vector<int32_t> log_;   // 2^w entries, log_[0] = -1

  // false if prim_poly is not of degree w or alpha = 2 is not primitive.
  bool init(int w_, uint32_t poly_) {
    w = w_; poly = poly_;
    if ((w != 8 && w != 16) || (poly >> w) != 1u) return false;
    q = (1u << w) - 1;
    exp_.assign(2 * (size_t)q, 0);
    log_.assign((size_t)1 << w, -1);
    uint32_t x = 1;
    for (uint32_t i = 0; i < q; ++i) {
      if (log_[x] != -1) return false;  // alpha's order < q
      exp_[i] = exp_[i + q] = x;
      log_[x] = (int32_t)i;
      x <<= 1;
      if (x >> w) x ^= poly;
    }
    return x == 1;
  }
  uint32_t mul(uint32_t a, uint32_t b) const {
    return (a && b) ? exp_[(size_t)log_[a] + (size_t)log_[b]] : 0;
  }
  uint32_t inv(uint32_t a) const { return a ? exp_[(q - (uint32_t)log_[a]) % q] : 0; }
  uint32_t alpha_pow(uint64_t e) const { return exp_[e % q]; }
};

// g(x) low -> high, monic, m+1 coefficients.
inline std::vector<uint32_t> generator_poly(const Field &F, int m) {
  std::vector<uint32_t> g{1};
  for (int i = 0; i < m; ++i) {
    uint32_t root = F.alpha_pow((uint64_t)i);
    std::vector<uint32_t> ng(g.size() + 1, 0);
    for (size_t l = 0; l < ng.size(); ++l) {
      uint32_t hi = l > 0 ? g[l - 1] : 0;
      uint32_t lo = l < g.size() ? F.mul(root, g[l]) : 0;
      ng[l] = hi ^ lo;
    }
    g.swap(ng);
  }
  return g;
}

// P[i*k + j]: coefficient of x^i in x^{m+j} mod g (p_i = sum_j P[i][j] d_j).
inline std::vector<uint32_t> parity_map(const Field &F, int k, int m, const std::vector<uint32_t> &g) {
  std::vector<uint32_t> P((size_t)m * k), col(g.begin(), g.begin() + m);
  for (int j = 0; j < k; ++j) {
    for (int i = 0; i < m; ++i) P[(size_t)i * k + j] = col[i];
    uint32_t top = col[m - 1];  // x * col overflows into x^m = sum_i g_i x^i
    for (int i = m - 1; i >= 0; --i) col[i] = (i ? col[i - 1] : 0) ^ F.mul(top, g[i]);
  }
  return P;
}

// In-place inverse of a t x t matrix (row-major) by Gauss-Jordan; false if singular.
inline bool invert(const Field &F, std::vector<uint32_t> &A, int t) {
  std::vector<uint32_t> I((size_t)t * t, 0);
  for (int i = 0; i < t; ++i) I[(size_t)i * t + i] = 1;
  for (int c = 0; c < t; ++c) {
    int p = -1;
    for (int r = c; r < t; ++r)
      if (A[(size_t)r * t + c]) { p = r; break; }
    if (p < 0) return false;
    if (p != c)
      for (int x = 0; x < t; ++x) {
        std::swap(A[(size_t)p * t + x], A[(size_t)c * t + x]);
        std::swap(I[(size_t)p * t + x], I[(size_t)c * t + x]);
      }
    uint32_t iv = F.inv(A[(size_t)c * t + c]);
    for (int x = 0; x < t; ++x) {
      A[(size_t)c * t + x] = F.mul(A[(size_t)c * t + x], iv);
      I[(size_t)c * t + x] = F.mul(I[(size_t)c * t + x], iv);
    }
    for (int r = 0; r < t; ++r) {
      uint32_t f = r == c ? 0 : A[(size_t)r * t + c];
      if (!f) continue;
      for (int x = 0; x < t; ++x) {
        A[(size_t)r * t + x] ^= F.mul(f, A[(size_t)c * t + x]);
        I[(size_t)r * t + x] ^= F.mul(f, I[(size_t)c * t + x]);
      }
    }
  }
  A.swap(I);
  return true;
}

// Syndrome-form encoder matrix Q (m x m, row-major): parity p = Q H where
// H_j = sum_b d_b alpha^{j b} (Horner over the data).  Every codeword has zero
// syndromes at the roots alpha^0..alpha^{m-1} of g, so
// sum_i p_i alpha^{j i} = alpha^{j m} H_j and Q = Vp^{-1} diag(alpha^{j m}),
// Vp[j][i] = alpha^{j i} -- the decoder used to encode.
inline std::vector<uint32_t> horner_q(const Field &F, int m) {
  std::vector<uint32_t> V((size_t)m * m);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < m; ++i) V[(size_t)j * m + i] = F.alpha_pow((uint64_t)j * (uint64_t)i);
  if (!invert(F, V, m)) return {};
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) V[(size_t)i * m + j] = F.mul(V[(size_t)i * m + j], F.alpha_pow((uint64_t)j * m));
  return V;
}

// Polynomial position of API block b (data b -> x^{m+b}, parity b -> x^{b-k}).
inline int position(int b, int k, int m) { return b < k ? m + b : b - k; }

}  // namespace rsb
