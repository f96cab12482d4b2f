// linear.cpp -- "linear jobs": per stripe, out_r = sum_v M[r][v] in_v over a pointer table of
// virtual blocks, through a JIT network (pass-through inputs XORed after the transpose back)
// or the generic split-nibble kernel.  Serves:
//   * the diff-update: parity ^= P_J (old ^ new), in place;
//   * the cross-GPU placement: partial parity of a data subset, and the XOR
//     reduction of the partials at the parity owner.
#include "plan_internal.hpp"

namespace rsp {

// ---- linear jobs (diff-update, partial encode, XOR reduction) ----------------
// Cached LinearHost for `sig`, built by `fill` (which sets nv, out, M, group_blocks).
std::shared_ptr<const LinearHost> linear_host(const rs_poly_plan &P, const std::string &sig,
                                              const std::function<void(LinearHost &)> &fill) {
  std::lock_guard<std::mutex> lock(P.mu);
  auto it = P.lin_cache.find(sig);
  if (it != P.lin_cache.end()) return it->second;
  auto lh = std::make_shared<LinearHost>();
  fill(*lh);
  lh->id = (int)P.lin_cache.size() + 1;
  lh->nout = (int)lh->out.size();
  std::memset(&lh->gp, 0, sizeof(lh->gp));
  lh->gp.n_in = lh->nv;
  lh->gp.n_out = lh->nout;
  for (int v = 0; v < lh->nv; ++v) lh->gp.in_blk[v] = (uint8_t)v;
  for (int r = 0; r < lh->nout; ++r) lh->gp.out_blk[r] = (uint8_t)lh->out[r];
  pack_generic_tables(P.F, P.w, lh->M, lh->nout, lh->nv, lh->tab);
  P.lin_cache.emplace(sig, lh);
  return lh;
}

rsb::jit::Spec linear_spec(const rs_poly_plan &P, const LinearHost &lh) {
  std::vector<int> in(lh.nv);
  for (int v = 0; v < lh.nv; ++v) in[v] = v;
  rsb::jit::Spec s = jit_spec(P, in, lh.out, lh.M);
  if (lh.group_blocks) s.group_blocks = lh.group_blocks;
  return s;
}

// Diff-update of the sorted changed set idx: virtual blocks [new_0, old_0, new_1, old_1, ...,
// parity_0..m-1]; parity_i <- sum_j P[i][j] (new_j + old_j) + parity_i, M = [P_J P_J | I].
std::shared_ptr<const LinearHost> update_host(const rs_poly_plan &P, const std::vector<int> &idx) {
  std::string sig = "U";
  for (int j : idx) sig += ":" + std::to_string(j);
  return linear_host(P, sig, [&](LinearHost &lh) {
    const int c = (int)idx.size(), m = P.m, k = P.k;
    lh.nv = 2 * c + m;
    for (int i = 0; i < m; ++i) lh.out.push_back(2 * c + i);
    lh.M.assign((size_t)m * lh.nv, 0);
    for (int i = 0; i < m; ++i) {
      for (int q = 0; q < c; ++q) {
        const uint32_t coef = P.pmap[(size_t)i * k + idx[q]];  // x^{m+j} mod g, coefficient of x^i
        lh.M[(size_t)i * lh.nv + 2 * q] = coef;      // new_j
        lh.M[(size_t)i * lh.nv + 2 * q + 1] = coef;  // old_j (char 2: + = -)
      }
      lh.M[(size_t)i * lh.nv + 2 * c + i] = 1;       // the old parity itself
    }
    lh.group_blocks = P.w == 8 ? 12 : 4;  // even: each (new_j, old_j) pair shares a CSE group
  });
}

// Partial parity of the data subset idx (cross-GPU placement): virtual blocks
// [d_0..d_{c-1}, partial_0..partial_{m-1}]; partial_i <- sum_j P[i][j] d_j (+ partial_i).
std::shared_ptr<const LinearHost> partial_host(const rs_poly_plan &P, const std::vector<int> &idx, bool acc) {
  std::string sig = acc ? "PA" : "P";
  for (int j : idx) sig += ":" + std::to_string(j);
  return linear_host(P, sig, [&](LinearHost &lh) {
    const int c = (int)idx.size(), m = P.m, k = P.k;
    lh.nv = c + m;
    for (int i = 0; i < m; ++i) lh.out.push_back(c + i);
    lh.M.assign((size_t)m * lh.nv, 0);
    for (int i = 0; i < m; ++i) {
      for (int q = 0; q < c; ++q) lh.M[(size_t)i * lh.nv + q] = P.pmap[(size_t)i * k + idx[q]];
      if (acc) lh.M[(size_t)i * lh.nv + c + i] = 1;
    }
    lh.group_blocks = P.w == 8 ? 12 : 3;
  });
}

// XOR of n_src blocks into one: virtual blocks [src_0..src_{n-1}, dst]; dst <- sum src.
std::shared_ptr<const LinearHost> xor_host(const rs_poly_plan &P, int n_src) {
  return linear_host(P, "X:" + std::to_string(n_src), [&](LinearHost &lh) {
    lh.nv = n_src + 1;
    lh.out.push_back(n_src);
    lh.M.assign((size_t)lh.nv, 0);
    for (int q = 0; q < n_src; ++q) lh.M[q] = 1;  // all pass-through: raw XOR, no transposes
  });
}

// ptrs: host [S][nv] virtual block addresses.
rs_status linear_impl(const rs_poly_plan *P, const LinearHost &lh, const std::vector<uint64_t> &ptrs,
                      size_t n_stripes, size_t B, cudaStream_t st) {
  Geometry G;
  G.L.base = nullptr;
  G.L.n = lh.nv;
  G.n_stripes = n_stripes;
  G.block_bytes = B;
  G.aligned32 = G.aligned16 = true;
  for (uint64_t a : ptrs) {
    G.aligned32 = G.aligned32 && ptr_aligned(a, 32);
    G.aligned16 = G.aligned16 && ptr_aligned(a, 16);
  }
  uint64_t body = body_units_of(*P, G);
  const rsb::jit::Kernel *jk = nullptr;
  if (body && jit_eligible(*P, lh.nout))
    jk = jit_get(*P, JitKey{kJitLinear, MaskKey{(uint64_t)lh.id, 0, 0, 0}}, [&] { return linear_spec(*P, lh); },
                 false);
  if (!jk) body = 0;
  Blob b;
  const size_t ptrs_off = b.add(ptrs.data(), sizeof(uint64_t) * ptrs.size());
  rsb::GenericPat gp = lh.gp;
  gp.table_off = 0;
  const size_t pats_off = b.add(&gp, sizeof(gp));
  const size_t tables_off = b.add(lh.tab.data(), lh.tab.size());
  DevBlob d;
  cudaError_t e = d.upload(*P, b, st);
  if (e == cudaSuccess) G.L.ptrs = reinterpret_cast<const uint64_t *>(d.p + ptrs_off);
  if (e == cudaSuccess && body) {
    e = launch_jit(*jk, G, nullptr, G.n_stripes, body, st);
    P->jit_launches++;
  }
  const uint64_t UB = 32ull * (uint64_t)P->w / 8;
  if (e == cudaSuccess)
    e = launch_generic_range(*P, G, body * UB, G.block_bytes, d.p, pats_off, SIZE_MAX, tables_off,
                             (uint32_t)((lh.nout + 3) / 4), (uint32_t)(lh.nv * (P->w == 8 ? 128 : 512)), st);
  cudaError_t ef = d.release();
  return cuda_status(e != cudaSuccess ? e : ef);
}

// Validates data_idx; returns the permutation sorting it (order[q] = caller position).
rs_status parse_update(const rs_poly_plan *P, const int *data_idx, int c, std::vector<int> &sorted,
                       std::vector<int> &order) {
  sorted.clear();
  order.clear();
  if (c < 0 || (c && !data_idx)) return RS_ERR_INVALID_ARG;
  if (c > P->k) return RS_ERR_BAD_ERASURE;
  if (2 * c + P->m > RS_POLY_MAX_N) return RS_ERR_INVALID_ARG;
  std::vector<char> seen(P->k, 0);
  for (int q = 0; q < c; ++q) {
    const int j = data_idx[q];
    if (j < 0 || j >= P->k || seen[j]) return RS_ERR_BAD_ERASURE;
    seen[j] = 1;
    order.push_back(q);
  }
  std::sort(order.begin(), order.end(), [&](int a, int b2) { return data_idx[a] < data_idx[b2]; });
  for (int q : order) sorted.push_back(data_idx[q]);
  return RS_OK;
}

}  // namespace rsp

extern "C" {

rs_status rs_poly_update(const rs_poly_plan *P, const int *data_idx, int n_changed, const void *const *old_data,
                         const void *const *new_data, void *const *parity, size_t block_bytes, void *stream) {
  NvtxRange nvtx_("rs_poly_update");
  if (!P) return RS_ERR_INVALID_ARG;
  std::vector<int> idx, order;
  rs_status rc = parse_update(P, data_idx, n_changed, idx, order);
  if (rc) return rc;
  rc = check_geometry(P, block_bytes);
  if (rc) return rc;
  if (n_changed == 0) return RS_OK;
  if (!old_data || !new_data || !parity) return RS_ERR_INVALID_ARG;
  const uint64_t a = (uint64_t)(P->w / 8);
  std::vector<uint64_t> ptrs;
  for (int q : order) {
    ptrs.push_back(reinterpret_cast<uint64_t>(new_data[q]));
    ptrs.push_back(reinterpret_cast<uint64_t>(old_data[q]));
  }
  for (int i = 0; i < P->m; ++i) ptrs.push_back(reinterpret_cast<uint64_t>(parity[i]));
  for (uint64_t v : ptrs)
    if (!v) return RS_ERR_INVALID_ARG;
    else if (v % a) return RS_ERR_GEOMETRY;
  auto uh = update_host(*P, idx);
  return linear_impl(P, *uh, ptrs, 1, block_bytes, static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_update_batch(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t stripe_stride,
                               size_t block_stride, size_t block_bytes, const int *data_idx, int n_changed,
                               const void *old_blocks, size_t old_stripe_stride, size_t old_block_stride,
                               void *stream) {
  NvtxRange nvtx_("rs_poly_update_batch");
  if (!P) return RS_ERR_INVALID_ARG;
  std::vector<int> idx, order;
  rs_status rc = parse_update(P, data_idx, n_changed, idx, order);
  if (rc) return rc;
  rc = check_strided(P, stripes, n_stripes, stripe_stride, block_stride, block_bytes);
  if (rc) return rc;
  if (n_changed == 0 || n_stripes == 0) return RS_OK;
  const uint64_t a = (uint64_t)(P->w / 8);
  if (!old_blocks) return RS_ERR_INVALID_ARG;
  if (reinterpret_cast<uint64_t>(old_blocks) % a || old_stripe_stride % a || old_block_stride % a)
    return RS_ERR_GEOMETRY;
  if (n_changed > 1 && old_block_stride < block_bytes) return RS_ERR_GEOMETRY;
  if (n_stripes > 1 && old_stripe_stride < (uint64_t)(n_changed - 1) * old_block_stride + block_bytes)
    return RS_ERR_GEOMETRY;
  auto uh = update_host(*P, idx);
  std::vector<uint64_t> ptrs;
  ptrs.reserve(n_stripes * (size_t)uh->nv);
  const uint64_t base = reinterpret_cast<uint64_t>(stripes), obase = reinterpret_cast<uint64_t>(old_blocks);
  for (size_t s = 0; s < n_stripes; ++s) {
    for (int q : order) {
      ptrs.push_back(base + s * stripe_stride + (uint64_t)data_idx[q] * block_stride);
      ptrs.push_back(obase + s * old_stripe_stride + (uint64_t)q * old_block_stride);
    }
    for (int i = 0; i < P->m; ++i) ptrs.push_back(base + s * stripe_stride + (uint64_t)(P->k + i) * block_stride);
  }
  return linear_impl(P, *uh, ptrs, n_stripes, block_bytes, static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_encode_partial(const rs_poly_plan *P, const int *data_idx, int n_data, const void *const *data,
                                 void *const *partial, size_t n_stripes, size_t block_bytes, int accumulate,
                                 void *stream) {
  NvtxRange nvtx_("rs_poly_encode_partial");
  if (!P) return RS_ERR_INVALID_ARG;
  std::vector<int> idx, order;
  rs_status rc = parse_update(P, data_idx, n_data, idx, order);
  if (rc) return rc;
  rc = check_geometry(P, block_bytes);
  if (rc) return rc;
  if (n_stripes == 0 || (n_data == 0 && accumulate)) return RS_OK;
  if (!partial || (n_data && !data)) return RS_ERR_INVALID_ARG;
  const uint64_t a = (uint64_t)(P->w / 8);
  auto lh = partial_host(*P, idx, accumulate != 0);
  std::vector<uint64_t> ptrs;
  ptrs.reserve(n_stripes * (size_t)lh->nv);
  for (size_t s = 0; s < n_stripes; ++s) {
    for (int q : order) ptrs.push_back(reinterpret_cast<uint64_t>(data[s * (size_t)n_data + q]));
    for (int i = 0; i < P->m; ++i) ptrs.push_back(reinterpret_cast<uint64_t>(partial[s * (size_t)P->m + i]));
  }
  for (uint64_t v : ptrs)
    if (!v) return RS_ERR_INVALID_ARG;
    else if (v % a) return RS_ERR_GEOMETRY;
  return linear_impl(P, *lh, ptrs, n_stripes, block_bytes, static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_xor_reduce(const rs_poly_plan *P, void *const *dst, const void *const *srcs, int n_src,
                             size_t n_stripes, size_t bytes, void *stream) {
  NvtxRange nvtx_("rs_poly_xor_reduce");
  if (!P || n_src < 1 || n_src + 1 > RS_POLY_MAX_N) return RS_ERR_INVALID_ARG;
  rs_status rc = check_geometry(P, bytes);
  if (rc) return rc;
  if (n_stripes == 0) return RS_OK;
  if (!dst || !srcs) return RS_ERR_INVALID_ARG;
  const uint64_t a = (uint64_t)(P->w / 8);
  auto lh = xor_host(*P, n_src);
  std::vector<uint64_t> ptrs;
  ptrs.reserve(n_stripes * (size_t)lh->nv);
  for (size_t s = 0; s < n_stripes; ++s) {
    for (int q = 0; q < n_src; ++q) ptrs.push_back(reinterpret_cast<uint64_t>(srcs[s * (size_t)n_src + q]));
    ptrs.push_back(reinterpret_cast<uint64_t>(dst[s]));
  }
  for (uint64_t v : ptrs)
    if (!v) return RS_ERR_INVALID_ARG;
    else if (v % a) return RS_ERR_GEOMETRY;
  return linear_impl(P, *lh, ptrs, n_stripes, bytes, static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_prepare_update(const rs_poly_plan *P, const int *data_idx, int n_changed) {
  if (!P) return RS_ERR_INVALID_ARG;
  std::vector<int> idx, order;
  rs_status rc = parse_update(P, data_idx, n_changed, idx, order);
  if (rc) return rc;
  if (n_changed == 0 || P->jit_mode == RS_JIT_OFF || !jit_eligible(*P, P->m)) return RS_OK;
  auto uh = update_host(*P, idx);
  jit_get(*P, JitKey{kJitLinear, MaskKey{(uint64_t)uh->id, 0, 0, 0}}, [&] { return linear_spec(*P, *uh); }, true);
  return RS_OK;
}

size_t rs_poly_update_jit_source(const rs_poly_plan *P, const int *data_idx, int n_changed, char *buf,
                                 size_t cap) {
  if (!P || n_changed < 1 || !jit_eligible(*P, P->m)) return 0;
  std::vector<int> idx, order;
  if (parse_update(P, data_idx, n_changed, idx, order)) return 0;
  const std::string s = rsb::jit::source(P->F, linear_spec(*P, *update_host(*P, idx)), nullptr);
  if (buf && cap) {
    const size_t nc = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), nc);
    buf[nc] = 0;
  }
  return s.size();
}

}  // extern "C"
