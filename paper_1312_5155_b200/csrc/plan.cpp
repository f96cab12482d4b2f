// plan.cpp -- host planner, decode-pattern cache and C ABI (include/rs_poly.h).
//
// Plan creation: field tables, g(x), parity map.
// Decode patterns (P:213-303 with the paper's Opt1-Opt3): for an
// erasure set E (t = |E| <= m) the planner builds, once per pattern,
//   V_E[j][e]  = (alpha^{pos_e})^j, j < t          (Step-2 Vandermonde matrix)
//   V_E^{-1}                                          (Opt3: inverted once)
//   W = V_E^{-1} H_par[0:t,:],  H_par[j][i] = alpha^{j i}   (bit-sliced path)
//   R = V_E^{-1} A_E,  A_E[j][s] = alpha^{j pos(s)} over survivors s (generic)
// and the packed split-nibble tables the kernels read.  Both are exact
// rewritings of y = V_E^{-1} (D(alpha^0..alpha^{t-1})) -- see DESIGN.md.
#include "plan_internal.hpp"

namespace rsp {


// Packed split-nibble tables for "out_r = sum_s M[r][s] in_s" (layout in rs_kernels.cuh).
void pack_generic_tables(const Field &F, int w, const std::vector<uint32_t> &M, int n_out, int n_in,
                         std::vector<uint8_t> &out) {
  const int groups = (n_out + 3) / 4;
  const int nh = w / 4;               // nibbles per symbol
  const size_t eb = (w == 8) ? 4 : 8;  // entry bytes
  out.assign((size_t)groups * n_in * nh * 16 * eb, 0);
  for (int g = 0; g < groups; ++g)
    for (int s = 0; s < n_in; ++s)
      for (int h = 0; h < nh; ++h)
        for (uint32_t v = 0; v < 16; ++v) {
          uint64_t packed = 0;
          for (int r = 0; r < 4 && 4 * g + r < n_out; ++r) {
            uint64_t prod = F.mul(M[(size_t)(4 * g + r) * n_in + s], v << (4 * h));
            packed |= prod << (w * r);
          }
          uint8_t *dst = out.data() + ((((size_t)g * n_in + s) * nh + h) * 16 + v) * eb;
          std::memcpy(dst, &packed, eb);  // little-endian host
        }
}

std::shared_ptr<const PatternHost> build_pattern(const rs_poly_plan &P, const std::vector<int> &er) {
  const Field &F = P.F;
  const int t = (int)er.size(), k = P.k, m = P.m, n = P.n;
  auto ph = std::make_shared<PatternHost>();
  ph->erased = er;
  // Opt1: alpha powers of the erased positions; Step-2 matrix
  std::vector<uint32_t> V((size_t)t * t), X(t);
  for (int e = 0; e < t; ++e) X[e] = F.alpha_pow((uint64_t)rsb::position(er[e], k, m));
  for (int j = 0; j < t; ++j)
    for (int e = 0; e < t; ++e) V[(size_t)j * t + e] = F.alpha_pow((uint64_t)F.log_[X[e]] * (uint64_t)j);
  if (!rsb::invert(F, V, t)) return nullptr;  // Opt3: V^{-1} once per pattern
  ph->Vinv = V;
  // W = V^{-1} H_par[0:t, :]  (t x m)
  std::vector<uint32_t> W((size_t)t * m, 0);
  for (int e = 0; e < t; ++e)
    for (int i = 0; i < m; ++i) {
      uint32_t acc = 0;
      for (int j = 0; j < t; ++j) acc ^= F.mul(V[(size_t)e * t + j], F.alpha_pow((uint64_t)j * (uint64_t)i));
      W[(size_t)e * m + i] = acc;
    }
  // R = V^{-1} A_E over the survivors (t x (n-t))
  std::vector<int> surv;
  std::vector<char> is_er(n, 0);
  for (int b : er) is_er[b] = 1;
  for (int b = 0; b < n; ++b)
    if (!is_er[b]) surv.push_back(b);
  const int ns = (int)surv.size();
  std::vector<uint32_t> R((size_t)t * ns, 0);
  for (int e = 0; e < t; ++e)
    for (int si = 0; si < ns; ++si) {
      uint32_t acc = 0;
      const uint64_t p = (uint64_t)rsb::position(surv[si], k, m);
      for (int j = 0; j < t; ++j) acc ^= F.mul(V[(size_t)e * t + j], F.alpha_pow((uint64_t)j * p));
      R[(size_t)e * ns + si] = acc;
    }
  ph->surv = surv;
  ph->R = R;
  ph->unknown = er;
  ph->Hm = ph->Vinv;
  if (P.read_policy == RS_READ_K_SURVIVORS && t < m) {
    // Read only k survivors K (data first, then parity, ascending): the m - t unread ones
    // join the unknowns U (|U| = m), solved from all m syndrome equations (j < m):
    // c_U = V_U^{-1} A_K c_K; only the E rows are produced.  Unique (MDS), so the
    // output is identical; the traffic is (k + t) B instead of (n - t) B + t B.
    std::vector<int> K, U = er;
    for (int b = 0; b < n && (int)K.size() < k; ++b)
      if (!is_er[b]) K.push_back(b);
    for (int b = 0; b < n; ++b)
      if (!is_er[b] && std::find(K.begin(), K.end(), b) == K.end()) U.push_back(b);
    std::sort(U.begin(), U.end());
    std::vector<uint32_t> VU((size_t)m * m);
    for (int j = 0; j < m; ++j)
      for (int u = 0; u < m; ++u)
        VU[(size_t)j * m + u] =
            F.alpha_pow((uint64_t)rsb::position(U[u], k, m) * (uint64_t)j);
    if (!rsb::invert(F, VU, m)) return nullptr;
    std::vector<int> rowE;  // row of V_U^{-1} for each erased block, in er order
    for (int b : er) rowE.push_back((int)(std::find(U.begin(), U.end(), b) - U.begin()));
    std::vector<uint32_t> RK((size_t)t * k, 0), Hm((size_t)t * m, 0);
    for (int e = 0; e < t; ++e) {
      for (int u = 0; u < m; ++u) Hm[(size_t)e * m + u] = VU[(size_t)rowE[e] * m + u];
      for (int q = 0; q < k; ++q) {
        uint32_t acc = 0;
        const uint64_t p = (uint64_t)rsb::position(K[q], k, m);
        for (int j = 0; j < m; ++j) acc ^= F.mul(Hm[(size_t)e * m + j], F.alpha_pow((uint64_t)j * p));
        RK[(size_t)e * k + q] = acc;
      }
    }
    ph->surv = K;
    ph->R = RK;
    ph->unknown = U;
    ph->Hm = Hm;
  }
  // sliced record
  if (P.sliced) {
    std::memset(&ph->sp, 0, sizeof(ph->sp));
    for (int b : er) ph->sp.erased_mask[b >> 5] |= 1u << (b & 31);
    ph->sp.t = t;
    for (int e = 0; e < t && e < 4; ++e) ph->sp.out_blk[e] = (uint8_t)er[e];
    if (P.w == 16) {
      // the w16 table kernel solves from the m syndromes of the received word (design C):
      // y = [V_E^{-1} | 0] S, S_j for j < m (only j < t enter)
      std::vector<uint32_t> Vx((size_t)t * m, 0);
      for (int e = 0; e < t; ++e)
        for (int j = 0; j < t; ++j) Vx[(size_t)e * m + j] = V[(size_t)e * t + j];
      pack_generic_tables(F, P.w, Vx, t, m, ph->wtab);
    } else {
      pack_generic_tables(F, P.w, W, t, m, ph->wtab);  // one group (t <= 4): [i][h][v]
    }
  }
  // generic record
  std::memset(&ph->gp, 0, sizeof(ph->gp));
  const int nin = (int)ph->surv.size();
  ph->gp.n_in = nin;
  ph->gp.n_out = t;
  for (int si = 0; si < nin; ++si) ph->gp.in_blk[si] = (uint8_t)ph->surv[si];
  for (int e = 0; e < t; ++e) ph->gp.out_blk[e] = (uint8_t)er[e];
  pack_generic_tables(F, P.w, ph->R, t, nin, ph->rtab);
  return ph;
}

rs_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return RS_OK;
  if (e == cudaErrorMemoryAllocation) return RS_ERR_NOMEM;
  return RS_ERR_CUDA;
}


bool jit_eligible(const rs_poly_plan &P, int n_out) { return P.w == 8 ? n_out <= 8 : n_out <= 4; }

rsb::jit::Spec jit_spec(const rs_poly_plan &P, const std::vector<int> &in, const std::vector<int> &out,
                        const std::vector<uint32_t> &M) {
  rsb::jit::Spec s;
  s.w = P.w;
  s.in_blk = in;
  s.out_blk = out;
  s.M = M;
  // CSE groups of input blocks (0 = one network over all inputs).  w16: 3 blocks keep the
  // planes in registers.  w8: one network while inputs + outputs fit in 14 blocks of planes
  // (RS(10,4) decode: 36 B spilled at 128 registers, grouping costs more than it saves);
  // beyond that it spills 136-300 B per thread, and groups of 10 - outputs blocks spill
  // nothing for +6-14% LOP3 (r01q: RS(10,6) encode 93% -> 103%, decode 77% -> 92%).
  const int n_io = (int)(in.size() + out.size());
  s.group_blocks = P.w == 8 ? (n_io > 14 ? std::max(2, 10 - (int)out.size()) : 0) : 3;
  // w8 at 4 CTAs/SM (128 registers): 3 CTAs/SM without spills is slower even for 5-6
  // outputs (r01q: RS(10,5) encode 88% vs 105%; 5 CTAs/SM spills more, profiles/r01q_w8_jit_occupancy.log).
  s.min_blocks = P.w == 8 ? 4 : 3;
  return s;
}

// __launch_bounds__ min CTAs/SM of the w16 JIT kernels: 3 (168 registers); 4 caps them at
// 128 and spills ~400 B (r01: 68% vs 80%), 2 (225 registers, no spill) is slower too
// (r02c: C4 per-stripe decode 0.76 vs 0.86 of the copy peak, profiles/r02c_w16_occupancy.log).
constexpr int kJitW16MinBlocks = 3;

// The encoder kernel of a code without a compiled network: w = 8 the parity-map
// network, w = 16 the syndrome form (Horner over the data, then Q).
rsb::jit::Spec encoder_spec(const rs_poly_plan &P) {
  std::vector<int> in(P.k), out(P.m);
  for (int j = 0; j < P.k; ++j) in[j] = j;
  for (int i = 0; i < P.m; ++i) out[i] = P.k + i;
  rsb::jit::Spec s = jit_spec(P, in, out, P.pmap);
  if (P.w == 16) {
    s.horner = true;
    s.poly = P.poly;
    s.T = P.m;
    s.M = rsb::horner_q(P.F, P.m);
    for (int j = P.k - 1; j >= 0; --j) s.seq.push_back(j);  // positions m+k-1 .. m
    s.min_blocks = kJitW16MinBlocks;
  }
  return s;
}

// The decoder kernel of one erasure pattern: w = 8 the network of R = V_E^{-1} A_E over
// the survivors; w = 16 Horner over all n positions (erased: multiply only), then V_E^{-1}.
rsb::jit::Spec decoder_spec(const rs_poly_plan &P, const PatternHost &ph) {
  rsb::jit::Spec s = jit_spec(P, ph.surv, ph.erased, ph.R);
  if (P.w == 16) {
    s.horner = true;
    s.poly = P.poly;
    s.T = (int)ph.unknown.size();
    s.M = ph.Hm;
    std::vector<char> er(P.n, 0);
    for (int b : ph.unknown) er[b] = 1;
    for (int pos = P.n - 1; pos >= 0; --pos) {
      const int b = pos >= P.m ? pos - P.m : P.k + pos;  // inverse of rsb::position
      s.seq.push_back(er[b] ? -1 : b);
    }
    s.min_blocks = kJitW16MinBlocks;
  }
  return s;
}

// One empty launch (a single CTA with no stripe selected: it returns at once) of a freshly
// loaded JIT kernel, on a library-private non-blocking stream: the driver's first-launch setup
// of the function then happens here, at prepare time, not inside the first decode call that
// uses it (C5 first decode after rs_poly_prepare_all: profiles/r02e_cold.log).  Not counted
// in rs_poly_launch_count (no user work); errors are dropped.
std::mutex g_warm_mu;
std::map<int, cudaStream_t> g_warm_streams;  // device -> stream of the warm launches

void warm_launch(const rsb::jit::Kernel &k) {
  std::mutex &mu = g_warm_mu;
  std::map<int, cudaStream_t> &streams = g_warm_streams;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaStream_t st = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = streams.find(dev);
    if (it == streams.end()) {
      if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return;
      }
      streams.emplace(dev, st);
    } else {
      st = it->second;
    }
  }
  rsb::jit::Args a{};
  a.n_sel = 0;
  a.units_per_cta = kSlicedThreads;
  a.ctas_per_stripe = 1;
  void *args[] = {&a};
  if (cudaLaunchKernel(reinterpret_cast<const void *>(k.fn), dim3(1), dim3(kSlicedThreads), args, 0, st) !=
      cudaSuccess)
    cudaGetLastError();
}

// Wait for the queued warm launches of the current device (rs_poly_prepare returns only after
// them: ~2 us of GPU time each, a prepare_all's 1470 would otherwise delay the next call).
void warm_sync() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  cudaStream_t st = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_warm_mu);
    auto it = g_warm_streams.find(dev);
    if (it != g_warm_streams.end()) st = it->second;
  }
  if (st && cudaStreamSynchronize(st) != cudaSuccess) cudaGetLastError();
}

// The compiled kernel for `key` if it is ready; schedules (background) or runs (sync /
// wait) its compilation on first request.  Must be called without holding P.mu.
const rsb::jit::Kernel *jit_get(const rs_poly_plan &P, const JitKey &key, const std::function<rsb::jit::Spec()> &mk,
                                bool wait) {
  if (P.jit_mode == RS_JIT_OFF || !rsb::jit::available()) return nullptr;
  std::shared_ptr<JitEntry> e;
  std::shared_ptr<std::promise<std::shared_ptr<rsb::jit::Kernel>>> prom;
  {
    std::lock_guard<std::mutex> lock(P.mu);
    auto it = P.jit.find(key);
    if (it != P.jit.end()) {
      e = it->second;
    } else if (P.jit.size() >= kMaxJitKernels) {
      return nullptr;  // bounded module count per plan: further patterns use the table kernels
    } else {
      e = std::make_shared<JitEntry>();
      prom = std::make_shared<std::promise<std::shared_ptr<rsb::jit::Kernel>>>();
      e->fut = prom->get_future().share();
      P.jit.emplace(key, e);
    }
  }
  const bool block = wait || P.jit_mode == RS_JIT_SYNC;
  if (prom) {
    int dev = 0;
    cudaGetDevice(&dev);
    auto job = [prom, spec = mk(), F = &P.F, dev]() {
      if (CompilePool::stopping()) {  // process exit: do not compile, do not touch CUDA
        auto k = std::make_shared<rsb::jit::Kernel>();
        k->log = "cancelled at exit";
        prom->set_value(k);
        return;
      }
      cudaSetDevice(dev);  // load the module under the caller's device, not device 0
      int xors = 0;
      const std::string src = rsb::jit::source(*F, spec, &xors);
      auto k = std::make_shared<rsb::jit::Kernel>(rsb::jit::compile(src));
      k->xors = xors;
      k->w = spec.w;
      if (k->ok) warm_launch(*k);
      if (!k->ok) {  // loud, once per process (the pattern then runs on the table kernel)
        static std::atomic<int> reported{0};
        if (reported.fetch_add(1) == 0 || std::getenv("RS_POLY_JIT_LOG"))
          std::fprintf(stderr, "[rs_poly] JIT compile/load failed (falling back to tables): %s\n", k->log.c_str());
      }
      prom->set_value(k);
    };
    if (block) job();
    else CompilePool::get().submit(job);
  }
  if (block) e->fut.wait();
  return e->kernel();
}

std::vector<cudaStream_t> side_streams(const rs_poly_plan &P) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(P.mu);
  auto &v = P.pool[dev];
  // Extra PDL chains for the per-pattern JIT launches: one extra for w = 8 (two ~20 KB
  // kernels share an SM well: C3 decode 89% -> 96%), none for w = 16 (two ~60 KB kernels
  // thrash the instruction cache: C4 78% -> 56%; profiles/r01q_side_streams.log,
  // r01t_w16_side_stream_recheck.log).
  const size_t want = P.w == 8 ? 1 : 0;
  if (want == 0) return {};
  while (v.size() < want) {
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) break;
    v.push_back(s);
  }
  return std::vector<cudaStream_t>(v.begin(), v.begin() + std::min(want, v.size()));
}

uint64_t body_units_of(const rs_poly_plan &P, const Geometry &G) {
  const uint64_t UB = 32ull * (uint64_t)P.w / 8;
  return G.aligned32 ? G.block_bytes / UB : 0;
}

int sm_count() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  int v = cache[dev].load();
  if (!v) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v);
  }
  return v;
}

// Units (32 columns each) per CTA so that a launch has about 4 (w = 8) or 8 (w = 16) CTAs
// per SM, in multiples of the CTA size, at most kSlicedUnitsPerCta.  Measured
// on per-stripe decode chains (r01p): w = 8 (C3, 4 CTAs/SM resident) runs best with 2 units
// per thread (97% vs 94% of the copy peak with 1, 92% with 4); w = 16 (3 CTAs/SM, a 4x
// longer body per unit) with 1 (80% vs 68% with 2).
uint32_t units_per_cta_for(uint64_t total, int w) {
  const uint64_t per_sm = w == 8 ? 4 : 8;
  const uint64_t target = (uint64_t)sm_count() * per_sm;
  uint64_t upc = (total + target - 1) / target;
  upc = (upc + kSlicedThreads - 1) / kSlicedThreads * kSlicedThreads;
  return (uint32_t)std::min<uint64_t>(std::max<uint64_t>(upc, kSlicedThreads), kSlicedUnitsPerCta);
}

cudaError_t launch_jit(const rsb::jit::Kernel &k, const Geometry &G, const int32_t *stripes, uint64_t n_sel,
                       uint64_t body_units, cudaStream_t st, bool pdl, uint64_t stripe_base, unsigned *flags) {
  rsb::jit::Args a{};
  a.stripe_base = stripe_base;
  a.flags = flags;
  a.base = G.L.base;
  a.stripe_stride = G.L.stripe_stride;
  a.block_stride = G.L.block_stride;
  a.ptrs = G.L.ptrs;
  a.n = G.L.n;
  a.stripes = stripes;
  a.n_sel = n_sel;
  a.units_per_stripe = body_units;
  a.units_per_cta = units_per_cta_for(n_sel * body_units, k.w);
  if (k.w == 16 && a.units_per_cta == kSlicedThreads) {
    // A w16 grid with a small partial second wave (at most a quarter wave past one full wave
    // of resident CTAs) becomes one wave of 2-unit CTAs: a PDL successor launches only once
    // every CTA has started, so the partial wave left SMs idle at each link of a per-stripe
    // chain.  RS(12,4) 4 MiB blocks (1.15 waves): 0.70 -> 0.75 of the copy peak; grids of 1.4
    // waves and more (5, 6, 8 MiB) lose 4-8% when re-cut (profiles/r02v_w16_grid_waves_ab.log).
    const uint64_t slots = (uint64_t)sm_count() * kJitW16MinBlocks;
    const uint64_t ctas = n_sel * ((body_units + kSlicedThreads - 1) / kSlicedThreads);
    if (ctas > slots && 4 * ctas <= 5 * slots) a.units_per_cta = 2 * kSlicedThreads;
  }
  a.ctas_per_stripe = (uint32_t)((body_units + a.units_per_cta - 1) / a.units_per_cta);
  const uint64_t grid = n_sel * a.ctas_per_stripe;
  if (grid == 0) return cudaSuccess;
  if (grid > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
  void *args[] = {&a};
  rsb::count_launch();
  if (!pdl)
    return cudaLaunchKernel(reinterpret_cast<const void *>(k.fn), dim3((unsigned)grid), dim3(kSlicedThreads), args,
                            0, st);
  // programmatic dependent launch (the generated kernels trigger at entry; their last CTA waits at exit)
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kSlicedThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(k.fn), args);
}

cudaError_t launch_sliced_body(const rs_poly_plan &P, bool decode, const Geometry &G, uint64_t body_units,
                               const uint8_t *dev, size_t pats_off, size_t idx_off, size_t tables_off,
                               cudaStream_t st) {
  rsb::SlicedArgs a{};
  a.L = G.L;
  a.n_stripes = G.n_stripes;
  a.units_per_stripe = body_units;
  a.units_per_cta = units_per_cta_for(G.n_stripes * body_units, P.w);
  a.ctas_per_stripe = (uint32_t)((body_units + a.units_per_cta - 1) / a.units_per_cta);
  if (decode) {
    a.pats = reinterpret_cast<const rsb::SlicedPat *>(dev + pats_off);
    a.pat_idx = reinterpret_cast<const int32_t *>(dev + idx_off);
    a.tables = dev + tables_off;
  }
  return rsb::launch_sliced(P.k, P.m, P.w, P.poly, decode, a, st);
}

cudaError_t launch_generic_range(const rs_poly_plan &P, const Geometry &G, uint64_t col_begin, uint64_t col_end,
                                 const uint8_t *dev, size_t pats_off, size_t idx_off, size_t tables_off,
                                 uint32_t groups, uint32_t smem, cudaStream_t st, unsigned *flags) {
  if (col_begin >= col_end) return cudaSuccess;
  rsb::GenericArgs a{};
  a.flags = flags;
  a.L = G.L;
  a.pats = reinterpret_cast<const rsb::GenericPat *>(dev + pats_off);
  a.pat_idx = idx_off == SIZE_MAX ? nullptr : reinterpret_cast<const int32_t *>(dev + idx_off);
  a.tables = dev + tables_off;
  a.n_stripes = G.n_stripes;
  a.col_begin = col_begin;
  a.col_end = col_end;
  const uint64_t span = col_end - col_begin;
  const uint64_t step = (uint64_t)kGenericThreads * 16;
  const uint64_t chunk = std::min<uint64_t>(kGenericChunk, (span + step - 1) / step * step);
  a.chunk_bytes = chunk;
  a.ctas_per_group = (uint32_t)((span + chunk - 1) / chunk);
  a.n_groups = groups;
  a.vec_ok = G.aligned16 ? 1u : 0u;
  a.smem_bytes = smem;
  return rsb::launch_generic(P.w, a, st);
}

// Process-wide pool (one per device) for the per-call blobs.  The default pool returns its
// memory to the driver at every synchronize (release threshold 0), so a call after a
// synchronize would re-map its blob: ~0.2 ms of host time before the first launch, with the
// GPU idle.  This pool keeps up to 64 MiB.  It lives for the process (never destroyed:
// destroying pools while other threads' plans tear down was measured to hang).
cudaError_t blob_pool(cudaMemPool_t *out) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pools.find(dev);
  if (it != pools.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  cudaMemPoolProps props{};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = dev;
  cudaMemPool_t pool = nullptr;
  e = cudaMemPoolCreate(&pool, &props);
  if (e != cudaSuccess) return e;
  uint64_t keep = 64ull << 20;  // blobs are small (constants, stripe lists, pointer tables)
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e != cudaSuccess) {
    cudaMemPoolDestroy(pool);
    return e;
  }
  pools[dev] = pool;
  *out = pool;
  return cudaSuccess;
}

// Copy `bytes` at `src` to device `dst` on stream `s` through one of the plan's pinned
// slots (reused once its previous copy has completed); pageable only if no slot can be had.
cudaError_t upload_pinned(const rs_poly_plan &P, void *dst, const void *src, size_t bytes, cudaStream_t s) {
  // At most kMaxSlots pinned slots.  When all are in flight the host is at least that
  // many calls ahead of the GPU, so it waits for the oldest copy instead of allocating:
  // a cudaHostAlloc inside a stream of back-to-back calls can starve the GPU.
  constexpr size_t kMaxSlots = 16;
  int dev = 0;
  cudaGetDevice(&dev);
  rs_poly_plan::PinnedSlot *slot = nullptr;
  {
    std::lock_guard<std::mutex> lock(P.stage_mu);
    for (auto &sl : P.stage)
      if (!sl.busy && sl.dev == dev && sl.cap >= bytes && cudaEventQuery(sl.ev) == cudaSuccess) {
        slot = &sl;
        break;
      }
    if (!slot && P.stage.size() >= kMaxSlots) {
      rs_poly_plan::PinnedSlot *oldest = nullptr;
      for (auto &sl : P.stage)
        if (!sl.busy && sl.dev == dev && sl.cap >= bytes && (!oldest || sl.seq < oldest->seq)) oldest = &sl;
      if (oldest && cudaEventSynchronize(oldest->ev) == cudaSuccess) slot = oldest;
    }
    if (!slot && P.stage.size() < kMaxSlots) {
      rs_poly_plan::PinnedSlot sl;
      sl.dev = dev;
      sl.cap = std::max<size_t>(bytes, 64 << 10);
      if (cudaHostAlloc(reinterpret_cast<void **>(&sl.p), sl.cap, cudaHostAllocDefault) == cudaSuccess &&
          cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming) == cudaSuccess) {
        P.stage.reserve(kMaxSlots);  // slots never move: pointers into the vector stay valid
        P.stage.push_back(sl);
        slot = &P.stage.back();
      } else {
        if (sl.p) cudaFreeHost(sl.p);
        cudaGetLastError();
      }
    }
    if (slot) {
      slot->busy = true;
      slot->seq = ++P.stage_seq;
    }
  }
  if (!slot) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
  std::memcpy(slot->p, src, bytes);
  cudaError_t e = cudaMemcpyAsync(dst, slot->p, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaEventRecord(slot->ev, s);
  if (e != cudaSuccess) cudaStreamSynchronize(s);  // never hand out a slot a copy may still read
  std::lock_guard<std::mutex> lock(P.stage_mu);
  slot->busy = false;
  return e;
}


rs_status check_geometry(const rs_poly_plan *P, size_t block_bytes) {
  if (!P) return RS_ERR_INVALID_ARG;
  if (block_bytes == 0 || block_bytes % (size_t)(P->w / 8)) return RS_ERR_GEOMETRY;
  return RS_OK;
}

// Plan-static device constants (uploaded once per plan and device).  A pageable cudaMemcpy
// may return before its DMA lands and runs on the legacy stream, which a non-blocking
// caller stream does not wait for: the copy is completed (legacy stream synchronized)
// before the pointer is published, so any later launch on any stream reads it whole.
uint8_t *upload_plan_consts(const std::vector<uint8_t> &h) {
  uint8_t *d = nullptr;
  if (cudaMalloc(reinterpret_cast<void **>(&d), h.size()) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaStreamSynchronize(cudaStreamLegacy) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  return d;
}

// Device copy of the encode tail constants [GenericPat | tables], made once per plan and
// device (upload_plan_consts: complete before first use on any stream).
const uint8_t *enc_consts(const rs_poly_plan &P) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(P.mu);
  auto it = P.enc_dev.find(dev);
  if (it != P.enc_dev.end()) return it->second;
  std::vector<uint8_t> h(kEncTablesOff + P.enc_tab.size(), 0);
  rsb::GenericPat gp = P.enc_gp;
  gp.table_off = 0;
  std::memcpy(h.data(), &gp, sizeof(gp));
  std::memcpy(h.data() + kEncTablesOff, P.enc_tab.data(), P.enc_tab.size());
  uint8_t *d = upload_plan_consts(h);
  if (d) P.enc_dev.emplace(dev, d);
  return d;
}

rs_status encode_impl(const rs_poly_plan *P, Geometry G, const uint64_t *ptrs, cudaStream_t st) {
  const rsb::jit::Kernel *jk = nullptr;
  uint64_t body = body_units_of(*P, G);
  if (body && !P->sliced && jit_eligible(*P, P->m)) {
    std::vector<int> in(P->k), out(P->m);
    for (int j = 0; j < P->k; ++j) in[j] = j;
    for (int i = 0; i < P->m; ++i) out[i] = P->k + i;
    jk = jit_get(*P, kEncodeKey, [&] { return encoder_spec(*P); }, false);
  }
  if (!P->sliced && !jk) body = 0;
  // Per call only the pointer table (pointer mode) is uploaded; the encode constants of the
  // generic tail kernel are plan-static and live on the device once per plan and device.
  const uint64_t UB0 = 32ull * (uint64_t)P->w / 8;
  const bool tail = body * UB0 < G.block_bytes;
  const uint8_t *cdev = nullptr;
  if (tail && !(cdev = enc_consts(*P))) return RS_ERR_CUDA;
  const size_t pats_off = 0, tables_off = kEncTablesOff;
  DevBlob d;
  cudaError_t e = cudaSuccess;
  if (ptrs) {
    Blob b;
    b.add(ptrs, sizeof(uint64_t) * (size_t)P->n * G.n_stripes);
    e = d.upload(*P, b, st);
    if (e == cudaSuccess) G.L.ptrs = reinterpret_cast<const uint64_t *>(d.p);
  }
  if (e == cudaSuccess && body) {
    if (P->sliced) {
      e = launch_sliced_body(*P, false, G, body, nullptr, 0, 0, 0, st);
    } else {
      e = launch_jit(*jk, G, nullptr, G.n_stripes, body, st);
      P->jit_launches++;
    }
  }
  if (e == cudaSuccess && tail)
    e = launch_generic_range(*P, G, body * UB0, G.block_bytes, cdev, pats_off, SIZE_MAX, tables_off,
                             (uint32_t)((P->m + 3) / 4), (uint32_t)(P->k * (P->w == 8 ? 128 : 512)), st);
  cudaError_t ef = d.release();
  return cuda_status(e != cudaSuccess ? e : ef);
}

// Distinct patterns of a batch, in order of first appearance, with each stripe's index.
rs_status collect_patterns(const rs_poly_plan *P, const std::vector<std::vector<int>> &rows,
                           std::vector<std::shared_ptr<const PatternHost>> &pats, std::vector<MaskKey> &keys,
                           std::vector<int32_t> &idx) {
  std::map<MaskKey, int> local;
  idx.assign(rows.size(), -1);
  std::lock_guard<std::mutex> lock(P->mu);
  for (size_t s = 0; s < rows.size(); ++s) {
    const auto &er = rows[s];
    if (er.empty()) continue;
    MaskKey key{0, 0, 0, 0};
    for (int b : er) key[b >> 6] |= 1ull << (b & 63);
    auto it = local.find(key);
    if (it != local.end()) {
      idx[s] = it->second;
      continue;
    }
    auto c = P->cache.find(key);
    std::shared_ptr<const PatternHost> ph;
    if (c != P->cache.end()) {
      ph = c->second;
    } else {
      ph = build_pattern(*P, er);
      if (!ph) return RS_ERR_INVALID_ARG;
      P->cache.emplace(key, ph);
    }
    idx[s] = (int32_t)pats.size();
    local.emplace(key, (int)pats.size());
    pats.push_back(ph);
    keys.push_back(key);
  }
  return RS_OK;
}


const rsb::jit::Kernel *pattern_jit(const rs_poly_plan &P, const PatternHost &ph, const MaskKey &key, bool wait) {
  if (!jit_eligible(P, (int)ph.erased.size())) return nullptr;
  return jit_get(P, JitKey{kJitDecode, key}, [&] { return decoder_spec(P, ph); }, wait);
}

// RS_POLY_HOST_PROFILE=1: per-call host time of each decode phase on stderr (diagnostics)
struct HostProfile {
  bool on;
  std::chrono::steady_clock::time_point t;
  std::string line;
  HostProfile() : on(enabled()), t(on ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{}) {}
  static bool enabled() {
    static const bool v = std::getenv("RS_POLY_HOST_PROFILE") != nullptr;
    return v;
  }
  void mark(const char *what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    line += std::string(" ") + what + "=" +
            std::to_string(std::chrono::duration<double, std::micro>(n - t).count()).substr(0, 8) + "us";
    t = n;
  }
  ~HostProfile() {
    if (on && !line.empty()) std::fprintf(stderr, "[rs_poly host]%s\n", line.c_str());
  }
};

// The per-pattern JIT kernels of one decode call, one launch per group (a pattern's stripes,
// or one run of adjacent stripes).
// Launches form programmatic-dependent-launch chains: each generated kernel triggers its
// dependents on entry and its last CTA waits for the predecessor before exit, so kernel i+1's CTAs
// fill kernel i's last wave (a C4 stripe is only ~2.3 waves) while completion stays in
// stream order.  The first kernel of a chain is launched without the attribute, so it
// never overlaps work queued before the call.  With side streams (side_streams()), the
// patterns are dealt round-robin over 1 + N chains forked from and joined back to `st`.
// dev_lists: device base of the per-pattern stripe lists (grp_off), or nullptr when every
// group is a contiguous stripe range (passed by value).
cudaError_t launch_jit_chains(const rs_poly_plan &P, const std::vector<const rsb::jit::Kernel *> &jk,
                              const std::vector<std::vector<int32_t>> &groups, const Geometry &G, uint64_t body,
                              const uint8_t *dev_lists, const std::vector<size_t> &grp_off, cudaStream_t st) {
  size_t nlaunch = 0;
  for (const auto &g : groups) nlaunch += g.empty() ? 0 : 1;
  std::vector<cudaStream_t> side = nlaunch > 1 ? side_streams(P) : std::vector<cudaStream_t>{};
  cudaError_t e = cudaSuccess;
  cudaEvent_t fork = nullptr;
  if (!side.empty()) {
    e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(fork, st);
  }
  std::vector<char> used(side.size(), 0), chained(side.size() + 1, 0);
  size_t rr = 0;
  for (size_t i = 0; i < groups.size() && e == cudaSuccess; ++i) {
    if (groups[i].empty()) continue;
    const size_t lane = rr++ % (side.size() + 1);
    cudaStream_t s = lane == 0 ? st : side[lane - 1];
    if (lane && !used[lane - 1]) {
      e = cudaStreamWaitEvent(s, fork, 0);
      used[lane - 1] = 1;
    }
    if (e != cudaSuccess) break;
    if (dev_lists)
      e = launch_jit(*jk[i], G, reinterpret_cast<const int32_t *>(dev_lists + grp_off[i]), groups[i].size(), body,
                     s, chained[lane] != 0);
    else
      e = launch_jit(*jk[i], G, nullptr, groups[i].size(), body, s, chained[lane] != 0, (uint64_t)groups[i][0]);
    chained[lane] = 1;
    P.jit_launches++;
  }
  for (size_t l = 0; l < side.size(); ++l) {
    if (!used[l]) continue;
    cudaEvent_t join = nullptr;
    cudaError_t e2 = cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    if (e2 == cudaSuccess) e2 = cudaEventRecord(join, side[l]);
    if (e2 == cudaSuccess) e2 = cudaStreamWaitEvent(st, join, 0);
    if (join) cudaEventDestroy(join);
    if (e == cudaSuccess) e = e2;
  }
  if (fork) cudaEventDestroy(fork);
  return e;
}

// rows: per stripe list of erased API indices (validated, sorted ascending)
rs_status decode_impl(const rs_poly_plan *P, Geometry G, const uint64_t *ptrs,
                      const std::vector<std::vector<int>> &rows, cudaStream_t st) {
  std::vector<std::shared_ptr<const PatternHost>> pats;
  std::vector<MaskKey> keys;
  std::vector<int32_t> idx;
  HostProfile hp;
  rs_status rc = collect_patterns(P, rows, pats, keys, idx);
  hp.mark("collect");
  if (rc) return rc;
  if (pats.empty()) return RS_OK;
  const uint64_t UB = 32ull * (uint64_t)P->w / 8;
  uint64_t body = body_units_of(*P, G);
  // JIT kernels for the patterns whose compile is done (others fall back to tables)
  std::vector<const rsb::jit::Kernel *> jk(pats.size(), nullptr);
  bool any_jit = false;
  if (body)
    for (size_t i = 0; i < pats.size(); ++i) {
      jk[i] = pattern_jit(*P, *pats[i], keys[i], false);
      any_jit = any_jit || jk[i];
    }
  hp.mark("jit_lookup");
  // the table-driven bit-sliced decode reads every survivor: not under RS_READ_K_SURVIVORS
  const bool sliced_rt = P->sliced && P->read_policy == RS_READ_ALL_SURVIVORS;
  if (!sliced_rt && !any_jit) body = 0;
  std::vector<int32_t> idx_rt(idx);
  std::vector<std::vector<int32_t>> groups(pats.size());
  bool any_rt = false;
  for (size_t s = 0; s < idx.size(); ++s) {
    if (idx[s] < 0) continue;
    if (jk[idx[s]]) {
      groups[idx[s]].push_back((int32_t)s);
      idx_rt[s] = -1;
    } else {
      any_rt = true;
    }
  }
  // Lean path: every pattern has its JIT kernel, no ragged tail, strided layout and each
  // pattern's stripes contiguous (one stripe, or one shared pattern) -- nothing to upload,
  // the kernels take the stripe range by value.
  bool contig = true;
  for (const auto &gr : groups)
    for (size_t q = 1; q < gr.size() && contig; ++q) contig = gr[q] == gr[0] + (int32_t)q;
  if (any_jit && !any_rt && !ptrs && contig && body * UB == G.block_bytes) {
    const rs_status r = cuda_status(launch_jit_chains(*P, jk, groups, G, body, nullptr, {}, st));
    hp.mark("launch(lean)");
    return r;
  }
  // A pattern that recurs on non-adjacent stripes: one lean launch per run of adjacent
  // stripes instead of a stripe list in an uploaded blob (each CTA would first load its
  // stripe index from it -- a dependent global load before any of its data loads).
  // Only while that adds few launches: at most twice the patterns' (alternating patterns
  // over many small stripes would otherwise turn one launch per pattern into one per stripe).
  size_t n_runs = 0, n_groups = 0;
  for (const auto &gr : groups) {
    n_groups += !gr.empty();
    for (size_t q = 0; q < gr.size(); ++q) n_runs += q == 0 || gr[q] != gr[q - 1] + 1;
  }
  if (any_jit && !any_rt && !ptrs && body * UB == G.block_bytes && n_runs <= 2 * n_groups) {
    std::vector<const rsb::jit::Kernel *> jr;
    std::vector<std::vector<int32_t>> runs;
    jr.reserve(n_runs);
    runs.reserve(n_runs);
    for (size_t i = 0; i < groups.size(); ++i)
      for (size_t q = 0; q < groups[i].size(); ++q) {
        if (q == 0 || groups[i][q] != groups[i][q - 1] + 1) {
          jr.push_back(jk[i]);
          runs.emplace_back();
        }
        runs.back().push_back(groups[i][q]);
      }
    const rs_status r = cuda_status(launch_jit_chains(*P, jr, runs, G, body, nullptr, {}, st));
    hp.mark("launch(runs)");
    return r;
  }
  Blob b;
  size_t ptrs_off = SIZE_MAX;
  if (ptrs) ptrs_off = b.add(ptrs, sizeof(uint64_t) * (size_t)P->n * G.n_stripes);
  const size_t idx_off = b.add(idx.data(), sizeof(int32_t) * idx.size());
  const size_t idx_rt_off = b.add(idx_rt.data(), sizeof(int32_t) * idx_rt.size());
  std::vector<size_t> grp_off(pats.size(), SIZE_MAX);
  for (size_t i = 0; i < pats.size(); ++i)
    if (!groups[i].empty()) grp_off[i] = b.add(groups[i].data(), sizeof(int32_t) * groups[i].size());
  const bool records = any_rt || body * UB < G.block_bytes;  // a table kernel will run
  std::vector<rsb::SlicedPat> sps(records ? pats.size() : 0);
  std::vector<rsb::GenericPat> gps(records ? pats.size() : 0);
  const size_t sliced_pats_off = b.add(nullptr, sizeof(rsb::SlicedPat) * sps.size());
  const size_t generic_pats_off = b.add(nullptr, sizeof(rsb::GenericPat) * gps.size());
  const size_t tables_off = b.add(nullptr, 0);
  uint32_t max_groups = 1, max_in = 1;
  // Table records only for the patterns a table kernel will read: every pattern when there
  // is a ragged tail, else only those still without a JIT kernel (a many-pattern batch
  // would otherwise upload ~2 KB of tables per pattern per call for nothing).
  const bool tail = body * UB < G.block_bytes;
  for (size_t i = 0; i < sps.size(); ++i) {
    const PatternHost &ph = *pats[i];
    const bool needs_rt = jk[i] == nullptr && any_rt;
    if (sliced_rt && needs_rt) {
      sps[i] = ph.sp;
      sps[i].table_off = (uint32_t)(b.add(ph.wtab.data(), ph.wtab.size()) - tables_off);
    }
    if (tail || (needs_rt && !sliced_rt)) {
      gps[i] = ph.gp;
      gps[i].table_off = (uint32_t)(b.add(ph.rtab.data(), ph.rtab.size()) - tables_off);
      max_groups = std::max<uint32_t>(max_groups, (uint32_t)((ph.gp.n_out + 3) / 4));
      max_in = std::max<uint32_t>(max_in, (uint32_t)ph.gp.n_in);
    }
  }
  std::memcpy(b.h.data() + sliced_pats_off, sps.data(), sizeof(rsb::SlicedPat) * sps.size());
  std::memcpy(b.h.data() + generic_pats_off, gps.data(), sizeof(rsb::GenericPat) * gps.size());
  const uint32_t smem = max_in * (P->w == 8 ? 128 : 512);

  hp.mark("blob");
  DevBlob d;
  cudaError_t e = d.upload(*P, b, st);
  hp.mark("upload");
  if (e == cudaSuccess && ptrs) G.L.ptrs = reinterpret_cast<const uint64_t *>(d.p + ptrs_off);
  // table-driven body for stripes without a ready JIT kernel
  if (e == cudaSuccess && body && any_rt) {
    if (sliced_rt) e = launch_sliced_body(*P, true, G, body, d.p, sliced_pats_off, idx_rt_off, tables_off, st);
    else e = launch_generic_range(*P, G, 0, body * UB, d.p, generic_pats_off, idx_rt_off, tables_off, max_groups,
                                  smem, st);
    P->table_launches++;
  }
  // ragged tails (and everything when there is no bit-sliced body)
  if (e == cudaSuccess)
    e = launch_generic_range(*P, G, body * UB, G.block_bytes, d.p, generic_pats_off, idx_off, tables_off,
                             max_groups, smem, st);
  if (e == cudaSuccess && any_jit) e = launch_jit_chains(*P, jk, groups, G, body, d.p, grp_off, st);
  hp.mark("launch");
  cudaError_t ef = d.release();
  return cuda_status(e != cudaSuccess ? e : ef);
}

rs_status parse_row(const rs_poly_plan *P, const int32_t *row, int count, std::vector<int> &out, bool allow_pad) {
  out.clear();
  std::vector<char> seen(P->n, 0);
  for (int i = 0; i < count; ++i) {
    int b = row[i];
    if (allow_pad && b == -1) continue;
    if (b < 0 || b >= P->n) return RS_ERR_BAD_ERASURE;
    if (seen[b]) return RS_ERR_BAD_ERASURE;
    seen[b] = 1;
    out.push_back(b);
  }
  if ((int)out.size() > P->m) return RS_ERR_TOO_MANY_ERASURES;
  std::sort(out.begin(), out.end());
  return RS_OK;
}

Geometry strided(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t ss, size_t bs, size_t B) {
  Geometry G;
  G.L.base = static_cast<uint8_t *>(stripes);
  G.L.stripe_stride = ss;
  G.L.block_stride = bs;
  G.L.n = P->n;
  G.n_stripes = n_stripes;
  G.block_bytes = B;
  const uint64_t base = reinterpret_cast<uint64_t>(stripes);
  G.aligned32 = ptr_aligned(base, 32) && ptr_aligned(ss, 32) && ptr_aligned(bs, 32);
  G.aligned16 = ptr_aligned(base, 16) && ptr_aligned(ss, 16) && ptr_aligned(bs, 16);
  return G;
}

rs_status check_strided(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t ss, size_t bs, size_t B) {
  rs_status rc = check_geometry(P, B);
  if (rc) return rc;
  if (n_stripes && !stripes) return RS_ERR_INVALID_ARG;
  const uint64_t a = (uint64_t)(P->w / 8);
  if (!ptr_aligned(reinterpret_cast<uint64_t>(stripes), a) || ss % a || bs % a) return RS_ERR_GEOMETRY;
  if (P->n > 1 && bs < B) return RS_ERR_GEOMETRY;                      // blocks overlap
  if (n_stripes > 1 && ss < (uint64_t)(P->n - 1) * bs + B) return RS_ERR_GEOMETRY;  // stripes overlap
  return RS_OK;
}

// ---- verify (scrub): are the stripes codewords? -----------------------------
// Every codeword vanishes at the roots alpha^0..alpha^{m-1} of g, i.e. its m
// syndromes S_j = sum_p c_p alpha^{j p} (Step 1 of the decode, with nothing
// erased) are zero; a stripe with any non-zero syndrome in any column is flagged.
rsb::jit::Spec verify_spec(const rs_poly_plan &P) {
  const int n = P.n, m = P.m;
  std::vector<int> in(n), out(m);
  for (int b = 0; b < n; ++b) in[b] = b;
  for (int i = 0; i < m; ++i) out[i] = i;  // nothing is stored in verify mode
  std::vector<uint32_t> A((size_t)m * n);
  for (int j = 0; j < m; ++j)
    for (int b = 0; b < n; ++b)
      A[(size_t)j * n + b] = P.F.alpha_pow((uint64_t)j * (uint64_t)rsb::position(b, P.k, m));
  rsb::jit::Spec s = jit_spec(P, in, out, A);
  s.verify = true;
  if (P.w == 16) {
    s.horner = true;
    s.poly = P.poly;
    s.T = m;
    for (int pos = n - 1; pos >= 0; --pos) s.seq.push_back(pos >= m ? pos - m : P.k + pos);
    s.min_blocks = kJitW16MinBlocks;
  } else {
    s.group_blocks = 10;  // n * 8 input planes in CSE groups of 10 blocks
  }
  return s;
}

// Device copy of [GenericPat | tables] for the syndrome map A (m x n), once per plan and device.
const uint8_t *ver_consts(const rs_poly_plan &P) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(P.mu);
  auto it = P.ver_dev.find(dev);
  if (it != P.ver_dev.end()) return it->second;
  const rsb::jit::Spec sp = verify_spec(P);
  std::vector<uint8_t> tab;
  pack_generic_tables(P.F, P.w, sp.M, P.m, P.n, tab);
  rsb::GenericPat gp;
  std::memset(&gp, 0, sizeof(gp));
  gp.n_in = P.n;
  gp.n_out = P.m;
  for (int b = 0; b < P.n; ++b) gp.in_blk[b] = (uint8_t)b;
  std::vector<uint8_t> h(kEncTablesOff + tab.size(), 0);
  std::memcpy(h.data(), &gp, sizeof(gp));
  std::memcpy(h.data() + kEncTablesOff, tab.data(), tab.size());
  uint8_t *d = upload_plan_consts(h);
  if (d) P.ver_dev.emplace(dev, d);
  return d;
}

rs_status verify_impl(const rs_poly_plan *P, Geometry G, unsigned *flags, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(unsigned) * G.n_stripes, st);
  uint64_t body = body_units_of(*P, G);
  const rsb::jit::Kernel *jk = nullptr;
  if (body && e == cudaSuccess && jit_eligible(*P, P->m))
    jk = jit_get(*P, JitKey{kJitVerify, MaskKey{0, 0, 0, 0}}, [&] { return verify_spec(*P); }, false);
  if (!jk) body = 0;
  const uint64_t UB = 32ull * (uint64_t)P->w / 8;
  const uint8_t *cdev = nullptr;
  if (e == cudaSuccess && body * UB < G.block_bytes && !(cdev = ver_consts(*P))) return RS_ERR_CUDA;
  if (e == cudaSuccess && body) {
    e = launch_jit(*jk, G, nullptr, G.n_stripes, body, st, false, 0, flags);
    P->jit_launches++;
  }
  if (e == cudaSuccess)
    e = launch_generic_range(*P, G, body * UB, G.block_bytes, cdev, 0, SIZE_MAX, kEncTablesOff,
                             (uint32_t)((P->m + 3) / 4), (uint32_t)(P->n * (P->w == 8 ? 128 : 512)), st, flags);
  return cuda_status(e);
}

}  // namespace rsp

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int rs_poly_abi_version(void) { return RS_POLY_ABI_VERSION; }
uint64_t rs_poly_launch_count(void) { return rsb::launches_total(); }

const char *rs_poly_strerror(rs_status s) {
  switch (s) {
    case RS_OK: return "ok";
    case RS_ERR_INVALID_ARG: return "invalid argument";
    case RS_ERR_NOT_PRIMITIVE: return "prim_poly is not a primitive polynomial of degree w with alpha=2";
    case RS_ERR_GEOMETRY: return "bad block geometry (size/alignment)";
    case RS_ERR_TOO_MANY_ERASURES: return "more than m erasures";
    case RS_ERR_BAD_ERASURE: return "erasure index out of range or duplicated";
    case RS_ERR_CUDA: return "CUDA error";
    case RS_ERR_NOMEM: return "out of memory";
  }
  return "unknown status";
}

rs_status rs_poly_plan_create(int k, int m, int w, uint32_t prim_poly, rs_poly_plan **out) {
  if (!out) return RS_ERR_INVALID_ARG;
  *out = nullptr;
  if (k < 1 || m < 1 || m > RS_POLY_MAX_M || (w != 8 && w != 16)) return RS_ERR_INVALID_ARG;
  const int n = k + m;
  if (n > RS_POLY_MAX_N || (uint32_t)n > (1u << w) - 1) return RS_ERR_INVALID_ARG;
  auto *P = new (std::nothrow) rs_poly_plan();
  if (!P) return RS_ERR_NOMEM;
  if (!P->F.init(w, prim_poly)) {
    delete P;
    return RS_ERR_NOT_PRIMITIVE;
  }
  P->k = k; P->m = m; P->w = w; P->n = n; P->poly = prim_poly;
  P->g = rsb::generator_poly(P->F, m);
  P->pmap = rsb::parity_map(P->F, k, m, P->g);
  P->sliced = rsb::sliced_available(k, m, w, prim_poly);
  std::memset(&P->enc_gp, 0, sizeof(P->enc_gp));
  P->enc_gp.n_in = k;
  P->enc_gp.n_out = m;
  for (int j = 0; j < k; ++j) P->enc_gp.in_blk[j] = (uint8_t)j;
  for (int i = 0; i < m; ++i) P->enc_gp.out_blk[i] = (uint8_t)(k + i);
  pack_generic_tables(P->F, w, P->pmap, m, k, P->enc_tab);
  *out = P;
  return RS_OK;
}

void rs_poly_plan_destroy(rs_poly_plan *plan) { delete plan; }

rs_status rs_poly_plan_set_jit(rs_poly_plan *P, int mode) {
  if (!P || mode < RS_JIT_OFF || mode > RS_JIT_SYNC) return RS_ERR_INVALID_ARG;
  P->jit_mode = mode;
  return RS_OK;
}

rs_status rs_poly_plan_set_read_policy(rs_poly_plan *P, int policy) {
  if (!P || (policy != RS_READ_ALL_SURVIVORS && policy != RS_READ_K_SURVIVORS)) return RS_ERR_INVALID_ARG;
  std::lock_guard<std::mutex> lock(P->mu);
  if (P->read_policy == policy) return RS_OK;
  P->read_policy = policy;
  P->cache.clear();
  for (auto it = P->jit.begin(); it != P->jit.end();) {
    if (it->first.first == kJitDecode) {  // erasure-pattern kernels depend on the policy
      P->retired.push_back(it->second);
      it = P->jit.erase(it);
    } else {
      ++it;
    }
  }
  return RS_OK;
}

rs_status rs_poly_prepare(const rs_poly_plan *P, const int32_t *erasures, size_t n_rows) {
  NvtxRange nvtx_("rs_poly_prepare");
  if (!P || (n_rows && !erasures)) return RS_ERR_INVALID_ARG;
  std::vector<std::vector<int>> rows(n_rows);
  for (size_t s = 0; s < n_rows; ++s) {
    rs_status rc = parse_row(P, erasures + s * (size_t)P->m, P->m, rows[s], true);
    if (rc) return rc;
  }
  std::vector<std::shared_ptr<const PatternHost>> pats;
  std::vector<MaskKey> keys;
  std::vector<int32_t> idx;
  rs_status rc = collect_patterns(P, rows, pats, keys, idx);
  if (rc) return rc;
  if (P->jit_mode == RS_JIT_OFF) return RS_OK;
  if (!P->sliced && jit_eligible(*P, P->m)) {
    std::vector<int> in(P->k), out(P->m);
    for (int j = 0; j < P->k; ++j) in[j] = j;
    for (int i = 0; i < P->m; ++i) out[i] = P->k + i;
    jit_get(*P, kEncodeKey, [&] { return encoder_spec(*P); }, false);
  }
  for (size_t i = 0; i < pats.size(); ++i) pattern_jit(*P, *pats[i], keys[i], false);  // queue all first
  std::vector<std::shared_ptr<JitEntry>> wait;
  {
    std::lock_guard<std::mutex> lock(P->mu);
    for (auto &kv : P->jit) wait.push_back(kv.second);
  }
  for (auto &e : wait)
    if (e->fut.valid()) e->fut.wait();
  side_streams(*P);  // the decode chains' side streams, created here rather than in the first call
  warm_sync();
  return RS_OK;
}

rs_status rs_poly_prepare_all(const rs_poly_plan *P, int max_t, size_t max_patterns) {
  NvtxRange nvtx_("rs_poly_prepare_all");
  if (!P || max_t < 0 || max_t > P->m) return RS_ERR_INVALID_ARG;
  const int n = P->n, m = P->m;
  uint64_t total = 0;
  for (int t = 1; t <= max_t; ++t) {  // C(n, t), exact in 64 bits for these sizes
    uint64_t c = 1;
    for (int q = 0; q < t; ++q) c = c * (uint64_t)(n - q) / (uint64_t)(q + 1);
    total += c;
    if (total > max_patterns || total > kMaxJitKernels) return RS_ERR_INVALID_ARG;
  }
  if (total == 0) return RS_OK;
  std::vector<int32_t> rows;
  rows.reserve((size_t)total * (size_t)m);
  std::vector<int> e;
  for (int t = 1; t <= max_t; ++t) {  // lexicographic t-subsets of [0, n)
    e.resize(t);
    for (int q = 0; q < t; ++q) e[q] = q;
    for (;;) {
      for (int q = 0; q < m; ++q) rows.push_back(q < t ? e[q] : -1);
      int q = t - 1;
      while (q >= 0 && e[q] == n - t + q) --q;
      if (q < 0) break;
      ++e[q];
      for (int r = q + 1; r < t; ++r) e[r] = e[r - 1] + 1;
    }
  }
  return rs_poly_prepare(P, rows.data(), (size_t)total);
}

size_t rs_poly_jit_source(const rs_poly_plan *P, const int *erasures, int n_erasures, char *buf, size_t cap) {
  if (!P || n_erasures < 0 || n_erasures > P->m || (n_erasures && !erasures)) return 0;
  rsb::jit::Spec spec;
  if (n_erasures == 0) {
    if (!jit_eligible(*P, P->m)) return 0;
    std::vector<int> in(P->k), out(P->m);
    for (int j = 0; j < P->k; ++j) in[j] = j;
    for (int i = 0; i < P->m; ++i) out[i] = P->k + i;
    spec = encoder_spec(*P);
  } else {
    std::vector<int32_t> row(erasures, erasures + n_erasures);
    std::vector<int> er;
    if (parse_row(P, row.data(), n_erasures, er, false) || !jit_eligible(*P, (int)er.size())) return 0;
    auto ph = build_pattern(*P, er);
    if (!ph) return 0;
    spec = decoder_spec(*P, *ph);
  }
  const std::string s = rsb::jit::source(P->F, spec, nullptr);
  if (buf && cap) {
    const size_t nc = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), nc);
    buf[nc] = 0;
  }
  return s.size();
}


rs_status rs_poly_ablation_decode(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t stripe_stride,
                                  size_t block_stride, size_t block_bytes, const int *erasures, int n_erasures,
                                  int opt_mask, void *stream) {
  NvtxRange nvtx_("rs_poly_ablation_decode");
  if (!P || P->w != 8 || P->n > 32 || n_erasures < 1 || n_erasures > std::min(P->m, 8) || !erasures ||
      opt_mask < 0 || opt_mask > 7)
    return RS_ERR_INVALID_ARG;
  rs_status rc = check_strided(P, stripes, n_stripes, stripe_stride, block_stride, block_bytes);
  if (rc) return rc;
  std::vector<int> er;
  rc = parse_row(P, erasures, n_erasures, er, false);
  if (rc) return rc;
  if (n_stripes == 0) return RS_OK;
  const Field &F = P->F;
  const int t = (int)er.size(), n = P->n;
  // consts: exp[512], log[256], apow[8][32] (alpha^{j*p}, row stride n), vinv[8][8] (row stride t)
  std::vector<uint8_t> c(768 + 8 * 32 + 8 * 8, 0);
  for (int i = 0; i < 512; ++i) c[i] = (uint8_t)F.alpha_pow((uint64_t)i);
  for (int v = 1; v < 256; ++v) c[512 + v] = (uint8_t)F.log_[v];
  for (int j = 0; j < t; ++j)
    for (int p = 0; p < n; ++p) c[768 + j * n + p] = (uint8_t)F.alpha_pow((uint64_t)j * (uint64_t)p);
  std::vector<uint32_t> V((size_t)t * t);
  for (int j = 0; j < t; ++j)
    for (int e = 0; e < t; ++e)
      V[(size_t)j * t + e] = F.alpha_pow((uint64_t)j * (uint64_t)rsb::position(er[e], P->k, P->m));
  if (!rsb::invert(F, V, t)) return RS_ERR_INVALID_ARG;
  for (int i = 0; i < t * t; ++i) c[768 + 256 + i] = (uint8_t)V[i];
  Blob b;
  const size_t off = b.add(c.data(), c.size());
  DevBlob d;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = d.upload(*P, b, st);
  Geometry G = strided(P, stripes, n_stripes, stripe_stride, block_stride, block_bytes);
  if (e == cudaSuccess)
    e = rsb::launch_polyrs_ablation(G.L, n_stripes, block_bytes, P->k, P->m, er.data(), t, d.p + off, opt_mask,
                                    sm_count(), st);
  cudaError_t ef = d.release();
  return cuda_status(e != cudaSuccess ? e : ef);
}

rs_status rs_poly_verify_batch(const rs_poly_plan *P, const void *stripes, size_t n_stripes, size_t stripe_stride,
                               size_t block_stride, size_t block_bytes, unsigned *flags, void *stream) {
  NvtxRange nvtx_("rs_poly_verify_batch");
  rs_status rc = check_strided(P, const_cast<void *>(stripes), n_stripes, stripe_stride, block_stride, block_bytes);
  if (rc) return rc;
  if (n_stripes == 0) return RS_OK;
  if (!flags) return RS_ERR_INVALID_ARG;
  return verify_impl(P, strided(P, const_cast<void *>(stripes), n_stripes, stripe_stride, block_stride, block_bytes),
                     flags, static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_plan_stats(const rs_poly_plan *P, rs_poly_stats *out) {
  if (!P || !out) return RS_ERR_INVALID_ARG;
  std::memset(out, 0, sizeof(*out));
  std::lock_guard<std::mutex> lock(P->mu);
  out->patterns = P->cache.size();
  for (auto &kv : P->jit) {
    if (!kv.second->ready()) out->jit_pending++;
    else if (const rsb::jit::Kernel *kk = kv.second->kernel()) {
      out->jit_ready++;
      out->jit_cache_hits += kk->cached ? 1 : 0;
    } else {
      out->jit_failed++;
    }
  }
  out->jit_launches = P->jit_launches.load();
  out->table_launches = P->table_launches.load();
  out->jit_available = rsb::jit::available() ? 1 : 0;
  out->jit_mode = P->jit_mode;
  return RS_OK;
}

rs_status rs_poly_plan_info(const rs_poly_plan *P, uint32_t *g_out, uint32_t *pmap_out) {
  if (!P) return RS_ERR_INVALID_ARG;
  if (g_out) std::memcpy(g_out, P->g.data(), sizeof(uint32_t) * P->g.size());
  if (pmap_out) std::memcpy(pmap_out, P->pmap.data(), sizeof(uint32_t) * P->pmap.size());
  return RS_OK;
}

int rs_poly_plan_kernel_kind(const rs_poly_plan *P) { return P && P->sliced ? 1 : 0; }

rs_status rs_poly_encode(const rs_poly_plan *P, const void *const *data, void *const *parity, size_t block_bytes,
                         void *stream) {
  NvtxRange nvtx_("rs_poly_encode");
  rs_status rc = check_geometry(P, block_bytes);
  if (rc) return rc;
  if (!data || !parity) return RS_ERR_INVALID_ARG;
  std::vector<uint64_t> ptrs(P->n);
  bool a32 = true, a16 = true;
  const uint64_t sa = (uint64_t)(P->w / 8);
  for (int b = 0; b < P->n; ++b) {
    const void *p = b < P->k ? data[b] : parity[b - P->k];
    if (!p) return RS_ERR_INVALID_ARG;
    ptrs[b] = reinterpret_cast<uint64_t>(p);
    if (ptrs[b] % sa) return RS_ERR_GEOMETRY;
    a32 = a32 && ptr_aligned(ptrs[b], 32);
    a16 = a16 && ptr_aligned(ptrs[b], 16);
  }
  Geometry G;
  G.L.n = P->n;
  G.n_stripes = 1;
  G.block_bytes = block_bytes;
  G.aligned32 = a32;
  G.aligned16 = a16;
  return encode_impl(P, G, ptrs.data(), static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_decode(const rs_poly_plan *P, void *const *blocks, size_t block_bytes, const int *erasures,
                         int n_erasures, void *stream) {
  NvtxRange nvtx_("rs_poly_decode");
  rs_status rc = check_geometry(P, block_bytes);
  if (rc) return rc;
  if (!blocks || n_erasures < 0 || (n_erasures > 0 && !erasures)) return RS_ERR_INVALID_ARG;
  if (n_erasures > P->m) return RS_ERR_TOO_MANY_ERASURES;
  std::vector<std::vector<int>> rows(1);
  std::vector<int32_t> row(erasures, erasures + n_erasures);
  rc = parse_row(P, row.data(), n_erasures, rows[0], false);
  if (rc) return rc;
  if (rows[0].empty()) return RS_OK;
  std::vector<uint64_t> ptrs(P->n);
  bool a32 = true, a16 = true;
  const uint64_t sa = (uint64_t)(P->w / 8);
  for (int b = 0; b < P->n; ++b) {
    if (!blocks[b]) return RS_ERR_INVALID_ARG;
    ptrs[b] = reinterpret_cast<uint64_t>(blocks[b]);
    if (ptrs[b] % sa) return RS_ERR_GEOMETRY;
    a32 = a32 && ptr_aligned(ptrs[b], 32);
    a16 = a16 && ptr_aligned(ptrs[b], 16);
  }
  Geometry G;
  G.L.n = P->n;
  G.n_stripes = 1;
  G.block_bytes = block_bytes;
  G.aligned32 = a32;
  G.aligned16 = a16;
  return decode_impl(P, G, ptrs.data(), rows, static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_encode_batch(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t stripe_stride,
                               size_t block_stride, size_t block_bytes, void *stream) {
  NvtxRange nvtx_("rs_poly_encode_batch");
  rs_status rc = check_strided(P, stripes, n_stripes, stripe_stride, block_stride, block_bytes);
  if (rc) return rc;
  if (n_stripes == 0) return RS_OK;
  Geometry G = strided(P, stripes, n_stripes, stripe_stride, block_stride, block_bytes);
  return encode_impl(P, G, nullptr, static_cast<cudaStream_t>(stream));
}

rs_status rs_poly_decode_batch(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t stripe_stride,
                               size_t block_stride, size_t block_bytes, const int32_t *erasures, void *stream) {
  NvtxRange nvtx_("rs_poly_decode_batch");
  rs_status rc = check_strided(P, stripes, n_stripes, stripe_stride, block_stride, block_bytes);
  if (rc) return rc;
  if (n_stripes == 0) return RS_OK;
  if (!erasures) return RS_ERR_INVALID_ARG;
  std::vector<std::vector<int>> rows(n_stripes);
  for (size_t s = 0; s < n_stripes; ++s) {
    rc = parse_row(P, erasures + s * (size_t)P->m, P->m, rows[s], true);
    if (rc) return rc;
  }
  Geometry G = strided(P, stripes, n_stripes, stripe_stride, block_stride, block_bytes);
  return decode_impl(P, G, nullptr, rows, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

