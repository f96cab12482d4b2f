// plan_internal.hpp -- types and helpers shared by the library's host files (plan.cpp,
// linear.cpp, host_pipeline.cpp).  Internal: not part of the C ABI.
#pragma once
#include <algorithm>
#include <array>
#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <future>
#include <map>
#include <string>
#include <memory>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only; a no-op unless a profiler (nsys, ncu) is attached

#include "../../include/rs_poly.h"
#include "gf.hpp"
#include "jit.hpp"
#include "rs_kernels.cuh"

namespace rsp {

using rsb::Field;

struct PatternHost {
  std::vector<int> erased;  // row order of W / R: ascending API index
  std::vector<int> surv;    // survivors, ascending API index (columns of R)
  std::vector<uint32_t> R;  // t x (n-t) decode matrix V_E^{-1} A_E
  std::vector<uint32_t> Vinv;  // t x t, V_E^{-1} (Step 2)
  // Syndrome-form (w16 JIT) solve: unknowns U (= E, or E + the survivors not read under
  // RS_READ_K_SURVIVORS), Hm = rows E of V_U^{-1} (t x |U|), |U| syndromes used.
  std::vector<int> unknown;
  std::vector<uint32_t> Hm;
  rsb::SlicedPat sp{};
  std::vector<uint8_t> wtab;  // sliced W tables
  rsb::GenericPat gp{};
  std::vector<uint8_t> rtab;  // generic R tables (all output groups)
};

using MaskKey = std::array<uint64_t, 4>;
// JIT cache key: (kind, mask).  Decode: the erased mask; encode: 0; linear job: its id.
enum JitKind { kJitDecode = 0, kJitEncode = 1, kJitLinear = 2, kJitVerify = 3 };
using JitKey = std::pair<int, MaskKey>;

// A "linear job": per stripe the kernels see nv virtual blocks (a pointer table) and
// compute out_r = sum_v M[r][v] in_v for the nout virtual blocks out[r] (which may also
// be inputs: in place).  Used by the diff-update, the partial encoder of the
// cross-GPU placement and the XOR reduction.  Cached per plan by a signature string.
struct LinearHost {
  int id = 0;               // JIT key
  int nv = 0, nout = 0;
  std::vector<int> out;     // virtual indices of the outputs
  std::vector<uint32_t> M;  // nout x nv
  int group_blocks = 0;     // JIT CSE group (0 = by field)
  rsb::GenericPat gp{};
  std::vector<uint8_t> tab;
};

// A run-time specialised kernel (jit.cpp), compiled once per pattern.
struct JitEntry {
  std::shared_future<std::shared_ptr<rsb::jit::Kernel>> fut;
  bool ready() const { return fut.valid() && fut.wait_for(std::chrono::seconds(0)) == std::future_status::ready; }
  const rsb::jit::Kernel *kernel() const {
    if (!ready()) return nullptr;
    const auto &k = fut.get();
    return (k && k->ok) ? k.get() : nullptr;
  }
};

// Fixed pool of compile workers shared by all plans (NVRTC is thread-safe).
class CompilePool {
 public:
  static CompilePool &get() {
    static CompilePool p;
    return p;
  }
  void submit(std::function<void()> fn) {
    std::lock_guard<std::mutex> l(mu_);
    q_.push_back(std::move(fn));
    cv_.notify_one();
  }
  // True once the process is tearing the pool down: queued jobs then resolve their
  // promises with a failed kernel instead of compiling (fast exit, no waiter left hanging).
  static bool stopping() { return stopping_flag().load(); }
  ~CompilePool() {
    stopping_flag().store(true);
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto &t : th_) t.join();
  }

 private:
  CompilePool() {
    unsigned n = std::max(2u, std::min(16u, std::thread::hardware_concurrency()));
    for (unsigned i = 0; i < n; ++i) th_.emplace_back([this] { run(); });
  }
  void run() {
    for (;;) {
      std::function<void()> fn;
      {
        std::unique_lock<std::mutex> l(mu_);
        cv_.wait(l, [this] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        fn = std::move(q_.front());
        q_.pop_front();
      }
      fn();
    }
  }
  static std::atomic<bool> &stopping_flag() {
    static std::atomic<bool> f{false};
    return f;
  }
  std::mutex mu_;
  std::condition_variable cv_;
  std::deque<std::function<void()>> q_;
  std::vector<std::thread> th_;
  bool stop_ = false;
};

}  // namespace rsp

using namespace rsp;  // internal header: the .cpp files of the library only

struct rs_poly_plan {
  int k = 0, m = 0, w = 0, n = 0;
  uint32_t poly = 0;
  Field F;
  std::vector<uint32_t> g, pmap;
  bool sliced = false;
  rsb::GenericPat enc_gp{};
  std::vector<uint8_t> enc_tab;
  mutable std::mutex mu;
  mutable std::map<MaskKey, std::shared_ptr<const PatternHost>> cache;
  mutable std::map<std::string, std::shared_ptr<const LinearHost>> lin_cache;  // linear jobs by signature
  // run-time specialised kernels: decode patterns (key = erased mask) and, for codes
  // without a compiled network, the encoder (key = kEncodeKey)
  int jit_mode = RS_JIT_BACKGROUND;
  int read_policy = RS_READ_ALL_SURVIVORS;
  mutable std::map<JitKey, std::shared_ptr<JitEntry>> jit;
  std::vector<std::shared_ptr<JitEntry>> retired;  // dropped by a policy change, released at destroy
  mutable std::map<int, std::vector<cudaStream_t>> pool;  // device -> side streams for concurrent launches
  mutable std::atomic<uint64_t> jit_launches{0}, table_launches{0};
  // pinned host slots for the per-call constant blob: a pageable cudaMemcpyAsync may
  // wait for the stream, stalling the host between back-to-back calls
  struct PinnedSlot {
    uint8_t *p = nullptr;
    size_t cap = 0;
    int dev = 0;
    cudaEvent_t ev = nullptr;
    bool busy = false;
    uint64_t seq = 0;  // order of last use
  };
  mutable uint64_t stage_seq = 0;
  mutable std::mutex stage_mu;
  mutable std::vector<PinnedSlot> stage;
  // device staging of the host entry points (rs_poly_*_host), one per device, reused
  // across calls: a fresh stream-ordered allocation per call would be re-mapped each
  // time the default pool trims at the call's final synchronize
  struct Staging {
    std::mutex busy;
    uint8_t *p = nullptr;
    size_t cap = 0;
  };
  mutable std::map<int, std::unique_ptr<Staging>> staging;
  mutable std::map<int, uint8_t *> enc_dev;  // device -> encode tail constants
  mutable std::map<int, uint8_t *> ver_dev;  // device -> verify constants (A = alpha^{j pos})
  ~rs_poly_plan() {
    for (auto *mp : {&enc_dev, &ver_dev})
      for (auto &kv : *mp) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first);
        cudaFree(kv.second);
        cudaSetDevice(cur);
      }
    for (auto &kv : staging)
      if (kv.second->p) {
        int cur = 0;
        cudaGetDevice(&cur);
        cudaSetDevice(kv.first);
        cudaFree(kv.second->p);
        cudaSetDevice(cur);
      }
    for (auto &sl : stage) {
      if (sl.ev) {
        cudaEventSynchronize(sl.ev);
        cudaEventDestroy(sl.ev);
      }
      if (sl.p) cudaFreeHost(sl.p);
    }
    for (auto &kv : jit) retired.push_back(kv.second);
    for (auto &e : retired) {
      if (e->fut.valid()) {
        auto k = e->fut.get();
        if (k) rsb::jit::release(*k);
      }
    }
    for (auto &kv : pool)
      for (cudaStream_t s : kv.second) cudaStreamDestroy(s);
  }
};

namespace rsp {

constexpr int kGenericThreads = 256;
constexpr int kSlicedThreads = 128;
constexpr uint32_t kSlicedUnitsPerCta = kSlicedThreads * 8;
constexpr uint64_t kGenericChunk = 64 * 1024;
const JitKey kEncodeKey{kJitEncode, MaskKey{0, 0, 0, 0}};
// At most this many JIT modules per plan (each is ~50-150 KB of code); RS(10,4) has 1001
// erasure patterns, RS(12,4) 2516.  Beyond it, new patterns run on the table kernels.
constexpr size_t kMaxJitKernels = 8192;
constexpr size_t kEncTablesOff = (sizeof(rsb::GenericPat) + 15) & ~(size_t)15;

// Per-call device blob: uploaded with one H2D copy, freed stream-ordered.
struct Blob {
  std::vector<uint8_t> h;
  size_t add(const void *p, size_t bytes) {
    size_t off = (h.size() + 15) & ~(size_t)15;
    h.resize(off + bytes);
    if (p && bytes) std::memcpy(h.data() + off, p, bytes);
    return off;
  }
};

struct Geometry {
  rsb::Layout L{};
  uint64_t n_stripes = 0, block_bytes = 0;
  bool aligned32 = false, aligned16 = false;
};

cudaError_t upload_pinned(const rs_poly_plan &P, void *dst, const void *src, size_t bytes, cudaStream_t s);

cudaError_t blob_pool(cudaMemPool_t *out);  // plan.cpp

struct DevBlob {
  uint8_t *p = nullptr;
  cudaStream_t st = nullptr;
  cudaError_t upload(const rs_poly_plan &P, const Blob &b, cudaStream_t s) {
    st = s;
    // The blob is copied from a pinned slot that later calls reuse: a CUDA graph replaying
    // this copy would read another call's constants.  Refuse to be captured.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
      return cudaErrorStreamCaptureUnsupported;
    cudaMemPool_t pool = nullptr;
    cudaError_t e = blob_pool(&pool);
    if (e == cudaSuccess)
      e = cudaMallocFromPoolAsync(reinterpret_cast<void **>(&p), std::max<size_t>(b.h.size(), 16), pool, s);
    if (e != cudaSuccess) return e;
    return upload_pinned(P, p, b.h.data(), b.h.size(), s);
  }
  cudaError_t release() {
    cudaError_t e = p ? cudaFreeAsync(p, st) : cudaSuccess;
    p = nullptr;
    return e;
  }
};

// NVTX range around a C ABI call (SURVEY section 5 tracing): names the library's work in
// profiler timelines.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};

// ---- shared helpers (plan.cpp unless noted) ---------------------------------------
inline bool ptr_aligned(uint64_t v, uint64_t a) { return (v % a) == 0; }
void pack_generic_tables(const Field &F, int w, const std::vector<uint32_t> &M, int n_out, int n_in,
                         std::vector<uint8_t> &out);
std::shared_ptr<const PatternHost> build_pattern(const rs_poly_plan &P, const std::vector<int> &er);
rs_status cuda_status(cudaError_t e);
bool jit_eligible(const rs_poly_plan &P, int n_out);
rsb::jit::Spec jit_spec(const rs_poly_plan &P, const std::vector<int> &in, const std::vector<int> &out,
                        const std::vector<uint32_t> &M);
rsb::jit::Spec encoder_spec(const rs_poly_plan &P);
rsb::jit::Spec decoder_spec(const rs_poly_plan &P, const PatternHost &ph);
const rsb::jit::Kernel *jit_get(const rs_poly_plan &P, const JitKey &key, const std::function<rsb::jit::Spec()> &mk,
                                bool wait);
std::vector<cudaStream_t> side_streams(const rs_poly_plan &P);
uint64_t body_units_of(const rs_poly_plan &P, const Geometry &G);
int sm_count();
uint32_t units_per_cta_for(uint64_t total, int w);
cudaError_t launch_jit(const rsb::jit::Kernel &k, const Geometry &G, const int32_t *stripes, uint64_t n_sel,
                       uint64_t body_units, cudaStream_t st, bool pdl = false, uint64_t stripe_base = 0,
                       unsigned *flags = nullptr);
cudaError_t launch_sliced_body(const rs_poly_plan &P, bool decode, const Geometry &G, uint64_t body_units,
                               const uint8_t *dev, size_t pats_off, size_t idx_off, size_t tables_off,
                               cudaStream_t st);
cudaError_t launch_generic_range(const rs_poly_plan &P, const Geometry &G, uint64_t col_begin, uint64_t col_end,
                                 const uint8_t *dev, size_t pats_off, size_t idx_off, size_t tables_off,
                                 uint32_t groups, uint32_t smem, cudaStream_t st, unsigned *flags = nullptr);
cudaError_t upload_pinned(const rs_poly_plan &P, void *dst, const void *src, size_t bytes, cudaStream_t s);
rs_status check_geometry(const rs_poly_plan *P, size_t block_bytes);
rs_status check_strided(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t ss, size_t bs, size_t B);
Geometry strided(const rs_poly_plan *P, void *stripes, size_t n_stripes, size_t ss, size_t bs, size_t B);
rs_status parse_row(const rs_poly_plan *P, const int32_t *row, int count, std::vector<int> &out, bool allow_pad);
rs_status encode_impl(const rs_poly_plan *P, Geometry G, const uint64_t *ptrs, cudaStream_t st);
rs_status decode_impl(const rs_poly_plan *P, Geometry G, const uint64_t *ptrs,
                      const std::vector<std::vector<int>> &rows, cudaStream_t st);
rs_status collect_patterns(const rs_poly_plan *P, const std::vector<std::vector<int>> &rows,
                           std::vector<std::shared_ptr<const PatternHost>> &pats, std::vector<MaskKey> &keys,
                           std::vector<int32_t> &idx);
const rsb::jit::Kernel *pattern_jit(const rs_poly_plan &P, const PatternHost &ph, const MaskKey &key, bool wait);

// linear.cpp: diff-update, partial encode, XOR reduction
std::shared_ptr<const LinearHost> update_host(const rs_poly_plan &P, const std::vector<int> &idx);
rsb::jit::Spec linear_spec(const rs_poly_plan &P, const LinearHost &lh);
rs_status parse_update(const rs_poly_plan *P, const int *data_idx, int c, std::vector<int> &sorted,
                       std::vector<int> &order);

}  // namespace rsp
