// host_pipeline.cpp -- rs_poly_encode_host / rs_poly_decode_host: end to end from HOST
// memory (include/rs_poly.h), chunks of stripes streamed through plan-owned device staging.
#include "plan_internal.hpp"

// ===========================================================================
// End to end from host memory: chunks of stripes stream through device
// staging buffers, H2D -> kernels -> D2H, overlapped over kNumLanes streams.
// ===========================================================================
namespace rsp {

constexpr int kNumLanes = 3;
constexpr uint64_t kStagingTarget = 256ull << 20;  // bytes of staging per lane

rs_status host_impl(const rs_poly_plan *P, bool decode, uint8_t *host, size_t n_stripes, size_t ss, size_t bs,
                    size_t B, const int32_t *erasures, cudaStream_t user, uint64_t *h2d, uint64_t *d2h) {
  rs_status rc = check_strided(P, host, n_stripes, ss, bs, B);
  if (rc) return rc;
  std::vector<std::vector<int>> rows;
  if (decode) {
    if (!erasures) return RS_ERR_INVALID_ARG;
    rows.resize(n_stripes);
    for (size_t s = 0; s < n_stripes; ++s) {
      rc = parse_row(P, erasures + s * (size_t)P->m, P->m, rows[s], true);
      if (rc) return rc;
    }
  }
  uint64_t in_bytes = 0, out_bytes = 0;
  if (n_stripes == 0) {
    if (h2d) *h2d = 0;
    if (d2h) *d2h = 0;
    return RS_OK;
  }
  const int n = P->n;
  const uint64_t Bp = (B + 255) & ~255ull;  // device block pitch (32-byte aligned for the sliced path)
  const uint64_t stripe_dev = Bp * (uint64_t)n;
  const uint64_t per_chunk = std::max<uint64_t>(1, kStagingTarget / stripe_dev);
  cudaStream_t lanes[kNumLanes] = {};
  uint8_t *stage[kNumLanes] = {};
  bool owned_async = false;  // staging from cudaMallocAsync (plan staging busy in another call)
  cudaEvent_t start = nullptr;
  cudaError_t e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(start, user);
  const size_t lane_bytes = per_chunk * stripe_dev;
  rs_poly_plan::Staging *sg = nullptr;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(P->mu);
    auto &slot = P->staging[dev];
    if (!slot) slot = std::make_unique<rs_poly_plan::Staging>();
    if (slot->busy.try_lock()) sg = slot.get();
  }
  if (sg && e == cudaSuccess && sg->cap < lane_bytes * kNumLanes) {
    if (sg->p) cudaFree(sg->p);  // idle: its last user synchronized before releasing it
    sg->p = nullptr;
    sg->cap = 0;
    e = cudaMalloc(reinterpret_cast<void **>(&sg->p), lane_bytes * kNumLanes);
    if (e == cudaSuccess) sg->cap = lane_bytes * kNumLanes;
  }
  owned_async = sg == nullptr;
  for (int l = 0; l < kNumLanes && e == cudaSuccess; ++l) {
    e = cudaStreamCreateWithFlags(&lanes[l], cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(lanes[l], start, 0);
    if (e != cudaSuccess) break;
    if (owned_async) e = cudaMallocAsync(reinterpret_cast<void **>(&stage[l]), lane_bytes, lanes[l]);
    else stage[l] = sg->p + (size_t)l * lane_bytes;
  }
  rc = cuda_status(e);
  for (size_t s0 = 0, ci = 0; rc == RS_OK && s0 < n_stripes; s0 += per_chunk, ++ci) {
    const size_t cnt = std::min<size_t>(per_chunk, n_stripes - s0);
    const int l = (int)(ci % kNumLanes);
    cudaStream_t st = lanes[l];
    // inputs host -> device
    for (size_t s = s0; s < s0 + cnt && e == cudaSuccess; ++s) {
      uint8_t *hs = host + s * ss, *ds = stage[l] + (s - s0) * stripe_dev;
      if (!decode) {
        e = cudaMemcpy2DAsync(ds, Bp, hs, bs, B, (size_t)P->k, cudaMemcpyHostToDevice, st);
        in_bytes += (uint64_t)P->k * B;
      } else {
        std::vector<char> er(n, 0);
        for (int b : rows[s]) er[b] = 1;
        if (rows[s].empty()) continue;
        for (int b = 0; b < n && e == cudaSuccess; ++b)
          if (!er[b]) {
            e = cudaMemcpyAsync(ds + b * Bp, hs + b * bs, B, cudaMemcpyHostToDevice, st);
            in_bytes += B;
          }
      }
    }
    if (e != cudaSuccess) { rc = cuda_status(e); break; }
    Geometry G = strided(P, stage[l], cnt, stripe_dev, Bp, B);
    if (!decode) {
      rc = encode_impl(P, G, nullptr, st);
    } else {
      std::vector<std::vector<int>> sub(rows.begin() + s0, rows.begin() + s0 + cnt);
      rc = decode_impl(P, G, nullptr, sub, st);
    }
    if (rc) break;
    // outputs device -> host
    for (size_t s = s0; s < s0 + cnt && e == cudaSuccess; ++s) {
      uint8_t *hs = host + s * ss, *ds = stage[l] + (s - s0) * stripe_dev;
      if (!decode) {
        e = cudaMemcpy2DAsync(hs + (size_t)P->k * bs, bs, ds + (size_t)P->k * Bp, Bp, B, (size_t)P->m,
                              cudaMemcpyDeviceToHost, st);
        out_bytes += (uint64_t)P->m * B;
      } else {
        for (int b : rows[s]) {
          if (e != cudaSuccess) break;
          e = cudaMemcpyAsync(hs + b * bs, ds + b * Bp, B, cudaMemcpyDeviceToHost, st);
          out_bytes += B;
        }
      }
    }
    if (e != cudaSuccess) rc = cuda_status(e);
  }
  for (int l = 0; l < kNumLanes; ++l) {
    if (stage[l] && owned_async) cudaFreeAsync(stage[l], lanes[l]);
    if (lanes[l]) {
      cudaError_t es = cudaStreamSynchronize(lanes[l]);
      if (rc == RS_OK && es != cudaSuccess) rc = cuda_status(es);
      cudaStreamDestroy(lanes[l]);
    }
  }
  if (sg) sg->busy.unlock();
  if (start) cudaEventDestroy(start);
  if (h2d) *h2d = in_bytes;
  if (d2h) *d2h = out_bytes;
  return rc;
}

}  // namespace rsp

extern "C" {

rs_status rs_poly_encode_host(const rs_poly_plan *P, void *host_stripes, size_t n_stripes, size_t stripe_stride,
                              size_t block_stride, size_t block_bytes, void *stream, uint64_t *h2d_bytes,
                              uint64_t *d2h_bytes) {
  NvtxRange nvtx_("rs_poly_encode_host");
  return host_impl(P, false, static_cast<uint8_t *>(host_stripes), n_stripes, stripe_stride, block_stride,
                   block_bytes, nullptr, static_cast<cudaStream_t>(stream), h2d_bytes, d2h_bytes);
}

rs_status rs_poly_decode_host(const rs_poly_plan *P, void *host_stripes, size_t n_stripes, size_t stripe_stride,
                              size_t block_stride, size_t block_bytes, const int32_t *erasures, void *stream,
                              uint64_t *h2d_bytes, uint64_t *d2h_bytes) {
  NvtxRange nvtx_("rs_poly_decode_host");
  return host_impl(P, true, static_cast<uint8_t *>(host_stripes), n_stripes, stripe_stride, block_stride,
                   block_bytes, erasures, static_cast<cudaStream_t>(stream), h2d_bytes, d2h_bytes);
}

}  // extern "C"
