/*
 * c_api_demo.c -- the library from plain C (no Python, no torch): include/rs_poly.h and
 * include/rs_synth.h against librs_poly.so / librs_synth.so and the CUDA runtime.
 *
 *   gcc -std=c99 -O2 -I include -I /usr/local/cuda/include tools/c_api_demo.c \
 *       -L paper_1312_5155_b200 -lrs_poly -lrs_synth -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1312_5155_b200 -o /tmp/c_api_demo && /tmp/c_api_demo
 *
 * C1-shaped workload (RS(10,4), GF(2^8), one stripe of 10 x 64 KiB): encode, erase four
 * blocks, decode, check every byte came back, verify (scrub) the stripe; then the per-call
 * latency of encode and decode measured with CUDA events (no interpreter in the loop).
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rs_poly.h"
#include "rs_synth.h"

#define CK(x)                                                                         \
  do {                                                                                \
    int rc_ = (int)(x);                                                               \
    if (rc_) {                                                                        \
      fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, rc_);               \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

int main(void) {
  const int k = 10, m = 4, n = 14, reps = 500;
  const size_t B = 64 * 1024, stripe = (size_t)n * B;
  rs_poly_plan *plan = NULL;
  CK(rs_poly_plan_create(k, m, 8, 0x11D, &plan));
  unsigned char *d = NULL, *golden = NULL;
  unsigned *flags = NULL;
  CK(cudaMalloc((void **)&d, stripe));
  CK(cudaMalloc((void **)&golden, stripe));
  CK(cudaMalloc((void **)&flags, sizeof(unsigned)));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  CK(rs_synth_fill(d, 1, stripe, B, B, k, 0, 0, st));
  CK(rs_poly_encode_batch(plan, d, 1, stripe, B, B, st));
  CK(cudaMemcpyAsync(golden, d, stripe, cudaMemcpyDeviceToDevice, st));
  const int32_t er[4] = {3, 8, 10, 11};
  CK(rs_poly_prepare(plan, er, 1));
  for (int e = 0; e < 4; ++e) CK(cudaMemsetAsync(d + (size_t)er[e] * B, 0, B, st));
  CK(rs_poly_decode_batch(plan, d, 1, stripe, B, B, er, st));
  CK(rs_poly_verify_batch(plan, d, 1, stripe, B, B, flags, st));
  CK(cudaStreamSynchronize(st));
  unsigned char *h1 = (unsigned char *)malloc(stripe), *h2 = (unsigned char *)malloc(stripe);
  unsigned hflag = 7;
  CK(cudaMemcpy(h1, d, stripe, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2, golden, stripe, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&hflag, flags, sizeof(unsigned), cudaMemcpyDeviceToHost));
  const int restored = memcmp(h1, h2, stripe) == 0;

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms_enc = 0, ms_dec = 0;
  for (int i = 0; i < 50; ++i) CK(rs_poly_encode_batch(plan, d, 1, stripe, B, B, st));
  CK(cudaEventRecord(e0, st));
  for (int i = 0; i < reps; ++i) CK(rs_poly_encode_batch(plan, d, 1, stripe, B, B, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms_enc, e0, e1));
  for (int i = 0; i < 50; ++i) CK(rs_poly_decode_batch(plan, d, 1, stripe, B, B, er, st));
  CK(cudaEventRecord(e0, st));
  for (int i = 0; i < reps; ++i) CK(rs_poly_decode_batch(plan, d, 1, stripe, B, B, er, st));
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms_dec, e0, e1));
  printf("{\"c_api\": true, \"abi\": %d, \"restored\": %s, \"verify_flag\": %u, "
         "\"c1_encode_us\": %.2f, \"c1_decode_us\": %.2f}\n",
         rs_poly_abi_version(), restored ? "true" : "false", hflag, 1e3f * ms_enc / reps, 1e3f * ms_dec / reps);
  rs_poly_plan_destroy(plan);
  return restored && hflag == 0 ? 0 : 2;
}
