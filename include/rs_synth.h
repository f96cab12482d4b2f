/*
 * rs_synth.h -- seeded synthetic inputs on the GPU (NOT part of the method).
 *
 * Device twin of synth/__init__.py (same counter-based generator, bit for bit;
 * tests/test_gpu_parity.py::test_synth_matches_host checks it).  It holds no
 * Reed-Solomon or GF(2^w) arithmetic; the benchmark uses it to fill 8-30 GiB
 * stripe batches in HBM without a host round trip.
 *
 * Data word q (8 bytes, little-endian) of data block j of stripe s:
 *     splitmix64(seed<<48 | (stripe0+s)<<32 | j<<24 | q)
 * (the paper stages uniform random data in memory).
 */
#ifndef RS_SYNTH_H
#define RS_SYNTH_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Fill data blocks 0..k-1 of n_stripes stripes (DEVICE memory, strided layout
 * as in rs_poly_encode_batch).  Returns 0 on success, -1 on bad arguments
 * (seed >= 2^16, stripe0 + n_stripes > 2^16, k > 254, block_bytes > 2^27),
 * or the cudaError_t of the launch. */
int rs_synth_fill(void *stripes, size_t n_stripes, size_t stripe_stride, size_t block_stride,
                  size_t block_bytes, int k, uint32_t seed, uint32_t stripe0, void *stream);

#ifdef __cplusplus
}
#endif
#endif
