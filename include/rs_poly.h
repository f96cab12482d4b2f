/*
 * rs_poly.h -- C ABI of the B200-native polynomial Reed-Solomon library.
 *
 * The operations are those of Sheykh Esmaili & Datta, "On the Effectiveness of
 * Polynomial Realization of Reed-Solomon Codes for Storage Systems" (arXiv
 * 1312.5155, PAPER.md; "P:n" = PAPER.md line n):
 *   - RS(k,m) over GF(2^w): k data elements are encoded into n = k+m so that any
 *     k of the n recover the object.
 *   - generator polynomial g(x) = prod_{i=0}^{m-1} (x + alpha^i), alpha = 2
 *     (P:170-177);
 *   - encode: parity p(x) = d(x) x^m mod g(x) (Eq. 1-2);
 *   - decode: Step 1 evaluates the survivors at alpha^0..alpha^{t-1}, Step 2
 *     solves the t x t Vandermonde system for the t erased symbols
 *     (P:213-303).  Results are bit-identical to the literal definitions.
 *
 * Layout and conventions:
 *   - A stripe holds n blocks of block_bytes bytes each.  API block index
 *     b in [0,n): 0..k-1 are data, k..n-1 are parity.
 *   - Column c of a stripe = symbol c of every block; each column is an
 *     independent codeword.  Data block j is the coefficient of x^{m+j}
 *     (P:191), parity block i the coefficient of x^i.
 *   - w = 8: one byte per symbol.  w = 16: little-endian uint16 per symbol, so
 *     block_bytes must be even.
 *   - "Device pointer" = CUDA global memory of the current device (e.g. a
 *     torch.cuda tensor's data_ptr()).  Streams are cudaStream_t passed as
 *     void* (NULL = legacy default stream).
 *
 * Ownership: the caller owns every block buffer and stream.  A plan owns its
 * host tables and its decode-pattern cache (mutex-guarded); a plan may be used
 * from several host threads and streams at once.
 *
 * Errors are returned synchronously after argument validation and before any
 * device work; on a validation error nothing is written.  Launch failures
 * return RS_ERR_CUDA; asynchronous device faults surface at stream sync.
 *
 * CUDA graph capture: a call that launches kernels only (arguments by value, plan-
 * owned device constants) may be captured on the caller's stream once the plan has
 * run once on that device: rs_poly_encode_batch, rs_poly_verify_batch, and
 * rs_poly_decode_batch when every pattern of the batch has its JIT kernel (after
 * rs_poly_prepare), the blocks have no ragged tail and the layout is strided (not
 * the pointer-array form) and each pattern's stripes form at most two runs of adjacent
 * stripes on average (a pattern recurring on non-adjacent stripes is launched once per
 * run).  Calls that upload per-call constants (ragged tails, pointer arrays, patterns
 * still without a JIT kernel, patterns scattered over many runs) return RS_ERR_CUDA
 * when the stream is capturing (nothing is enqueued).
 * There is no CPU fallback: every entry point that computes runs CUDA kernels.
 */
#ifndef RS_POLY_H
#define RS_POLY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_POLY_ABI_VERSION 2 /* 2: rs_poly_stats.jit_cache_hits */
#define RS_POLY_MAX_N 255 /* k+m <= 255 (also k+m <= 2^w-1, reading G7) */
#define RS_POLY_MAX_M 32

typedef struct rs_poly_plan rs_poly_plan; /* opaque */

typedef enum {
  RS_OK = 0,
  RS_ERR_INVALID_ARG = 1,       /* null pointer, k<1, m<1, m>RS_POLY_MAX_M, w not 8/16, k+m > min(255, 2^w-1) */
  RS_ERR_NOT_PRIMITIVE = 2,     /* prim_poly not of degree w, or ord(alpha=2) != 2^w-1              */
  RS_ERR_GEOMETRY = 3,          /* block_bytes == 0, block_bytes % (w/8) != 0, pointer/stride not w/8-aligned */
  RS_ERR_TOO_MANY_ERASURES = 4, /* |E| > m: the code recovers at most m erasures                  */
  RS_ERR_BAD_ERASURE = 5,       /* erasure index outside [0,n) or listed twice                              */
  RS_ERR_CUDA = 6,              /* a CUDA runtime call or kernel launch failed                               */
  RS_ERR_NOMEM = 7              /* host or device allocation failed                                          */
} rs_status;

/* ---- plan ------------------------------------------------------------------
 * Builds, on the host: exp/log of GF(2^w) from prim_poly with alpha = 2,
 * g(x), the k x m parity map (column j = x^{m+j} mod g, the
 * generator-matrix form of g) and the kernels' packed constants.
 * No device memory is touched; constants reach the device as kernel
 * parameters / per-call uploads.  *out receives the plan, or NULL on error. */
rs_status rs_poly_plan_create(int k, int m, int w, uint32_t prim_poly, rs_poly_plan **out);
void rs_poly_plan_destroy(rs_poly_plan *plan); /* NULL is a no-op */

/* g_out[0..m] receives g low->high (monic); pmap_out[i*k + j] (m x k,
 * row = parity i, column = data j) the parity map P with p_i = sum_j P[i][j] d_j.
 * Either pointer may be NULL.  Host memory.  Host-only (no GPU needed). */
rs_status rs_poly_plan_info(const rs_poly_plan *plan, uint32_t *g_out, uint32_t *pmap_out);

/* Which kernel family the plan uses: 1 = bit-sliced XOR network specialised at
 * compile time for this (k,m,w,prim_poly); 0 = generic split-nibble tables.   */
int rs_poly_plan_kernel_kind(const rs_poly_plan *plan);

/* ---- single stripe (pointer arrays) ---------------------------------------
 * data:   HOST array of k DEVICE pointers (read only).
 * parity: HOST array of m DEVICE pointers (overwritten with p_0..p_{m-1}).
 * Encode: all-zero data gives all-zero parity. */
rs_status rs_poly_encode(const rs_poly_plan *plan, const void *const *data, void *const *parity,
                         size_t block_bytes, void *stream);

/* blocks: HOST array of n DEVICE pointers, data 0..k-1 then parity k..n-1.
 * erasures: HOST array of n_erasures API block indices, any order, 0 <= n_erasures <= m.
 * Decode: writes the original bytes into exactly the erased blocks
 * (their prior contents are don't-care) and never writes a survivor.
 * n_erasures == 0 is a successful no-op. */
rs_status rs_poly_decode(const rs_poly_plan *plan, void *const *blocks, size_t block_bytes,
                         const int *erasures, int n_erasures, void *stream);

/* ---- batched, strided layout ------------------------------------------------
 * Block b of stripe s lives at stripes + s*stripe_stride + b*block_stride
 * (bytes; DEVICE memory).  The usual layout is [S][n][B]: block_stride = B,
 * stripe_stride = n*B.  Strides must be multiples of w/8.
 * Encode writes blocks k..n-1 of every stripe. */
rs_status rs_poly_encode_batch(const rs_poly_plan *plan, void *stripes, size_t n_stripes,
                               size_t stripe_stride, size_t block_stride, size_t block_bytes, void *stream);

/* erasures: HOST int32 [n_stripes][m], row s lists stripe s's erased API block
 * indices padded with -1 (each stripe may have its own pattern; an all -1 row
 * leaves that stripe untouched).  The per-pattern decode constants (the
 * paper's Opt1/Opt3: alpha powers and the inverted Vandermonde
 * matrix, computed once per pattern) are cached in the plan. */
rs_status rs_poly_decode_batch(const rs_poly_plan *plan, void *stripes, size_t n_stripes,
                               size_t stripe_stride, size_t block_stride, size_t block_bytes,
                               const int32_t *erasures, void *stream);

/* ---- verify (scrub) -----------------------------------------------------------
 * Every codeword vanishes at the roots alpha^0..alpha^{m-1} of g: its m
 * syndromes S_j = sum_p c_p alpha^{j*pos(p)} (Step 1 of the decode, with
 * nothing erased) are zero.  For each stripe of the batch (layout as in
 * rs_poly_encode_batch; nothing is written to it) sets flags[s] = 0 if every column is a
 * codeword, 1 otherwise (silent corruption of any data or parity byte).  flags: DEVICE
 * array of n_stripes uint32, overwritten.  Reads n*B bytes per stripe. */
rs_status rs_poly_verify_batch(const rs_poly_plan *plan, const void *stripes, size_t n_stripes,
                               size_t stripe_stride, size_t block_stride, size_t block_bytes,
                               unsigned *flags, void *stream);

/* ---- end to end from HOST memory ---------------------------------------------
 * Same operations, but `host_stripes` is HOST memory (page-locked for full
 * speed, e.g. cudaHostAlloc / torch pin_memory), laid out as in the batched
 * calls.  The library streams chunks of stripes through device staging
 * buffers on `stream`'s device (3 lanes of ~256 MiB, kept by the plan for reuse
 * and freed by rs_poly_plan_destroy; a call that finds them in use by another
 * thread allocates its own for the call): host->device copy of the inputs
 * (encode: the k data blocks; decode: the n-t survivors), the kernel, and the
 * device->host copy of the outputs (encode: m parity blocks; decode: the t
 * erased blocks), overlapped across chunks.  Returns after the results are in
 * host memory.  *h2d_bytes / *d2h_bytes (optional) receive the bytes copied. */
rs_status rs_poly_encode_host(const rs_poly_plan *plan, void *host_stripes, size_t n_stripes,
                              size_t stripe_stride, size_t block_stride, size_t block_bytes,
                              void *stream, uint64_t *h2d_bytes, uint64_t *d2h_bytes);
rs_status rs_poly_decode_host(const rs_poly_plan *plan, void *host_stripes, size_t n_stripes,
                              size_t stripe_stride, size_t block_stride, size_t block_bytes,
                              const int32_t *erasures, void *stream, uint64_t *h2d_bytes,
                              uint64_t *d2h_bytes);

/* ---- diff-update ----------------------------------------------------------
 * The polynomial realization is linear: if data blocks J = data_idx[0..c-1] change
 * from old to new, then p(new) = p(old) + (x^m * sum_{j in J} (new_j - old_j) x^j mod
 * g), i.e. p_i ^= sum_{j in J} P[i][j] (old_j ^ new_j) with P the parity map (column
 * j = x^{m+j} mod g).  The parity blocks are updated IN PLACE; the other data
 * blocks are not read.  Traffic: (2c + 2m) * block_bytes per stripe.
 *   data_idx   HOST array of c distinct data indices in [0,k) (any order); c = 0 is a
 *              no-op; c > k, an index out of range or a duplicate -> RS_ERR_BAD_ERASURE.
 *   old_data / new_data   HOST arrays of c DEVICE pointers (old_data[i] / new_data[i]
 *              are the old / new contents of data block data_idx[i]);
 *   parity     HOST array of m DEVICE pointers, read and overwritten.
 * Result: bit-identical to rs_poly_encode of the new data (tests pin it to the oracle). */
rs_status rs_poly_update(const rs_poly_plan *plan, const int *data_idx, int n_changed,
                         const void *const *old_data, const void *const *new_data,
                         void *const *parity, size_t block_bytes, void *stream);

/* Compile (NVRTC) and cache the diff-update kernel of the changed set data_idx[0..c-1],
 * blocking until it is ready, so that the first rs_poly_update* call for that set does not
 * run on the table kernel while it compiles.  Host + NVRTC only; no kernel runs. */
rs_status rs_poly_prepare_update(const rs_poly_plan *plan, const int *data_idx, int n_changed);

/* Batched diff-update: `stripes` ([S][n][B] as in rs_poly_encode_batch) holds the NEW
 * data (already in place) and the OLD parity, which is updated in place; the old
 * contents of the changed blocks are in `old_blocks` at old_blocks + s*old_stripe_stride
 * + i*old_block_stride for block data_idx[i] of stripe s.  The same data_idx for every
 * stripe. */
rs_status rs_poly_update_batch(const rs_poly_plan *plan, void *stripes, size_t n_stripes,
                               size_t stripe_stride, size_t block_stride, size_t block_bytes,
                               const int *data_idx, int n_changed, const void *old_blocks,
                               size_t old_stripe_stride, size_t old_block_stride, void *stream);

/* ---- cross-GPU stripe placement ---------------------------------
 * When the blocks of a stripe live on different GPUs (block b of stripe s
 * on rank (b + s) mod N), parity = sum_j P[:,j] d_j (linear) splits by
 * rank: each rank computes the partial parity of the data blocks it holds, and the
 * owner of each parity block adds (XORs) the partials it receives.
 * rs_poly_encode_partial, for stripes s = 0..S-1:
 *   partial[s][i] (^)= sum_q P[i][data_idx[q]] * data[s][q],   i = 0..m-1
 * data: HOST array [S][c] of DEVICE pointers (block data_idx[q] of stripe s), partial:
 * HOST array [S][m] of DEVICE pointers; accumulate != 0 XORs into partial, else
 * overwrites it.  data_idx: c distinct indices in [0,k) (else RS_ERR_BAD_ERASURE); c = 0
 * writes zero partials (accumulate = 0) or is a no-op.
 * rs_poly_xor_reduce: dst[s] = srcs[s][0] ^ ... ^ srcs[s][n_src-1] (HOST arrays of DEVICE
 * pointers, [S] and [S][n_src]; dst may be one of its sources); bytes % (w/8) == 0. */
rs_status rs_poly_encode_partial(const rs_poly_plan *plan, const int *data_idx, int n_data,
                                 const void *const *data, void *const *partial, size_t n_stripes,
                                 size_t block_bytes, int accumulate, void *stream);
rs_status rs_poly_xor_reduce(const rs_poly_plan *plan, void *const *dst, const void *const *srcs, int n_src,
                             size_t n_stripes, size_t bytes, void *stream);

/* ---- the paper's optimisation study (measurement only) ------------
 * Decodes like rs_poly_decode_batch (one erasure list for every stripe) with a
 * per-column, table-driven implementation of the two-step decode as the paper describes
 * HDFS-RAID's code, with its optimisations selected by opt_mask:
 *   bit 0 Opt1 precomputed alpha powers, bit 1 Opt2 skip erased positions in Step 1,
 *   bit 2 Opt3 V_E inverted once (else a Gauss-Jordan elimination per column).
 * opt_mask 0 = "PolyRS" (the HDFS-RAID port), 7 = "OptPolyRS".  Encoding is the same call
 * with the m parity blocks as the erasures.  Same bytes as the product kernels.
 * Limits: w = 8, k + m <= 32, 1 <= n_erasures <= min(m, 8); otherwise RS_ERR_INVALID_ARG. */
rs_status rs_poly_ablation_decode(const rs_poly_plan *plan, void *stripes, size_t n_stripes,
                                  size_t stripe_stride, size_t block_stride, size_t block_bytes,
                                  const int *erasures, int n_erasures, int opt_mask, void *stream);

/* ---- run-time specialised kernels (JIT) ----------------------------------------
 * For every erasure pattern E the decode map survivors -> erased symbols is a fixed
 * GF(2)-linear map (R_E = V_E^{-1} A_E, the paper's Step 1 + Step 2 with Opt1/Opt3
 * precomputed once per pattern).  With JIT on, the plan compiles (NVRTC,
 * sm_100a) a bit-sliced XOR-network kernel for each pattern it meets, exactly like
 * the compiled encoder, and uses it once ready; until then (or if NVRTC is absent)
 * the table-driven kernels serve the pattern.  Results are identical either way.
 * Codes without a compiled encoder network get a JIT encoder the same way.
 *   RS_JIT_OFF        never compile (table-driven kernels only)
 *   RS_JIT_BACKGROUND compile on a worker pool, never block a call (default)
 *   RS_JIT_SYNC       compile inside the first call that meets a pattern
 * rs_poly_plan_set_jit is a configuration call: make it before sharing the plan. */
#define RS_JIT_OFF 0
#define RS_JIT_BACKGROUND 1
#define RS_JIT_SYNC 2
rs_status rs_poly_plan_set_jit(rs_poly_plan *plan, int mode);

/* Decode read policy.  RS_READ_ALL_SURVIVORS (default, the paper's
 * method: Step 1 sums over every non-erased position, Opt2 of P:321) reads the n-t
 * survivors.  RS_READ_K_SURVIVORS reads only k of them (data first) when t < m and
 * solves the m x m system of the t erased plus m-t unread blocks from all m syndromes:
 * identical output (the code is MDS), traffic (k+t)*B instead of (k+m)*B per
 * stripe; the unread survivors may hold anything.  (Under this policy the fallback
 * for a pattern whose JIT kernel is not ready is the generic kernel, not the
 * bit-sliced table kernel, which reads every survivor.)  A configuration call: it drops the plan's
 * decode-pattern cache; make it before sharing the plan. */
#define RS_READ_ALL_SURVIVORS 0
#define RS_READ_K_SURVIVORS 1
rs_status rs_poly_plan_set_read_policy(rs_poly_plan *plan, int policy);

/* Precompute (Opt1/Opt3) the decode constants of every pattern listed in
 * `erasures` (HOST int32 [n_rows][m], -1 padded, as in rs_poly_decode_batch) and,
 * unless JIT is off, compile their kernels, blocking until they are ready.  Also
 * compiles the JIT encoder for codes without a compiled one.  Host + NVRTC only; no
 * kernel runs.  Returns RS_OK even if a compile fails (those patterns keep the
 * table-driven kernels; see rs_poly_plan_stats). */
rs_status rs_poly_prepare(const rs_poly_plan *plan, const int32_t *erasures, size_t n_rows);

/* rs_poly_prepare for EVERY erasure pattern of 1..max_t blocks (sum_t C(n,t) patterns:
 * 1470 for RS(10,4) with max_t = 4, 2516 for RS(12,4)): the paper's "once per pattern"
 * precomputation (Opt1/Opt3) done up front, so that no later decode call
 * ever runs a pattern on the slower table kernels while its JIT kernel compiles.
 * Blocks until every kernel is compiled (or loaded from the on-disk cubin cache).
 * max_t in [0, m] (0 = nothing to do); returns RS_ERR_INVALID_ARG when the count
 * exceeds max_patterns or the plan's JIT module limit (8192); nothing is prepared then. */
rs_status rs_poly_prepare_all(const rs_poly_plan *plan, int max_t, size_t max_patterns);

typedef struct {
  uint64_t patterns;       /* decode patterns in the cache                        */
  uint64_t jit_ready;      /* JIT kernels compiled and loaded                     */
  uint64_t jit_pending;    /* JIT compiles in flight                              */
  uint64_t jit_failed;     /* JIT compiles that failed (NVRTC missing or error)   */
  uint64_t jit_launches;   /* kernel launches that used a JIT kernel              */
  uint64_t table_launches; /* decode body launches that used the table kernels    */
  int jit_available;       /* 1 if NVRTC could be loaded                          */
  int jit_mode;
  uint64_t jit_cache_hits; /* ready JIT kernels loaded from the on-disk cubin cache
                              ($RS_POLY_JIT_CACHE, else ~/.cache/rs_poly_jit; "off"
                              disables it) instead of being compiled               */
} rs_poly_stats;
rs_status rs_poly_plan_stats(const rs_poly_plan *plan, rs_poly_stats *out);

/* Introspection: the CUDA source the JIT generates for erasure list `erasures`
 * (n_erasures >= 1), or for the encoder when n_erasures == 0.  Copies at most cap
 * bytes (NUL-terminated when cap > 0) into buf and returns the full length, or 0 if
 * the arguments are invalid or the pattern is not JIT-eligible.  Host only. */
size_t rs_poly_jit_source(const rs_poly_plan *plan, const int *erasures, int n_erasures, char *buf, size_t cap);

/* Same for the diff-update kernel of the changed-block set data_idx[0..c-1] (c >= 1). */
size_t rs_poly_update_jit_source(const rs_poly_plan *plan, const int *data_idx, int n_changed, char *buf,
                                 size_t cap);

/* ---- misc ----------------------------------------------------------------- */
const char *rs_poly_strerror(rs_status status);
int rs_poly_abi_version(void);

/* Kernels launched by this library since load (all entry points, all threads). */
uint64_t rs_poly_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* RS_POLY_H */
