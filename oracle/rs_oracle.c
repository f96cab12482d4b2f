/*
 * rs_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the polynomial
 * Reed-Solomon hot path computes, written from the paper
 *   Sheykh Esmaili & Datta, "On the Effectiveness of Polynomial Realization of
 *   Reed-Solomon Codes for Storage Systems" (arXiv 1312.5155) = PAPER.md.
 * Citations "P:n" are PAPER.md line numbers.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code, header, table or
 * constant generator with the CUDA library under paper_1312_5155_b200/csrc.
 *
 * Conventions:
 *   - API block index b in [0,n): 0..k-1 data, k..n-1 parity.
 *   - polynomial position pos(b) = m+b for data (Eq. 2: data d_i sits at
 *     x^{m+i}, pinned by the P:204 example 48x^3+6x^4+112x^5+70x^6),
 *     pos(b) = b-k for parity (parity p_i is the coefficient of x^i).
 *   - alpha = 2, GF(2^w) reduced by prim_poly (0x11D is forced by the
 *     P:278 matrix entry alpha^8 = 29; reading G1).
 *   - w=16 symbols are little-endian uint16 (reading G10).
 *
 * Every function here is scalar; the bulk functions add only (a) their own
 * log/exp tables, checked exhaustively against orc_gf_mul by the tests,
 * (b) V^{-1} once per erasure pattern -- the paper's Opt3 -- and
 * (c) threads over stripes.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXN 256
#define ORC_MAXM 64

/* ------------------------------------------------------------------------- */
/* GF(2^w) element arithmetic (add is XOR in characteristic 2).      */
/* ------------------------------------------------------------------------- */

int orc_field_ok(int w, uint32_t poly) {
  return (w == 8 || w == 16) && (poly >> w) == 1u;
}

/* Shift-and-add carry-less multiply, reducing by poly whenever bit w is set.
 * No tables.  a, b < 2^w. */
uint32_t orc_gf_mul(uint32_t a, uint32_t b, int w, uint32_t poly) {
  uint32_t r = 0;
  while (b) {
    if (b & 1u) r ^= a;
    b >>= 1;
    a <<= 1;
    if (a >> w) a ^= poly;
  }
  return r;
}

/* a^e by square-and-multiply over orc_gf_mul. */
uint32_t orc_gf_pow(uint32_t a, uint64_t e, int w, uint32_t poly) {
  uint32_t r = 1;
  while (e) {
    if (e & 1u) r = orc_gf_mul(r, a, w, poly);
    a = orc_gf_mul(a, a, w, poly);
    e >>= 1;
  }
  return r;
}

/* a^{-1} = a^(2^w - 2) (Fermat).  Returns 0 for a == 0 ("zero divisor"). */
uint32_t orc_gf_inv(uint32_t a, int w, uint32_t poly) {
  if (a == 0) return 0;
  return orc_gf_pow(a, ((uint64_t)1 << w) - 2, w, poly);
}

/* Multiplicative order of alpha = 2: the field is usable only if
 * this is 2^w - 1 (prim_poly primitive). */
uint32_t orc_order_of_alpha(int w, uint32_t poly) {
  uint32_t x = 2, ord = 1;
  uint32_t lim = (1u << w);
  while (x != 1 && ord < lim) {
    x = orc_gf_mul(x, 2, w, poly);
    ++ord;
  }
  return x == 1 ? ord : 0;
}

/* ------------------------------------------------------------------------- */
/* Generator polynomial:                                          */
/*   g(x) = sum_{i=0}^{m} g_i x^i = (x + alpha^0)(x + alpha^1)...(x + alpha^{m-1}) */
/* g[0..m] low -> high, monic.                                                */
/* ------------------------------------------------------------------------- */
int orc_gen_poly(int m, int w, uint32_t poly, uint32_t *g) {
  if (!orc_field_ok(w, poly) || m < 1 || m > ORC_MAXM) return -1;
  uint32_t cur[ORC_MAXM + 1] = {0}, nxt[ORC_MAXM + 1];
  cur[0] = 1; /* g = 1 */
  for (int i = 0; i < m; ++i) {
    uint32_t root = orc_gf_pow(2, (uint64_t)i, w, poly); /* alpha^i */
    /* multiply by (x + alpha^i): nxt[l] = cur[l-1] + alpha^i * cur[l] */
    for (int l = 0; l <= i + 1; ++l) {
      uint32_t hi = l > 0 ? cur[l - 1] : 0;
      uint32_t lo = l <= i ? orc_gf_mul(root, cur[l], w, poly) : 0;
      nxt[l] = hi ^ lo;
    }
    memcpy(cur, nxt, sizeof(uint32_t) * (size_t)(i + 2));
  }
  memcpy(g, cur, sizeof(uint32_t) * (size_t)(m + 1));
  return 0;
}

static int pos_of(int b, int k, int m) { return b < k ? m + b : b - k; }

/* ------------------------------------------------------------------------- */
/* Encode one column (Eq. 1-2): the remainder of d(x) x^m by g(x),  */
/* by literal polynomial long division.                                       */
/*   d[0..k-1]: data symbols (d_j is the coefficient of x^{m+j});             */
/*   p[0..m-1]: parity out (p_i is the coefficient of x^i).                   */
/* ------------------------------------------------------------------------- */
int orc_encode_column(int k, int m, int w, uint32_t poly, const uint32_t *d, uint32_t *p) {
  if (!orc_field_ok(w, poly) || k < 1 || m < 1 || k + m > ORC_MAXN || m > ORC_MAXM) return -1;
  int n = k + m;
  uint32_t g[ORC_MAXM + 1], c[ORC_MAXN];
  orc_gen_poly(m, w, poly, g);
  for (int i = 0; i < m; ++i) c[i] = 0;     /* d(x) * x^m */
  for (int j = 0; j < k; ++j) c[m + j] = d[j];
  for (int i = n - 1; i >= m; --i) {         /* divide by g (monic) */
    uint32_t q = c[i];
    if (q == 0) continue;
    for (int l = 0; l <= m; ++l) c[i - m + l] ^= orc_gf_mul(q, g[l], w, poly);
  }
  for (int i = 0; i < m; ++i) p[i] = c[i];   /* remainder = parity */
  return 0;
}

/* Evaluate the codeword polynomial c(x) = sum_b c_b x^{pos(b)} at x = a
 * (Horner over positions n-1..0).  cw is in API order.  Used for the root
 * property c(alpha^j) = 0, j < m. */
uint32_t orc_eval_codeword(int k, int m, int w, uint32_t poly, const uint32_t *cw, uint32_t a) {
  int n = k + m;
  uint32_t byp[ORC_MAXN];
  for (int b = 0; b < n; ++b) byp[pos_of(b, k, m)] = cw[b];
  uint32_t acc = 0;
  for (int p = n - 1; p >= 0; --p) acc = orc_gf_mul(acc, a, w, poly) ^ byp[p];
  return acc;
}

/* Solve A y = s over GF(2^w) by Gauss-Jordan with the first nonzero pivot.
 * A is t x t row-major, destroyed.  Returns 0, or -1 if singular. */
static int gauss_jordan(int t, uint32_t *A, uint32_t *s, uint32_t *y, int w, uint32_t poly) {
  for (int col = 0; col < t; ++col) {
    int piv = -1;
    for (int r = col; r < t; ++r)
      if (A[r * t + col]) { piv = r; break; }
    if (piv < 0) return -1;
    if (piv != col) {
      for (int c = 0; c < t; ++c) { uint32_t tmp = A[col * t + c]; A[col * t + c] = A[piv * t + c]; A[piv * t + c] = tmp; }
      uint32_t tmp = s[col]; s[col] = s[piv]; s[piv] = tmp;
    }
    uint32_t inv = orc_gf_inv(A[col * t + col], w, poly);
    for (int c = 0; c < t; ++c) A[col * t + c] = orc_gf_mul(A[col * t + c], inv, w, poly);
    s[col] = orc_gf_mul(s[col], inv, w, poly);
    for (int r = 0; r < t; ++r) {
      if (r == col) continue;
      uint32_t f = A[r * t + col];
      if (!f) continue;
      for (int c = 0; c < t; ++c) A[r * t + c] ^= orc_gf_mul(f, A[col * t + c], w, poly);
      s[r] ^= orc_gf_mul(f, s[col], w, poly);
    }
  }
  for (int i = 0; i < t; ++i) y[i] = s[i];
  return 0;
}

static int check_erasures(int n, int m, const int *er, int t) {
  if (t < 0 || t > m) return -2;
  for (int i = 0; i < t; ++i) {
    if (er[i] < 0 || er[i] >= n) return -3;
    for (int j = 0; j < i; ++j)
      if (er[j] == er[i]) return -3;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Decode one column.                                             */
/*   cw[0..n-1]: codeword in API order; erased entries are don't-care.        */
/*   er[0..t-1]: erased API indices (any order), t <= m.                      */
/* Step 1: D(alpha^j) over the survivors, j = 0..t-1 -- erased    */
/*   entries are zeroed so they contribute nothing (Opt2, skips them). */
/* Step 2: the t x t Vandermonde system                           */
/*   D(alpha^j) = sum_e y_e (alpha^{pos_e})^j, solved by Gauss-Jordan.        */
/* Erased parity positions are unknowns in the same system (reading G6).     */
/* syn_out (optional, t entries) receives the Step-1 values D(alpha^j).       */
/* ------------------------------------------------------------------------- */
int orc_decode_column(int k, int m, int w, uint32_t poly, uint32_t *cw, const int *er, int t,
                      uint32_t *syn_out) {
  int n = k + m;
  if (!orc_field_ok(w, poly) || k < 1 || m < 1 || n > ORC_MAXN || m > ORC_MAXM) return -1;
  int rc = check_erasures(n, m, er, t);
  if (rc) return rc;
  if (t == 0) return 0;
  uint32_t c[ORC_MAXN];
  memcpy(c, cw, sizeof(uint32_t) * (size_t)n);
  for (int i = 0; i < t; ++i) c[er[i]] = 0;
  /* Step 1 */
  uint32_t S[ORC_MAXM], V[ORC_MAXM * ORC_MAXM], y[ORC_MAXM];
  for (int j = 0; j < t; ++j) {
    uint32_t aj = orc_gf_pow(2, (uint64_t)j, w, poly);
    S[j] = orc_eval_codeword(k, m, w, poly, c, aj);
  }
  if (syn_out)
    for (int j = 0; j < t; ++j) syn_out[j] = S[j];
  /* Step 2 */
  for (int j = 0; j < t; ++j)
    for (int e = 0; e < t; ++e) {
      uint32_t X = orc_gf_pow(2, (uint64_t)pos_of(er[e], k, m), w, poly); /* alpha^{pos_e} */
      V[j * t + e] = orc_gf_pow(X, (uint64_t)j, w, poly);
    }
  if (gauss_jordan(t, V, S, y, w, poly)) return -4;
  for (int e = 0; e < t; ++e) cw[er[e]] = y[e];
  return 0;
}

/* The t x t Vandermonde matrix of Step 2, for inspection by the
 * pins (P:276-278 prints it for the worked example). */
int orc_decode_matrix(int k, int m, int w, uint32_t poly, const int *er, int t, uint32_t *V) {
  int n = k + m;
  int rc = check_erasures(n, m, er, t);
  if (rc) return rc;
  for (int j = 0; j < t; ++j)
    for (int e = 0; e < t; ++e) {
      uint32_t X = orc_gf_pow(2, (uint64_t)pos_of(er[e], k, m), w, poly);
      V[j * t + e] = orc_gf_pow(X, (uint64_t)j, w, poly);
    }
  return 0;
}

/* Independent cross-check of Step 2: Forney's formula with first consecutive
 * root alpha^0 (textbook erasure decoding; not in the paper).
 *   S_j = c'(alpha^j), Lambda(x) = prod_e (1 + X_e x), X_e = alpha^{pos_e},
 *   Omega(x) = S(x) Lambda(x) mod x^t,  Y_e = X_e Omega(X_e^-1) / Lambda'(X_e^-1). */
int orc_decode_column_forney(int k, int m, int w, uint32_t poly, uint32_t *cw, const int *er, int t) {
  int n = k + m;
  if (!orc_field_ok(w, poly) || k < 1 || m < 1 || n > ORC_MAXN || m > ORC_MAXM) return -1;
  int rc = check_erasures(n, m, er, t);
  if (rc) return rc;
  if (t == 0) return 0;
  uint32_t c[ORC_MAXN], S[ORC_MAXM], L[ORC_MAXM + 1] = {0}, O[ORC_MAXM] = {0}, X[ORC_MAXM];
  memcpy(c, cw, sizeof(uint32_t) * (size_t)n);
  for (int i = 0; i < t; ++i) c[er[i]] = 0;
  for (int j = 0; j < t; ++j) S[j] = orc_eval_codeword(k, m, w, poly, c, orc_gf_pow(2, (uint64_t)j, w, poly));
  L[0] = 1;
  for (int e = 0; e < t; ++e) {
    X[e] = orc_gf_pow(2, (uint64_t)pos_of(er[e], k, m), w, poly);
    for (int l = e + 1; l >= 1; --l) L[l] ^= orc_gf_mul(L[l - 1], X[e], w, poly);
  }
  for (int i = 0; i < t; ++i)
    for (int j = 0; j <= i; ++j) O[i] ^= orc_gf_mul(S[j], L[i - j], w, poly);
  for (int e = 0; e < t; ++e) {
    uint32_t xi = orc_gf_inv(X[e], w, poly), num = 0, den = 0, pw = 1;
    for (int i = 0; i < t; ++i) { num ^= orc_gf_mul(O[i], pw, w, poly); pw = orc_gf_mul(pw, xi, w, poly); }
    /* formal derivative in characteristic 2: only odd-degree terms survive */
    pw = 1;
    for (int l = 1; l <= t; ++l) {
      if (l & 1) den ^= orc_gf_mul(L[l], pw, w, poly);
      pw = orc_gf_mul(pw, xi, w, poly);
    }
    if (den == 0) return -4;
    cw[er[e]] = orc_gf_mul(orc_gf_mul(X[e], num, w, poly), orc_gf_inv(den, w, poly), w, poly);
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Bulk mode: the same steps over whole stripes.               */
/* Layout: stripe s, block b at base + s*stripe_stride + b*block_stride;      */
/* block_bytes bytes per block; w=16 symbols little-endian.                   */
/* ------------------------------------------------------------------------- */
typedef struct {
  int w;
  uint32_t poly, q; /* q = 2^w - 1 */
  uint32_t *lg;     /* log table, 2^w entries (lg[0] unused) */
  uint32_t *ex;     /* exp table, 2q entries */
} orc_tables;

static int tables_make(orc_tables *T, int w, uint32_t poly) {
  T->w = w; T->poly = poly; T->q = (1u << w) - 1;
  T->lg = (uint32_t *)calloc((size_t)1 << w, sizeof(uint32_t));
  T->ex = (uint32_t *)calloc((size_t)2 * T->q, sizeof(uint32_t));
  if (!T->lg || !T->ex) return -1;
  uint32_t x = 1;
  for (uint32_t i = 0; i < T->q; ++i) {
    T->ex[i] = x; T->ex[i + T->q] = x; T->lg[x] = i;
    x = orc_gf_mul(x, 2, w, poly);
  }
  return 0;
}
static void tables_free(orc_tables *T) { free(T->lg); free(T->ex); }
static inline uint32_t tmul(const orc_tables *T, uint32_t a, uint32_t b) {
  return (a && b) ? T->ex[T->lg[a] + T->lg[b]] : 0;
}

/* Exposed so the tests can check the bulk tables against orc_gf_mul on every pair. */
int orc_bulk_table_mul(int w, uint32_t poly, const uint32_t *a, const uint32_t *b, uint32_t *out, size_t cnt) {
  if (!orc_field_ok(w, poly)) return -1;
  orc_tables T;
  if (tables_make(&T, w, poly)) return -1;
  for (size_t i = 0; i < cnt; ++i) out[i] = tmul(&T, a[i], b[i]);
  tables_free(&T);
  return 0;
}

static inline uint32_t sym_get(const uint8_t *p, size_t c, int w) {
  return w == 8 ? p[c] : (uint32_t)p[2 * c] | ((uint32_t)p[2 * c + 1] << 8);
}
static inline void sym_put(uint8_t *p, size_t c, int w, uint32_t v) {
  if (w == 8) p[c] = (uint8_t)v;
  else { p[2 * c] = (uint8_t)(v & 0xFF); p[2 * c + 1] = (uint8_t)(v >> 8); }
}

typedef struct {
  int k, m, w, op; /* op 0 = encode, 1 = decode */
  uint32_t poly;
  uint8_t *base;
  size_t stripe_stride, block_stride, block_bytes;
  const int32_t *erasures; /* [S][m], -1 padded */
  size_t s0, s1;           /* stripe range */
  const orc_tables *T;
  const uint32_t *g;
  int rc;
} bulk_job;

static void encode_stripe(bulk_job *J, size_t s) {
  const orc_tables *T = J->T;
  int k = J->k, m = J->m, n = k + m, w = J->w;
  size_t ncol = J->block_bytes / (size_t)(w / 8);
  uint8_t *st = J->base + s * J->stripe_stride;
  uint32_t c[ORC_MAXN];
  for (size_t col = 0; col < ncol; ++col) {
    /* literal long division of d(x) x^m by g(x) */
    for (int i = 0; i < m; ++i) c[i] = 0;
    for (int j = 0; j < k; ++j) c[m + j] = sym_get(st + (size_t)j * J->block_stride, col, w);
    for (int i = n - 1; i >= m; --i) {
      uint32_t q = c[i];
      if (!q) continue;
      for (int l = 0; l <= m; ++l) c[i - m + l] ^= tmul(T, q, J->g[l]);
    }
    for (int i = 0; i < m; ++i) sym_put(st + (size_t)(k + i) * J->block_stride, col, w, c[i]);
  }
}

static void decode_stripe(bulk_job *J, size_t s) {
  const orc_tables *T = J->T;
  int k = J->k, m = J->m, n = k + m, w = J->w;
  const int32_t *row = J->erasures + s * (size_t)m;
  int er[ORC_MAXM] = {0}, t = 0;
  for (int i = 0; i < m; ++i)
    if (row[i] >= 0) er[t++] = row[i];
  if (check_erasures(n, m, er, t)) { J->rc = -3; return; }
  if (t == 0) return;
  /* Opt1: the alpha-power coefficients alpha^{j*pos} are common to all
   * columns; Opt3: V is inverted once per erasure pattern. */
  uint32_t V[ORC_MAXM * ORC_MAXM], Vi[ORC_MAXM * ORC_MAXM];
  for (int j = 0; j < t; ++j)
    for (int e = 0; e < t; ++e)
      V[j * t + e] = orc_gf_pow(orc_gf_pow(2, (uint64_t)pos_of(er[e], k, m), w, J->poly), (uint64_t)j, w, J->poly);
  for (int col = 0; col < t; ++col) { /* V^-1 column by column via Gauss-Jordan */
    uint32_t A[ORC_MAXM * ORC_MAXM], e[ORC_MAXM] = {0}, y[ORC_MAXM];
    memcpy(A, V, sizeof(uint32_t) * (size_t)(t * t));
    e[col] = 1;
    if (gauss_jordan(t, A, e, y, w, J->poly)) { J->rc = -4; return; }
    for (int r = 0; r < t; ++r) Vi[r * t + col] = y[r];
  }
  int erased[ORC_MAXN] = {0};
  for (int i = 0; i < t; ++i) erased[er[i]] = 1;
  int surv[ORC_MAXN], ns = 0;
  for (int b = 0; b < n; ++b)
    if (!erased[b]) surv[ns++] = b;
  uint32_t coef[ORC_MAXM][ORC_MAXN]; /* coef[j][i] = (alpha^j)^{pos(surv_i)} */
  for (int j = 0; j < t; ++j)
    for (int i = 0; i < ns; ++i)
      coef[j][i] = orc_gf_pow(orc_gf_pow(2, (uint64_t)j, w, J->poly), (uint64_t)pos_of(surv[i], k, m), w, J->poly);
  uint8_t *st = J->base + s * J->stripe_stride;
  size_t ncol = J->block_bytes / (size_t)(w / 8);
  for (size_t col = 0; col < ncol; ++col) {
    uint32_t S[ORC_MAXM] = {0};
    for (int i = 0; i < ns; ++i) { /* Step 1 over survivors only (Opt2) */
      uint32_t v = sym_get(st + (size_t)surv[i] * J->block_stride, col, w);
      if (!v) continue;
      for (int j = 0; j < t; ++j) S[j] ^= tmul(T, v, coef[j][i]);
    }
    for (int e = 0; e < t; ++e) { /* Step 2: y = V^-1 S */
      uint32_t y = 0;
      for (int j = 0; j < t; ++j) y ^= tmul(T, Vi[e * t + j], S[j]);
      sym_put(st + (size_t)er[e] * J->block_stride, col, w, y);
    }
  }
}

static void *bulk_worker(void *arg) {
  bulk_job *J = (bulk_job *)arg;
  for (size_t s = J->s0; s < J->s1; ++s) {
    if (J->op == 0) encode_stripe(J, s);
    else decode_stripe(J, s);
  }
  return NULL;
}

static int bulk_run(int op, int k, int m, int w, uint32_t poly, uint8_t *base, size_t n_stripes,
                    size_t stripe_stride, size_t block_stride, size_t block_bytes,
                    const int32_t *erasures, int nthreads) {
  if (!orc_field_ok(w, poly) || k < 1 || m < 1 || k + m > ORC_MAXN || m > ORC_MAXM) return -1;
  if (block_bytes % (size_t)(w / 8)) return -1;
  if (orc_order_of_alpha(w, poly) != (1u << w) - 1 || (uint32_t)(k + m) > (1u << w) - 1) return -1;
  if (nthreads < 1) nthreads = 1;
  if ((size_t)nthreads > n_stripes) nthreads = (int)(n_stripes ? n_stripes : 1);
  orc_tables T;
  uint32_t g[ORC_MAXM + 1];
  if (tables_make(&T, w, poly)) return -1;
  orc_gen_poly(m, w, poly, g);
  bulk_job *jobs = (bulk_job *)calloc((size_t)nthreads, sizeof(bulk_job));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int i = 0; i < nthreads; ++i) {
    bulk_job *J = &jobs[i];
    J->k = k; J->m = m; J->w = w; J->op = op; J->poly = poly; J->base = base;
    J->stripe_stride = stripe_stride; J->block_stride = block_stride; J->block_bytes = block_bytes;
    J->erasures = erasures; J->T = &T; J->g = g; J->rc = 0;
    J->s0 = n_stripes * (size_t)i / (size_t)nthreads;
    J->s1 = n_stripes * (size_t)(i + 1) / (size_t)nthreads;
    if (nthreads == 1) bulk_worker(J);
    else pthread_create(&th[i], NULL, bulk_worker, J);
  }
  int rc = 0;
  for (int i = 0; i < nthreads; ++i) {
    if (nthreads > 1) pthread_join(th[i], NULL);
    if (jobs[i].rc) rc = jobs[i].rc;
  }
  free(jobs); free(th); tables_free(&T);
  return rc;
}

int orc_encode_bulk(int k, int m, int w, uint32_t poly, uint8_t *base, size_t n_stripes,
                    size_t stripe_stride, size_t block_stride, size_t block_bytes, int nthreads) {
  return bulk_run(0, k, m, w, poly, base, n_stripes, stripe_stride, block_stride, block_bytes, NULL, nthreads);
}

int orc_decode_bulk(int k, int m, int w, uint32_t poly, uint8_t *base, size_t n_stripes,
                    size_t stripe_stride, size_t block_stride, size_t block_bytes,
                    const int32_t *erasures, int nthreads) {
  return bulk_run(1, k, m, w, poly, base, n_stripes, stripe_stride, block_stride, block_bytes, erasures, nthreads);
}
