#!/usr/bin/env python3
"""Build-time generator of the bit-sliced encode networks (product side).

For each supported instance (k, m, w, prim_poly) it

1. builds GF(2^w) with alpha = 2 and g(x) = prod_{i<m}(x + alpha^i)
   (P:170-177);
2. forms the parity map P (m x k; column j = x^{m+j} mod g -- the generator-matrix
   form of g), so that p_i = sum_j P[i][j] d_j is exactly the remainder of
   Eq. 1-2;
3. expands P into its GF(2) bit-matrix (m*w rows x k*w columns): output bit o of
   parity i is the XOR of input bits b of data j where bit o of P[i][j]*alpha^b is 1;
4. shrinks the XOR count by greedy common-subexpression elimination (repeatedly
   factor out the input pair shared by the most rows -- Paar's heuristic);
5. emits a straight-line CUDA function over 32-column bit-planes.

This is the paper's own "bit-matrix" future-work direction applied to the
polynomial realization.  The emitted code is checked bit-exactly against the CPU
oracle by tests/test_gpu_parity.py; tests/test_plan_host.py checks this script's
parity map against the C++ builder and the oracle.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

# (k, m, w, prim_poly) instances compiled into librs_poly.so.  Others use the generic
# split-nibble kernel.  Fused bit-sliced decode packs t <= m <= 4 outputs per word.
INSTANCES = [
    # (k, m, w, prim_poly, data blocks per CSE group)
    (10, 4, 8, 0x11D, 10),   # paper's RS(10,4); configs C1, C3, C5
    (6, 3, 8, 0x11D, 6),     # config C2
    (4, 3, 8, 0x11D, 4),     # the paper's worked example RS(4,3)
    (10, 2, 8, 0x11D, 10),   # P:440 (10,2)
    (10, 3, 8, 0x11D, 10),
    (12, 4, 8, 0x11D, 12),
    (8, 4, 8, 0x11D, 8),
    (6, 4, 8, 0x11D, 6),
    (12, 4, 16, 0x1100B, 0),  # config C4: syndrome-form (Horner + Q) encoder, see emit_horner
]
# w = 16 instances use the syndrome form of the encoder (P:237-241 with the symmetric use of
# P:306): H_j = Horner over the data planes with step alpha^j (sparse, compile-time in
# bitslice_device.cuh), then parity = Q H with Q = Vp^{-1} diag(alpha^{jm}) emitted here.
# A direct 64 x 192 parity-map network needs ~2400 XORs in register-sized CSE groups;
# Horner (~715 LOP3) + Q (~620 XORs) streams one block at a time.
HORNER_W = (16,)

# CSE: cse3 factors pairs and triples by estimated 3-input-gate (LOP3) savings; paar (the
# classic pair-only greedy, fewest 2-input XORs) compiled to 727 vs 630 LOP3 per RS(10,4)
# unit and ran 2-6% slower (round 1), so it is kept for reference only.

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "rs_networks.cuh")


def gf_mul(a: int, b: int, w: int, poly: int) -> int:
    r = 0
    while b:
        if b & 1:
            r ^= a
        b >>= 1
        a <<= 1
        if a >> w:
            a ^= poly
    return r


def generator(m: int, w: int, poly: int) -> list[int]:
    g = [1]
    root = 1
    for _ in range(m):
        ng = [0] * (len(g) + 1)
        for l in range(len(ng)):
            hi = g[l - 1] if l > 0 else 0
            lo = gf_mul(root, g[l], w, poly) if l < len(g) else 0
            ng[l] = hi ^ lo
        g = ng
        root = gf_mul(root, 2, w, poly)
    return g


def parity_map(k: int, m: int, w: int, poly: int) -> list[list[int]]:
    g = generator(m, w, poly)
    col = g[:m]
    P = [[0] * k for _ in range(m)]
    for j in range(k):
        for i in range(m):
            P[i][j] = col[i]
        top = col[m - 1]
        col = [(col[i - 1] if i else 0) ^ gf_mul(top, g[i], w, poly) for i in range(m)]
    return P


def bit_matrix(k: int, m: int, w: int, poly: int) -> np.ndarray:
    P = parity_map(k, m, w, poly)
    R = np.zeros((m * w, k * w), dtype=bool)
    for i in range(m):
        for j in range(k):
            for b in range(w):
                prod = gf_mul(P[i][j], 1 << b, w, poly)
                for o in range(w):
                    if (prod >> o) & 1:
                        R[i * w + o, j * w + b] = True
    return R


def paar(R: np.ndarray):
    """Greedy CSE.  Returns (temps, rows): temps[t] = (u, v) meaning var (nin+t) = u ^ v;
    rows[r] = sorted list of vars whose XOR is output r."""
    nrow, nin = R.shape
    cap = nin + int(R.sum())
    M = np.zeros((nrow, cap), dtype=np.float32)
    M[:, :nin] = R
    nv = nin
    temps = []
    while True:
        A = M[:, :nv]
        C = A.T @ A
        np.fill_diagonal(C, 0)
        C = np.triu(C)
        idx = int(np.argmax(C))
        a, b = divmod(idx, nv)
        if C[a, b] < 2:
            break
        rows = (M[:, a] > 0) & (M[:, b] > 0)
        M[rows, a] = 0
        M[rows, b] = 0
        M[rows, nv] = 1
        temps.append((a, b))
        nv += 1
    rows = [sorted(np.nonzero(M[r, :nv])[0].tolist()) for r in range(nrow)]
    return temps, rows


def cse3(R: np.ndarray):
    """Greedy CSE for 3-input XOR gates (one LOP3 each).  A row of r terms costs about
    (r - 1) / 2 gates, so factoring a set of s variables shared by c rows saves about
    (s - 1) c / 2 - 1 gates; repeatedly factor the pair or triple with the largest saving.
    Returns (temps, rows): temps[t] = tuple of 2 or 3 vars XORed into var (nin + t);
    rows[r] = sorted vars whose XOR is output r.  Rows <= 64 (column masks are uint64)."""
    nrow, nin = R.shape
    assert nrow <= 64
    cols = [int(sum(1 << r for r in range(nrow) if R[r, c])) for c in range(nin)]
    temps = []
    while True:
        arr = np.array(cols, dtype=np.uint64)
        pc = np.bitwise_count(arr)
        best, pick = 0.0, None
        nv = len(cols)
        for a in range(nv):
            if pc[a] < 2:
                continue
            ab = arr[a] & arr[a + 1:]
            cab = np.bitwise_count(ab)
            for off in np.nonzero(cab >= 2)[0]:
                b = a + 1 + int(off)
                c2 = int(cab[off])
                if c2 / 2 - 1 > best:
                    best, pick = c2 / 2 - 1, (a, b)
                if b + 1 < nv and c2 - 1 > best:  # else no triple within (a, b) can beat it
                    c3 = np.bitwise_count(ab[off] & arr[b + 1:])
                    j = int(np.argmax(c3))
                    if c3[j] >= 2 and c3[j] - 1 > best:
                        best, pick = float(c3[j] - 1), (a, b, b + 1 + j)
        if pick is None:
            break
        common = cols[pick[0]]
        for v in pick[1:]:
            common &= cols[v]
        for v in pick:
            cols[v] &= ~common
        cols.append(common)
        temps.append(pick)
    rows = [sorted(v for v in range(len(cols)) if (cols[v] >> r) & 1) for r in range(nrow)]
    return temps, rows


def CSE(R: np.ndarray):
    return cse3(R)


def gf_pow(a: int, e: int, w: int, poly: int) -> int:
    r = 1
    for _ in range(e):
        r = gf_mul(r, a, w, poly)
    return r


def gf_inv_matrix(A: list[list[int]], w: int, poly: int) -> list[list[int]]:
    t = len(A)
    M = [list(row) + [1 if r == c else 0 for c in range(t)] for r, row in enumerate(A)]
    for c in range(t):
        p = next(r for r in range(c, t) if M[r][c])
        M[c], M[p] = M[p], M[c]
        iv = gf_pow(M[c][c], (1 << w) - 2, w, poly)
        M[c] = [gf_mul(iv, v, w, poly) for v in M[c]]
        for r in range(t):
            if r != c and M[r][c]:
                f = M[r][c]
                M[r] = [v ^ gf_mul(f, u, w, poly) for v, u in zip(M[r], M[c])]
    return [row[t:] for row in M]


def horner_q(k: int, m: int, w: int, poly: int) -> list[list[int]]:
    """Q (m x m): parity p = Q H, H_j = sum_b d_b alpha^{j b} (Horner over the data).

    Every codeword has zero syndromes at alpha^0..alpha^{m-1} (roots of g), so
    sum_i p_i alpha^{j i} = S_j(data) = alpha^{j m} H_j (char 2); p = Vp^{-1} diag(alpha^{jm}) H."""
    a = 2
    Vp = [[gf_pow(gf_pow(a, i, w, poly), j, w, poly) for i in range(m)] for j in range(m)]
    Vi = gf_inv_matrix(Vp, w, poly)
    return [[gf_mul(Vi[i][j], gf_pow(a, j * m, w, poly), w, poly) for j in range(m)] for i in range(m)]


def gf_bit_matrix(M: list[list[int]], w: int, poly: int) -> np.ndarray:
    rows, cols = len(M), len(M[0])
    R = np.zeros((rows * w, cols * w), dtype=bool)
    for i in range(rows):
        for j in range(cols):
            for b in range(w):
                prod = gf_mul(M[i][j], 1 << b, w, poly)
                for o in range(w):
                    if (prod >> o) & 1:
                        R[i * w + o, j * w + b] = True
    return R


def emit_horner(k: int, m: int, w: int, poly: int) -> str:
    R = gf_bit_matrix(horner_q(k, m, w, poly), w, poly)
    temps, rows = CSE(R)
    nin = m * w

    def name(v: int) -> str:
        return f"h[{v}]" if v < nin else f"t{v - nin}"

    xors = sum(len(t) - 1 for t in temps) + sum(max(0, len(r) - 1) for r in rows)
    out = [
        f"// RS({k},{m}) over GF(2^{w}) / 0x{poly:X}: syndrome-form encoder.  Q = Vp^-1 diag(alpha^jm),",
        f"// bit-matrix {m * w}x{m * w} with {int(R.sum())} ones -> {xors} two-input XORs after CSE.",
        f"template <> struct RsQNet<{k}, {m}, {w}, 0x{poly:X}u> {{",
        f"  static constexpr bool kHorner = true;",
        f"  static constexpr int kXors = {xors};",
        f"  static __device__ __forceinline__ void run(const uint32_t (&h)[{nin}], uint32_t (&y)[{m * w}]) {{",
    ]
    for t, ops in enumerate(temps):
        out.append(f"    const uint32_t t{t} = " + " ^ ".join(name(v) for v in ops) + ";")
    for r, terms in enumerate(rows):
        expr = " ^ ".join(name(v) for v in terms) if terms else "0u"
        out.append(f"    y[{r}] = {expr};")
    out += ["  }", "};", ""]
    return "\n".join(out)


def emit_instance(k: int, m: int, w: int, poly: int, gsize: int) -> str:
    if w in HORNER_W:
        return emit_horner(k, m, w, poly)
    R = bit_matrix(k, m, w, poly)
    ngroups = (k + gsize - 1) // gsize
    total_xors = 0
    body = []
    for g in range(ngroups):
        j0, j1 = g * gsize, min(k, (g + 1) * gsize)
        sub = R[:, j0 * w: j1 * w]
        nin = (j1 - j0) * w
        temps, rows = CSE(sub)

        def name(v: int) -> str:
            return f"x[{v}]" if v < nin else f"t{v - nin}"

        xors = sum(len(t) - 1 for t in temps) + sum(max(0, len(r) - 1) for r in rows) + \
            (0 if g == 0 else sum(1 for r in rows if r))
        total_xors += xors
        body += [
            f"// group {g}: data blocks {j0}..{j1 - 1}, {int(sub.sum())} ones, {len(temps)} temps, {xors} XORs",
            f"template <> struct RsNetGroup<{k}, {m}, {w}, 0x{poly:X}u, {g}> {{",
            f"  static constexpr int kFirstBlock = {j0}, kBlocks = {j1 - j0};",
            f"  static __device__ __forceinline__ void run(const uint32_t (&x)[{nin}], uint32_t (&y)[{m * w}]) {{",
        ]
        for t, ops in enumerate(temps):
            body.append(f"    const uint32_t t{t} = " + " ^ ".join(name(v) for v in ops) + ";")
        for r, terms in enumerate(rows):
            expr = " ^ ".join(name(v) for v in terms) if terms else "0u"
            body.append(f"    y[{r}] = {expr};" if g == 0 else (f"    y[{r}] ^= {expr};" if terms else ""))
        body += ["  }", "};", ""]
    head = [
        f"// RS({k},{m}) over GF(2^{w}) / 0x{poly:X}: bit-matrix {m * w}x{k * w} with {int(R.sum())} ones;",
        f"// {ngroups} CSE group(s) of <= {gsize} data blocks; {total_xors} two-input XORs per 32 columns.",
        f"template <> struct RsNet<{k}, {m}, {w}, 0x{poly:X}u> {{",
        f"  static constexpr int kGroups = {ngroups}, kGroupBlocks = {gsize}, kXors = {total_xors};",
        "};",
    ]
    return "\n".join(head + body)


def source_digest() -> str:
    with open(os.path.abspath(__file__), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def generate(out: str = OUT, force: bool = False) -> bool:
    digest = source_digest()
    if not force and os.path.exists(out):
        with open(out) as f:
            if f"generator-digest: {digest}" in f.read(4096):
                return False
    parts = [
        "// GENERATED by gen_networks.py -- do not edit.",
        f"// generator-digest: {digest}",
        "// Straight-line GF(2) networks computing the parity planes y (m*w planes of 32",
        "// columns) from the data planes x (k*w planes): y[i*w+o] = bit o of parity i.",
        "#pragma once",
        "#include <cstdint>",
        "",
        "template <int K, int M, int W, uint32_t POLY> struct RsNet;  // only the instances below exist",
        "template <int K, int M, int W, uint32_t POLY, int G> struct RsNetGroup;",
        "// syndrome-form encoders (w = 16): kHorner = true and run() = the Q network",
        "template <int K, int M, int W, uint32_t POLY> struct RsQNet { static constexpr bool kHorner = false; };",
        "",
        "#define RS_NET_INSTANCES(X) \\",
    ]
    parts += [f"  X({k}, {m}, {w}, 0x{poly:X}u) \\" for (k, m, w, poly, _) in INSTANCES]
    parts += ["", ""]
    for inst in INSTANCES:
        parts.append(emit_instance(*inst))
    tmp = out + ".tmp"
    with open(tmp, "w") as f:
        f.write("\n".join(parts))
    os.replace(tmp, out)
    return True


if __name__ == "__main__":
    changed = generate(force="--force" in sys.argv)
    print(("generated " if changed else "up to date ") + OUT)
