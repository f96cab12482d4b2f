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
    (12, 4, 16, 0x1100B, 3),  # config C4 (groups keep the 192 input planes out of registers)
]

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


def emit_instance(k: int, m: int, w: int, poly: int, gsize: int) -> str:
    R = bit_matrix(k, m, w, poly)
    ngroups = (k + gsize - 1) // gsize
    total_xors = 0
    body = []
    for g in range(ngroups):
        j0, j1 = g * gsize, min(k, (g + 1) * gsize)
        sub = R[:, j0 * w: j1 * w]
        nin = (j1 - j0) * w
        temps, rows = paar(sub)

        def name(v: int) -> str:
            return f"x[{v}]" if v < nin else f"t{v - nin}"

        xors = len(temps) + sum(max(0, len(r) - 1) for r in rows) + (0 if g == 0 else sum(1 for r in rows if r))
        total_xors += xors
        body += [
            f"// group {g}: data blocks {j0}..{j1 - 1}, {int(sub.sum())} ones, {len(temps)} temps, {xors} XORs",
            f"template <> struct RsNetGroup<{k}, {m}, {w}, 0x{poly:X}u, {g}> {{",
            f"  static constexpr int kFirstBlock = {j0}, kBlocks = {j1 - j0};",
            f"  static __device__ __forceinline__ void run(const uint32_t (&x)[{nin}], uint32_t (&y)[{m * w}]) {{",
        ]
        for t, (a, b) in enumerate(temps):
            body.append(f"    const uint32_t t{t} = {name(a)} ^ {name(b)};")
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
