"""Test-side GF(2^w) arithmetic, deliberately a DIFFERENT algorithm from the oracle's.

The oracle multiplies by interleaved shift-and-add with reduction at every step
(oracle/rs_oracle.c: orc_gf_mul).  Here a product is formed as a full carry-less
polynomial product in GF(2)[x] first (up to degree 2w-2), and only then reduced
modulo prim_poly by polynomial long division from the top bit down.  Agreement of
the two on every pair (w=8) pins the oracle's multiply to the definition of the
field GF(2)[x]/(prim_poly) rather than to itself.
"""
from __future__ import annotations

import numpy as np


def clmul(a: int, b: int) -> int:
    """Carry-less product of two GF(2)[x] polynomials encoded as ints."""
    r = 0
    i = 0
    while b >> i:
        if (b >> i) & 1:
            r ^= a << i
        i += 1
    return r


def polymod(a: int, poly: int) -> int:
    """a mod poly in GF(2)[x] by long division."""
    dp = poly.bit_length() - 1
    while a.bit_length() - 1 >= dp:
        a ^= poly << (a.bit_length() - 1 - dp)
    return a


def mul(a: int, b: int, poly: int) -> int:
    return polymod(clmul(a, b), poly)


def mul_np(a: np.ndarray, b: np.ndarray, w: int, poly: int) -> np.ndarray:
    """Vectorised: carry-less product to 2w-1 bits, then reduce from the top bit down."""
    a = a.astype(np.uint64)
    b = b.astype(np.uint64)
    r = np.zeros_like(a)
    for i in range(w):
        r ^= np.where((b >> np.uint64(i)) & np.uint64(1), a << np.uint64(i), np.uint64(0))
    for bit in range(2 * w - 2, w - 1, -1):
        r ^= np.where((r >> np.uint64(bit)) & np.uint64(1), np.uint64(poly) << np.uint64(bit - w), np.uint64(0))
    return r.astype(np.uint32)


class Tables:
    """log/exp tables generated from :func:`mul` (for fast vectorised checks)."""

    def __init__(self, w: int, poly: int):
        self.w, self.poly, self.q = w, poly, (1 << w) - 1
        self.exp = np.zeros(2 * self.q, dtype=np.int64)
        self.log = np.full(1 << w, -1, dtype=np.int64)
        x = 1
        for i in range(self.q):
            self.exp[i] = self.exp[i + self.q] = x
            if self.log[x] != -1:
                raise ValueError("alpha=2 is not primitive for this polynomial")
            self.log[x] = i
            x = mul(x, 2, poly)
        if x != 1:
            raise ValueError("alpha=2 is not primitive for this polynomial")

    def mul(self, a, b):
        a = np.asarray(a, dtype=np.int64)
        b = np.asarray(b, dtype=np.int64)
        out = self.exp[(self.log[np.maximum(a, 1)] + self.log[np.maximum(b, 1)]) % self.q]
        return np.where((a == 0) | (b == 0), 0, out)

    def pow_alpha(self, e: int) -> int:
        return int(self.exp[e % self.q])

    def eval_positions(self, coeffs_by_pos: np.ndarray, x: int) -> np.ndarray:
        """Evaluate sum_p c_p x^p for each column; coeffs_by_pos is [n][cols]."""
        acc = np.zeros(coeffs_by_pos.shape[1:], dtype=np.int64)
        for p in range(coeffs_by_pos.shape[0] - 1, -1, -1):
            acc = self.mul(acc, x) ^ coeffs_by_pos[p]
        return acc


def positions(k: int, m: int) -> list[int]:
    """pos(b) for API block index b: data b -> m+b, parity b -> b-k."""
    return [m + b if b < k else b - k for b in range(k + m)]


def by_position(codeword_api, k: int, m: int) -> np.ndarray:
    cw = np.asarray(codeword_api, dtype=np.int64)
    out = np.zeros_like(cw)
    for b, p in enumerate(positions(k, m)):
        out[p] = cw[b]
    return out
