"""Seeded synthetic inputs for the RS-poly workloads.

This module is the ONE thing the oracle side (``oracle/``, ``tests/``) and the
product side (``paper_1312_5155_b200``) may both use.  It holds no Reed-Solomon
or GF(2^w) arithmetic: only a counter-based generator (splitmix64) and the
erasure-pattern draw built on it.  The CUDA library carries its own copy of the
same counter-based generator (``csrc/synth.cu``) so that 20-30 GiB batches can
be generated in HBM; ``tests/test_synth.py`` checks the two agree bit-for-bit.

Recipe (the paper stages uniform random data in memory):

* data word q (8 bytes, little-endian) of data block j of stripe s under the
  config seed sigma is ``splitmix64(sigma<<48 | s<<32 | j<<24 | q)``;
* the erasure stream of stripe s is ``r_i = splitmix64(sigma<<48 | s<<32 |
  0xFF<<24 | i)``; a partial Fisher-Yates over the candidate list takes
  ``r_i mod (len - i)`` as the swap index; the chosen set is sorted ascending.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_scalar(x: int) -> int:
    """One splitmix64 output for counter x (pure Python reference)."""
    z = (x + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 over a uint64 array (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _check_ranges(seed: int, stripe: int, block: int, nwords: int) -> None:
    if not (0 <= seed < 1 << 16 and 0 <= stripe < 1 << 16 and 0 <= block < 0xFF and nwords <= 1 << 24):
        raise ValueError("generator counter out of range (seed<2^16, stripe<2^16, block<255, words<=2^24)")


def data_block(seed: int, stripe: int, block: int, block_bytes: int) -> np.ndarray:
    """Bytes of data block ``block`` of stripe ``stripe`` (uint8, length block_bytes)."""
    nwords = (block_bytes + 7) // 8
    _check_ranges(seed, stripe, block, nwords)
    base = (seed << 48) | (stripe << 32) | (block << 24)
    ctr = np.arange(nwords, dtype=np.uint64) | np.uint64(base)
    return splitmix64(ctr).view(np.uint8)[:block_bytes].copy()


def stripes_array(seed: int, stripe_ids, k: int, m: int, block_bytes: int, threads: int = 1) -> np.ndarray:
    """``[len(stripe_ids)][k+m][block_bytes]`` uint8 with data filled, parity zeroed.

    ``threads`` > 1 fills the blocks from a thread pool (numpy's ufunc loops release the GIL)."""
    stripe_ids = list(stripe_ids)
    out = np.zeros((len(stripe_ids), k + m, block_bytes), dtype=np.uint8)
    jobs = [(si, s, j) for si, s in enumerate(stripe_ids) for j in range(k)]

    def fill(job):
        si, s, j = job
        out[si, j] = data_block(seed, s, j, block_bytes)

    if threads > 1 and len(jobs) > 1:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(threads, len(jobs))) as ex:
            list(ex.map(fill, jobs))
    else:
        for job in jobs:
            fill(job)
    return out


def erasure_draw(seed: int, stripe: int, candidates, count: int) -> list[int]:
    """Partial Fisher-Yates: ``count`` distinct entries of ``candidates``, sorted."""
    cand = list(candidates)
    if count > len(cand):
        raise ValueError("more erasures than candidates")
    base = (seed << 48) | (stripe << 32) | (0xFF << 24)
    for i in range(count):
        r = splitmix64_scalar(base | i)
        j = i + r % (len(cand) - i)
        cand[i], cand[j] = cand[j], cand[i]
    return sorted(cand[:count])


# ---------------------------------------------------------------------------
# The five BASELINE.json workloads (SURVEY.md §8(d) "Inputs per config").
# ---------------------------------------------------------------------------
CONFIGS = {
    # name: (k, m, w, prim_poly, n_stripes, block_bytes, seed)
    "C1": dict(k=10, m=4, w=8, poly=0x11D, stripes=1, block_bytes=64 << 10, seed=0),
    "C2": dict(k=6, m=3, w=8, poly=0x11D, stripes=256, block_bytes=1 << 20, seed=0),
    "C3": dict(k=10, m=4, w=8, poly=0x11D, stripes=512, block_bytes=4 << 20, seed=0),
    "C4": dict(k=12, m=4, w=16, poly=0x1100B, stripes=256, block_bytes=8 << 20, seed=0),
    "C5": dict(k=10, m=4, w=8, poly=0x11D, stripes=51, block_bytes=16 << 20, seed=None),  # seed = rank
}


def erasure_pattern(config: str, seed: int, stripe: int) -> list[int]:
    """Per-stripe erasure list (API block indices; data 0..k-1, parity k..n-1).

    C1/C4/C5: ``m`` of all ``n`` blocks.  C3: even stripes draw 4 of the k data
    blocks, odd stripes 4 of all n ("50% of patterns restricted to data blocks").
    C2 uses the explicit sweep of :func:`c2_decode_sweep` instead.
    """
    c = CONFIGS[config]
    k, m = c["k"], c["m"]
    n = k + m
    if config == "C3" and stripe % 2 == 0:
        return erasure_draw(seed, stripe, range(k), m)
    if config == "C2":
        raise ValueError("C2 uses c2_decode_sweep()")
    return erasure_draw(seed, stripe, range(n), m)


def erasure_table(config: str, seed: int, n_stripes: int) -> np.ndarray:
    """``[n_stripes][m]`` int32, -1 padded (the layout rs_poly_decode_batch takes)."""
    m = CONFIGS[config]["m"]
    tab = np.full((n_stripes, m), -1, dtype=np.int32)
    for s in range(n_stripes):
        e = erasure_pattern(config, seed, s)
        tab[s, : len(e)] = e
    return tab


def c2_decode_sweep(k: int = 6, m: int = 3, stripes=(0, 1, 2, 3)) -> list[tuple[int, list[int]]]:
    """C2: every single-block pattern (9) and every 3-block data-only pattern (20) on stripes 0..3."""
    from itertools import combinations

    pats = [[b] for b in range(k + m)] + [list(c) for c in combinations(range(k), 3)]
    return [(s, p) for s in stripes for p in pats]
