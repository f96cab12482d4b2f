"""Whole-batch bit-exact verification against the oracle -- TEST INFRASTRUCTURE ONLY.

Used by ``tests/test_gpu_fullsize.py`` and by ``bench.py`` outside its timed region
("the bit-exact verification still covers all stripes").  Encoding
is a unique remainder and decoding for |E| <= m a unique solution (MDS), so the
device's batch must equal the oracle's byte for byte.

Nothing here touches a GPU: the caller passes ``fetch(ids) -> uint8 [len(ids)][n][B]``
(a device -> host copy of those stripes).  The oracle's inputs come from ``synth``
(host generator) only; its expected values come from ``encode_bulk`` / ``decode_bulk``
(oracle/rs_oracle.c), never from the CUDA path.

Cost: one synth + oracle encode per stripe for ``check_encode``; synth + encode +
decode per stripe for ``check_decode``; the work is streamed in chunks of ``threads``
stripes, so host memory stays at two chunks.
"""
from __future__ import annotations

import time

import numpy as np

import synth

from . import decode_bulk, encode_bulk


def _chunks(ids, size):
    ids = list(ids)
    for i in range(0, len(ids), size):
        yield ids[i:i + size]


def oracle_codewords(c: dict, ids, threads: int) -> np.ndarray:
    """Oracle codewords (data from synth, parity by the oracle's long division) of stripes ``ids``."""
    st = synth.stripes_array(c["seed"], ids, c["k"], c["m"], c["block_bytes"], threads=threads)
    encode_bulk(st, c["k"], c["m"], c["w"], c["poly"], threads=max(1, min(threads, len(ids))))
    return st


def check_encode(fetch, c: dict, ids, threads: int) -> dict:
    """Every byte of every stripe in ``ids`` (data and parity) vs the oracle's encode."""
    t0, bad, nbytes = time.perf_counter(), [], 0
    for chunk in _chunks(ids, max(1, threads)):
        want = oracle_codewords(c, chunk, threads)
        got = fetch(chunk)
        for i, s in enumerate(chunk):
            if not np.array_equal(got[i], want[i]):
                bad.append(int(s))
        nbytes += want.nbytes
        del want, got
    return {"stripes": len(list(ids)), "bytes": nbytes, "mismatched_stripes": bad,
            "seconds": round(time.perf_counter() - t0, 2)}


def check_decode(fetch, c: dict, erasures: np.ndarray, ids, threads: int, scribble: int = 0xEE) -> dict:
    """Every byte of every stripe in ``ids`` after the device decode vs the oracle's own decode
     of its codeword with the same blocks erased (their contents scribbled)."""
    t0, bad, nbytes = time.perf_counter(), [], 0
    m = c["m"]
    for chunk in _chunks(ids, max(1, threads)):
        st = oracle_codewords(c, chunk, threads)
        er = np.ascontiguousarray(erasures[chunk], dtype=np.int32).reshape(len(chunk), m)
        for i in range(len(chunk)):
            lost = er[i][er[i] >= 0]
            st[i, lost] = scribble
        decode_bulk(st, er, c["k"], m, c["w"], c["poly"], threads=max(1, min(threads, len(chunk))))
        got = fetch(chunk)
        for i, s in enumerate(chunk):
            if not np.array_equal(got[i], st[i]):
                bad.append(int(s))
        nbytes += st.nbytes
        del st, got
    return {"stripes": len(list(ids)), "bytes": nbytes, "mismatched_stripes": bad,
            "seconds": round(time.perf_counter() - t0, 2)}
