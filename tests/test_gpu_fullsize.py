"""GPU parity at BASELINE.json's full sizes (C1-C5), in bench.py's launch configuration.

The whole batch is encoded and decoded on the device exactly as bench.py times it
(default plan: compiled networks for encode, per-pattern JIT kernels after
rs_poly_prepare for decode), and EVERY byte of every stripe is compared with the CPU
oracle (oracle/fullcheck.py, all host cores, streamed stripe by stripe):

* encode: the device batch equals the oracle's long division (encode_bulk) of the
  seeded inputs, data and parity;
* decode: after the erased blocks are scribbled and decoded on the device, the batch
  equals the oracle's own decode (decode_bulk) of its codewords with the
  same erasures; the device round trip (decode restores the encoded batch) is kept as
  an extra check.
Plus 64 single columns drawn at random over the batch re-encoded by the literal
column long division (oracle.encode_column).
"""
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import fullcheck

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

THREADS = max(1, len(os.sched_getaffinity(0)))


def fetcher(st):
    """Device -> host copy of the listed stripes (uint8 [len][n][B])."""
    return lambda ids: np.stack([st[s].cpu().numpy() for s in ids])


def rs():
    import paper_1312_5155_b200 as m
    return m


def run_config(cfg, seed=0):
    c = synth.CONFIGS[cfg]
    k, m, w, B, S, poly = c["k"], c["m"], c["w"], c["block_bytes"], c["stripes"], c["poly"]
    n = k + m
    seed = c["seed"] if c["seed"] is not None else seed
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    st = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
    m_.synth_fill(st, k, seed=seed)
    plan.encode_batch(st)
    torch.cuda.synchronize()

    # ---- encode vs the oracle: every byte of every stripe ----
    picks = sorted({0, S // 2, S - 1})
    r = fullcheck.check_encode(fetcher(st), dict(c, seed=seed), range(S), THREADS)
    assert r["mismatched_stripes"] == [], f"{cfg}: encode mismatch on stripes {r['mismatched_stripes']}"
    assert r["bytes"] == S * n * B
    rng = np.random.default_rng(7)
    sym = w // 8
    for _ in range(64):
        s = int(rng.integers(S))
        col = int(rng.integers(B // sym)) * sym
        data = synth.stripes_array(seed, [s], k, m, B)[0, :k, col:col + sym]
        words = [int.from_bytes(bytes(data[j]), "little") for j in range(k)]
        par = oracle.encode_column(words, m, w, poly)
        got = st[s, k:, col:col + sym].cpu().numpy()
        assert [int.from_bytes(bytes(got[i]), "little") for i in range(m)] == par, f"{cfg}: column {s}/{col}"
    return plan, st, (k, m, w, B, S, poly, n, seed, picks)


def check_decode(plan, st, er, geom, cfg):
    k, m, w, B, S, poly, n, seed, picks = geom
    plan.prepare(er)
    golden = st.clone()
    for s in range(S):
        idx = er[s][er[s] >= 0]
        if len(idx):
            st[s, torch.from_numpy(idx.astype(np.int64)).cuda()] = 0xA5
    plan.decode_batch(st, er)
    torch.cuda.synchronize()
    assert torch.equal(st, golden), f"{cfg}: decode did not restore every erased byte"
    del golden
    # every byte of every stripe equals the oracle's own decode of its codewords
    c = dict(synth.CONFIGS[cfg], seed=seed)
    r = fullcheck.check_decode(fetcher(st), c, er, range(S), THREADS)
    assert r["mismatched_stripes"] == [], f"{cfg}: decode differs from the oracle on {r['mismatched_stripes']}"
    assert r["bytes"] == S * n * B


@pytest.mark.parametrize("cfg", ["C1", "C3", "C4", "C5"])
def test_fullsize_encode_decode(cfg):
    plan, st, geom = run_config(cfg)
    er = synth.erasure_table(cfg, geom[7], geom[4])
    check_decode(plan, st, er, geom, cfg)
    del st
    torch.cuda.empty_cache()


def test_fullsize_c2_encode_and_decode_sweep():
    """C2: encode the 256 x 6 x 1 MiB batch; decode every single-block pattern and every
    data-only triple on stripes 0..3 (116 decodes in one batched call)."""
    plan, st, geom = run_config("C2")
    k, m, w, B, S, poly, n, seed, picks = geom
    sweep = synth.c2_decode_sweep(k, m)
    batch = torch.stack([st[s] for s, _ in sweep])
    er = np.full((len(sweep), m), -1, dtype=np.int32)
    for i, (_, p) in enumerate(sweep):
        er[i, :len(p)] = p
    golden = batch.clone()
    for i, (_, p) in enumerate(sweep):
        batch[i, torch.tensor(p, dtype=torch.int64).cuda()] = 0
    plan.prepare(er)
    plan.decode_batch(batch, er)
    torch.cuda.synchronize()
    assert torch.equal(batch, golden)
    # every sweep entry, every byte: the oracle's own decode of the stripe with that pattern
    want = golden.cpu().numpy()
    lost = want.copy()
    for i, (_, p) in enumerate(sweep):
        lost[i, p] = 0x5A
    oracle.decode_bulk(lost, er, k, m, w, poly, threads=THREADS)
    assert np.array_equal(lost, want)
    assert np.array_equal(batch.cpu().numpy(), lost)
    del st, batch, golden
    torch.cuda.empty_cache()
