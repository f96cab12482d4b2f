"""GPU parity at BASELINE.json's full sizes (C1-C5), in bench.py's launch configuration.

The whole batch is encoded and decoded on the device exactly as bench.py times it
(default plan: compiled networks for encode, per-pattern JIT kernels after
rs_poly_prepare for decode).  The oracle cannot redo 11-32 GiB in test time, so:

* encode: sampled columns -- the first and last 64 KiB of every block of stripes
  0, S/2 and S-1, plus 64 single columns drawn at random over the whole batch --
  are recomputed by oracle/ (bulk long division) from the seeded inputs;
* decode: every erased byte of every stripe must come back (property valid at any
  size: decode(encode(d) with E erased) = encode(d)), and on the sampled stripes
  the oracle's own decode of the sampled columns must equal the GPU's output.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SPAN = 64 << 10


def rs():
    import paper_1312_5155_b200 as m
    return m


def sampled_columns(host_or_dev, B, w):
    """[S'][n][2*SPAN] view of the first and last SPAN bytes of each block (numpy)."""
    span = min(B // 2, SPAN) // (w // 8) * (w // 8)
    a = host_or_dev
    return np.concatenate([a[..., :span], a[..., B - span:]], axis=-1).copy()


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

    # ---- encode vs the oracle on sampled columns ----
    picks = sorted({0, S // 2, S - 1})
    for s in picks:
        ref = sampled_columns(synth.stripes_array(seed, [s], k, m, B), B, w)
        oracle.encode_bulk(ref, k, m, w, poly, threads=4)
        got = sampled_columns(st[s:s + 1].cpu().numpy(), B, w)
        assert np.array_equal(got, ref), f"{cfg}: encode mismatch on stripe {s}"
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
    # the oracle's decode of the sampled columns equals the GPU's
    for s in picks:
        cols = sampled_columns(golden[s:s + 1].cpu().numpy(), B, w)
        want = cols.copy()
        for b in er[s][er[s] >= 0]:
            cols[0, b] = 0
        oracle.decode_bulk(cols, er[s:s + 1], k, m, w, poly, threads=4)
        assert np.array_equal(cols, want), f"{cfg}: oracle decode of stripe {s} disagrees"
    del golden


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
    # one sweep entry per pattern checked against the oracle on sampled columns
    for i in range(0, len(sweep), 4):
        cols = sampled_columns(golden[i:i + 1].cpu().numpy(), B, w)
        want = cols.copy()
        for b in sweep[i][1]:
            cols[0, b] = 0
        oracle.decode_bulk(cols, er[i:i + 1], k, m, w, poly, threads=4)
        assert np.array_equal(cols, want)
    del st, batch, golden
    torch.cuda.empty_cache()
