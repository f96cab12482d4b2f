"""Seeded fuzz: random codes, geometries, alignments, erasure patterns, JIT modes and read
policies -- encode, verify (clean and one flipped bit), decode and diff-update against the
oracle, bit for bit."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
POLY = {8: 0x11D, 16: 0x1100B}


def rs():
    import paper_1312_5155_b200 as m
    return m


@pytest.mark.parametrize("case", range(200))
def test_fuzz_against_oracle(case):
    rng = np.random.default_rng(1000 + case)
    w = int(rng.choice([8, 16]))
    k = int(rng.integers(1, 21))
    m = int(rng.integers(1, 9))
    sym = w // 8
    B = int(rng.integers(1, 40000)) // sym * sym or sym
    S = int(rng.integers(1, 5))
    shift = int(rng.choice([0, 0, sym, 32, 16 * sym]))   # misalign the whole batch sometimes
    m_ = rs()
    plan = m_.Plan(k, m, w, POLY[w])
    plan.set_jit(int(rng.choice([m_.RS_JIT_OFF, m_.RS_JIT_SYNC, m_.RS_JIT_BACKGROUND])))
    plan.set_read_policy(int(rng.integers(0, 2)))
    ref = synth.stripes_array(case, range(S), k, m, B)
    oracle.encode_bulk(ref, k, m, w, POLY[w], threads=4)
    n = k + m
    flat = torch.zeros(S * n * B + shift, dtype=torch.uint8, device="cuda")
    d = flat[shift:].view(S, n, B)
    d.copy_(torch.from_numpy(ref))
    d[:, k:] = 0
    plan.encode_batch(d)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref), "encode"
    flags = torch.full((S,), 9, dtype=torch.int32, device="cuda")
    plan.verify_batch(d, flags)
    torch.cuda.synchronize()
    assert flags.cpu().tolist() == [0] * S, "verify (clean)"
    s_bad, b_bad, x_bad = int(rng.integers(S)), int(rng.integers(k + m)), int(rng.integers(B))
    d[s_bad, b_bad, x_bad] ^= 0x20
    plan.verify_batch(d, flags)
    torch.cuda.synchronize()
    assert [i for i, f in enumerate(flags.cpu().tolist()) if f] == [s_bad], "verify (one flip)"
    d[s_bad, b_bad, x_bad] ^= 0x20
    er = np.full((S, m), -1, dtype=np.int32)
    for s in range(S):
        t = int(rng.integers(0, m + 1))
        er[s, :t] = rng.choice(n, t, replace=False)
        for b in er[s, :t]:
            d[s, int(b)] = 0x6B
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref), "decode"
    c = int(rng.integers(1, k + 1))
    idx = sorted(rng.choice(k, c, replace=False).tolist())
    new = ref.copy()
    for j in idx:
        new[:, j] = rng.integers(0, 256, (S, B), dtype=np.uint8)
    want = new.copy()
    oracle.encode_bulk(want, k, m, w, POLY[w], threads=4)
    old = d[:, idx].clone()
    d[:, idx] = torch.from_numpy(np.ascontiguousarray(new[:, idx])).cuda()
    if 2 * c + m <= 255:
        plan.update_batch(d, idx, old)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), want), "update"


@pytest.mark.parametrize("case", range(40))
def test_fuzz_pattern_sequences(case):
    """Batches whose stripes draw their erasure pattern from a small set in random order
    (runs of adjacent stripes, recurring patterns, patterns still compiling): decode is
    bit-exact whichever launch plan the batch gets (one launch per pattern, per run, or the
    table kernel)."""
    rng = np.random.default_rng(5000 + case)
    w = int(rng.choice([8, 8, 16]))
    k, m = (10, 4) if w == 8 else (12, 4)
    sym = w // 8
    B = int(rng.choice([4096, 8192, 64 * 1024, int(rng.integers(1, 9000)) // sym * sym or sym]))
    S = int(rng.integers(2, 48))
    n = k + m
    m_ = rs()
    plan = m_.Plan(k, m, w, POLY[w])
    plan.set_jit(int(rng.choice([m_.RS_JIT_SYNC, m_.RS_JIT_BACKGROUND])))
    npat = int(rng.integers(1, 5))
    pats = [np.sort(rng.choice(n, int(rng.integers(1, m + 1)), replace=False)) for _ in range(npat)]
    if rng.integers(2):   # runs
        seq = []
        while len(seq) < S:
            seq += [int(rng.integers(npat))] * int(rng.integers(1, 8))
        seq = seq[:S]
    else:                 # independent draws
        seq = [int(rng.integers(npat)) for _ in range(S)]
    er = np.full((S, m), -1, dtype=np.int32)
    for s, p in enumerate(seq):
        er[s, :len(pats[p])] = pats[p]
    if rng.integers(2):
        plan.prepare(er)
    ref = synth.stripes_array(7000 + case, range(S), k, m, B)
    oracle.encode_bulk(ref, k, m, w, POLY[w], threads=4)
    bad = ref.copy()
    for s in range(S):
        for b in er[s]:
            if b >= 0:
                bad[s, b] = 0xA5
    d = torch.from_numpy(bad).cuda()
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
