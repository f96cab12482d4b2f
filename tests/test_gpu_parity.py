"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit for bit.

Every expected value comes from oracle/ on the same seeded inputs (synth/).  Sizes
span several 32-column units and CTAs plus a ragged tail; edge cases cover empty
patterns, parity-only/data-only/mixed patterns, every pattern of small codes,
misaligned blocks (generic scalar path) and the host-memory (e2e) entry points.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

P8, P16 = 0x11D, 0x1100B


class _TablesOnly:
    """The table-driven / compiled-network kernels (JIT off); tests/test_gpu_jit.py covers the JIT path."""

    def __init__(self, mod):
        self._m = mod

    def __getattr__(self, name):
        return getattr(self._m, name)

    def Plan(self, *a, **kw):
        p = self._m.Plan(*a, **kw)
        p.set_jit(self._m.RS_JIT_OFF)
        return p


def rs():
    import paper_1312_5155_b200 as m
    return _TablesOnly(m)


def host_stripes(k, m, B, S, seed=0, stripe0=0):
    return synth.stripes_array(seed, range(stripe0, stripe0 + S), k, m, B)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def oracle_encoded(st, k, m, w, poly):
    ref = st.copy()
    oracle.encode_bulk(ref, k, m, w, poly, threads=8)
    return ref


# (k, m, w, poly, B): bit-sliced instances and generic fallbacks, B with ragged tails
CASES = [
    (10, 4, 8, P8, 3 * 4096 + 40),     # sliced + generic tail (40 B)
    (6, 3, 8, P8, 64 * 1024 + 17),
    (4, 3, 8, P8, 1000),
    (10, 2, 8, P8, 8192),
    (12, 4, 16, P16, 2 * 8192 + 6),    # sliced w16 + tail
    (5, 2, 8, P8, 5000),               # generic only
    (10, 6, 8, P8, 4096 + 3),          # generic, m > 4 (two output groups)
    (20, 8, 8, P8, 777),
    (10, 4, 16, P16, 4098),            # generic w16
    (1, 1, 8, P8, 100),                # RAID-5 degenerate
]


@pytest.mark.parametrize("k,m,w,poly,B", CASES)
def test_encode_batch_matches_oracle(k, m, w, poly, B):
    S = 5
    st = host_stripes(k, m, B, S, seed=1)
    ref = oracle_encoded(st, k, m, w, poly)
    plan = rs().Plan(k, m, w, poly)
    d = to_dev(st)
    d[:, k:] = 0xA5  # parity is overwritten, not accumulated
    plan.encode_batch(d)
    torch.cuda.synchronize()
    got = d.cpu().numpy()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("k,m,w,poly,B", CASES)
def test_decode_batch_random_patterns(k, m, w, poly, B):
    S = 24
    n = k + m
    st = oracle_encoded(host_stripes(k, m, B, S, seed=2), k, m, w, poly)
    rng = np.random.default_rng(k * 7 + m)
    er = np.full((S, m), -1, dtype=np.int32)
    for s in range(S):
        t = int(rng.integers(0, m + 1)) if s > 3 else [m, 0, 1, m][s]
        e = rng.choice(n, t, replace=False)
        rng.shuffle(e)
        er[s, :t] = e
    bad = st.copy()
    for s in range(S):
        for b in er[s]:
            if b >= 0:
                bad[s, b] = rng.integers(0, 256, B, dtype=np.uint8)
    plan = rs().Plan(k, m, w, poly)
    d = to_dev(bad)
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), st)


@pytest.mark.parametrize("k,m,w,poly", [(4, 3, 8, P8), (6, 3, 8, P8), (10, 4, 8, P8), (12, 4, 16, P16)])
def test_decode_every_pattern(k, m, w, poly):
    """All sum_{t<=m} C(n,t) patterns at once (1471 for (10,4), 2517 for (12,4)), one per stripe."""
    n = k + m
    pats = [p for t in range(m + 1) for p in itertools.combinations(range(n), t)]
    B = 96 if w == 8 else 128  # 3 (w8) / 2 (w16) bit-sliced units + a ragged tail when B % 32
    base = oracle_encoded(host_stripes(k, m, B, 1, seed=3), k, m, w, poly)[0]
    st = np.repeat(base[None], len(pats), axis=0)
    er = np.full((len(pats), m), -1, dtype=np.int32)
    bad = st.copy()
    for s, p in enumerate(pats):
        er[s, :len(p)] = p
        for b in p:
            bad[s, b] = (s * 31 + b) & 0xFF
    plan = rs().Plan(k, m, w, poly)
    d = to_dev(bad)
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), st)


def test_paper_example_on_gpu():
    """P:199-208 and P:233-301 through the C ABI: 48,6,112,70 -> 243,125,142; erase d0..d2 -> back."""
    plan = rs().Plan(4, 3, 8, P8)
    B = 64
    data = [torch.full((B,), v, dtype=torch.uint8, device="cuda") for v in (48, 6, 112, 70)]
    par = [torch.zeros(B, dtype=torch.uint8, device="cuda") for _ in range(3)]
    plan.encode(data, par, B)
    torch.cuda.synchronize()
    assert [int(p[0]) for p in par] == [243, 125, 142] and all(bool((p == p[0]).all()) for p in par)
    for b in data[:3]:
        b.zero_()
    plan.decode(data + par, B, [2, 0, 1])
    torch.cuda.synchronize()
    assert [int(b[5]) for b in data] == [48, 6, 112, 70]


@pytest.mark.parametrize("k,m,w,poly", [(10, 4, 8, P8), (12, 4, 16, P16), (5, 2, 8, P8)])
def test_pointer_api_and_misaligned_blocks(k, m, w, poly):
    """Single-stripe pointer API; blocks offset by one symbol so the sliced path cannot be used."""
    B = 4096 + 2 * 7
    sym = w // 8
    st = host_stripes(k, m, B, 1, seed=4)[0]
    ref = oracle_encoded(st[None], k, m, w, poly)[0]
    plan = rs().Plan(k, m, w, poly)
    for shift in (0, sym):
        bufs = [torch.zeros(B + 64, dtype=torch.uint8, device="cuda") for _ in range(k + m)]
        views = [b[shift:shift + B] for b in bufs]
        for j in range(k):
            views[j].copy_(torch.from_numpy(st[j]))
        plan.encode(views[:k], views[k:], B)
        torch.cuda.synchronize()
        got = np.stack([v.cpu().numpy() for v in views])
        assert np.array_equal(got, ref)
        er = [k + m - 1, 0, k // 2][:m]
        for b in er:
            views[b].fill_(0x77)
        plan.decode(views, B, er)
        torch.cuda.synchronize()
        assert np.array_equal(np.stack([v.cpu().numpy() for v in views]), ref)


def test_strided_layout_with_padding():
    """Batch layout with block_stride > B and stripe_stride > n*block_stride."""
    k, m, B = 10, 4, 2048 + 96
    S = 3
    st = host_stripes(k, m, B, S, seed=5)
    ref = oracle_encoded(st, k, m, 8, P8)
    big = torch.zeros((S, k + m, B + 160), dtype=torch.uint8, device="cuda")
    big = torch.zeros((S + 1) * (k + m) * (B + 160) + 512, dtype=torch.uint8, device="cuda")
    view = big[: S * (k + m) * (B + 160)].view(S, k + m, B + 160)[:, :, :B]
    view.copy_(torch.from_numpy(st))
    plan = rs().Plan(k, m)
    plan.encode_batch(view)
    torch.cuda.synchronize()
    assert np.array_equal(view.cpu().numpy(), ref)


def test_empty_and_noop_cases():
    plan = rs().Plan(10, 4)
    d = to_dev(oracle_encoded(host_stripes(10, 4, 1024, 2, seed=6), 10, 4, 8, P8))
    before = d.clone()
    plan.decode_batch(d, np.full((2, 4), -1, dtype=np.int32))  # no erasures: no-op
    plan.decode(list(d[0]), 1024, [])
    torch.cuda.synchronize()
    assert torch.equal(d, before)
    plan.encode_batch(d[:0])  # zero stripes


def test_error_codes():
    m = rs()
    plan = m.Plan(10, 4)
    d = torch.zeros((2, 14, 64), dtype=torch.uint8, device="cuda")
    with pytest.raises(m.RSError) as e:
        plan.decode(list(d[0]), 64, [0, 1, 2, 3, 4])
    assert e.value.status == 4
    with pytest.raises(m.RSError) as e:
        plan.decode(list(d[0]), 64, [1, 1])
    assert e.value.status == 5
    with pytest.raises(m.RSError) as e:
        plan.decode_batch(d, np.array([[0, 14, -1, -1], [-1] * 4], dtype=np.int32))
    assert e.value.status == 5
    p16 = m.Plan(12, 4, 16)
    with pytest.raises(m.RSError) as e:
        p16.encode_batch(torch.zeros((1, 16, 63), dtype=torch.uint8, device="cuda"))
    assert e.value.status == 3


def test_synth_matches_host():
    k, m, B, S = 10, 4, 4096 + 5, 3
    d = torch.zeros((S, k + m, B), dtype=torch.uint8, device="cuda")
    rs().synth_fill(d, k, seed=7, stripe0=11)
    torch.cuda.synchronize()
    ref = host_stripes(k, m, B, S, seed=7, stripe0=11)
    assert np.array_equal(d.cpu().numpy(), ref)


@pytest.mark.parametrize("k,m,w,poly", [(10, 4, 8, P8), (12, 4, 16, P16)])
def test_host_entry_points(k, m, w, poly):
    """rs_poly_encode_host / rs_poly_decode_host: pinned host buffers, chunked through HBM."""
    B, S = 96 * 1024 + 32, 7
    n = k + m
    st = host_stripes(k, m, B, S, seed=8)
    ref = oracle_encoded(st, k, m, w, poly)
    h = torch.from_numpy(st).pin_memory()
    plan = rs().Plan(k, m, w, poly)
    h2d, d2h = plan.encode_host(h)
    assert np.array_equal(h.numpy(), ref)
    assert h2d == S * k * B and d2h == S * m * B
    er = synth.erasure_table("C5", 0, S) if n == 14 else np.array(
        [synth.erasure_draw(0, s, range(n), m) for s in range(S)], dtype=np.int32)
    er[1] = -1
    hv = h.numpy()
    for s in range(S):
        for b in er[s]:
            if b >= 0:
                hv[s, b] = 0
    h2d, d2h = plan.decode_host(h, er)
    assert np.array_equal(h.numpy(), ref)
    t_total = int((er >= 0).sum())
    assert d2h == t_total * B and h2d == (S - 1) * (n * B) - (t_total * B)


def test_launch_counter_moves():
    m = rs()
    before = m.launch_count()
    plan = m.Plan(10, 4)
    d = torch.zeros((1, 14, 4096), dtype=torch.uint8, device="cuda")
    plan.encode_batch(d)
    torch.cuda.synchronize()
    assert m.launch_count() > before


@pytest.mark.parametrize("k,m,w,poly,B", [(223, 32, 8, P8, 777), (240, 15, 8, P8, 64), (1, 1, 8, P8, 1),
                                          (3, 2, 16, P16, 2), (100, 32, 16, P16, 34)])
def test_extreme_geometries(k, m, w, poly, B):
    """Maximum n = 255 (w8) and m = 32, one-symbol blocks: encode and an m-erasure decode."""
    S = 2
    ref = oracle_encoded(host_stripes(k, m, B, S, seed=8), k, m, w, poly)
    plan = rs().Plan(k, m, w, poly)
    d = to_dev(ref)
    d[:, k:] = 0
    plan.encode_batch(d)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    rng = np.random.default_rng(k)
    er = np.stack([np.sort(rng.choice(k + m, m, replace=False)) for _ in range(S)]).astype(np.int32)
    for s in range(S):
        d[s, torch.from_numpy(er[s].astype(np.int64)).cuda()] = 0x99
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)


@pytest.mark.parametrize("k,m,w,poly,B", [(10, 4, 8, P8, 4096 + 40), (12, 4, 16, P16, 8192 + 6), (5, 2, 8, P8, 999)])
def test_no_writes_outside_blocks(k, m, w, poly, B):
    """Every block sits between canary bytes (padding of the block and stripe strides); encode,
    decode (JIT and table paths), diff-update and the XOR reduction leave the canaries intact."""
    import paper_1312_5155_b200 as mod
    S, pad = 3, 96
    ref = oracle_encoded(host_stripes(k, m, B, S, seed=9), k, m, w, poly)
    for jit in (mod.RS_JIT_SYNC, mod.RS_JIT_OFF):
        big = torch.full((S, k + m, B + pad), 0xA7, dtype=torch.uint8, device="cuda")
        view = big[:, :, :B]
        view.copy_(torch.from_numpy(ref))
        view[:, k:] = 0
        plan = mod.Plan(k, m, w, poly)
        plan.set_jit(jit)
        plan.encode_batch(view)
        er = np.array([[0, k, -1, -1][:m] + [-1] * (m - 2)] * S, dtype=np.int32)[:, :m]
        for s in range(S):
            view[s, torch.from_numpy(er[s][er[s] >= 0].astype(np.int64)).cuda()] = 0
        plan.decode_batch(view, er)
        old = view[:, [1]].clone()
        view[:, 1] ^= 0x5C
        plan.update_batch(view, [1], old)
        view[:, 1] ^= 0x5C
        plan.update_batch(view, [1], old ^ 0x5C)
        plan.xor_reduce([view[s, 0] for s in range(S)], [[view[s, 0], view[s, 2], view[s, 2]] for s in range(S)], B)
        torch.cuda.synchronize()
        assert np.array_equal(view.cpu().numpy(), ref)
        assert bool((big[:, :, B:] == 0xA7).all()), "write outside a block"


@pytest.mark.parametrize("units,tail", [(48, 0), (33, 32), (33, 10), (31, 0), (96, 6), (65, 32), (1, 2)])
@pytest.mark.parametrize("jit", [True, False])
def test_w16_partial_warp_layouts(units, tail, jit):
    """GF(2^16) unit layout (bitslice_device.cuh unit_offset): full warps interleave their two
    32-byte halves 1 KiB apart, a warp cut by the end of the block keeps them contiguous.
    Block lengths with 1..96 units (partial warps, one full warp + a partial one) and ragged
    tails, encode + a mixed 4-erasure decode, compiled/table and JIT kernels, vs the oracle."""
    import paper_1312_5155_b200 as mod
    k, m, S = 12, 4, 3
    B = 64 * units + tail
    st = host_stripes(k, m, B, S, seed=9)
    ref = oracle_encoded(st, k, m, 16, P16)
    plan = mod.Plan(k, m, 16, P16)
    plan.set_jit(mod.RS_JIT_SYNC if jit else mod.RS_JIT_OFF)
    d = to_dev(st)
    plan.encode_batch(d)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    er = np.array([[0, 5, 12, 15], [3, 4, 11, 13], [13, 14, -1, -1]], dtype=np.int32)
    for s in range(S):
        d[s, torch.from_numpy(er[s][er[s] >= 0].astype(np.int64)).cuda()] = 0x3C
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    if jit and B % 32 == 0:  # (the bit-sliced body needs 32-byte aligned blocks)
        assert plan.stats()["jit_launches"] > 0
