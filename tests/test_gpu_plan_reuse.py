"""Decode-plan reuse: a stripe's columns are independent codewords,
so decoding the block range in two calls -- first half, then second half, the second call
reusing the cached pattern plan and kernels -- restores the same bytes as one call over the
whole range.  Checked bit for bit against the oracle's codewords, with the split aligned (both
halves on the bit-sliced kernels) and misaligned (the second half on the generic kernel)."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P8, P16 = 0x11D, 0x1100B


@pytest.mark.parametrize("k,m,w,poly,B,split", [
    (10, 4, 8, P8, 64 * 1024 + 48, 32 * 1024),       # aligned split
    (10, 4, 8, P8, 64 * 1024 + 48, 32 * 1024 + 3),   # misaligned second half
    (12, 4, 16, P16, 48 * 1024 + 6, 16 * 1024),
    (12, 4, 16, P16, 48 * 1024 + 6, 16 * 1024 + 2),
])
def test_decode_halves_equal_whole(k, m, w, poly, B, split):
    import paper_1312_5155_b200 as rs
    S = 4
    ref = synth.stripes_array(90 + split % 7, range(S), k, m, B)
    oracle.encode_bulk(ref, k, m, w, poly, threads=4)
    er = synth.erasure_table("C5", 5, S) if w == 8 else synth.erasure_table("C4", 5, S)
    plan = rs.Plan(k, m, w, poly)
    plan.set_jit(rs.RS_JIT_SYNC)
    bad = ref.copy()
    for s in range(S):
        bad[s, [b for b in er[s] if b >= 0]] = 0xC3
    whole = torch.from_numpy(bad).cuda()
    plan.decode_batch(whole, er)
    halves = torch.from_numpy(bad).cuda()
    plan.decode_batch(halves[:, :, :split], er)
    n0 = plan.stats()["patterns"]
    plan.decode_batch(halves[:, :, split:], er)
    torch.cuda.synchronize()
    assert plan.stats()["patterns"] == n0              # the second call reused the plans
    assert np.array_equal(whole.cpu().numpy(), ref)
    assert np.array_equal(halves.cpu().numpy(), ref)
