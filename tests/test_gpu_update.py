"""GPU parity of the diff-update (parity ^= encode(new - old) of the changed
blocks) against the oracle's full re-encoding of the new data, bit for bit."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P8, P16 = 0x11D, 0x1100B


def rs():
    import paper_1312_5155_b200 as m
    return m


def encoded(k, m, w, poly, B, S, seed):
    st = synth.stripes_array(seed, range(S), k, m, B)
    oracle.encode_bulk(st, k, m, w, poly, threads=8)
    return st


CASES = [
    (10, 4, 8, P8, 64 * 1024, [3]),            # JIT body, one changed block
    (10, 4, 8, P8, 3 * 4096 + 40, [9, 0, 4]),  # JIT body + generic tail, unsorted list
    (6, 3, 8, P8, 8192 + 17, [5, 1]),
    (12, 4, 16, P16, 2 * 8192 + 6, [11, 2]),   # w16
    (5, 2, 8, P8, 5000, [0, 1, 2, 3, 4]),      # every data block changes
    (10, 6, 8, P8, 4096 + 3, [2]),              # m > 4 (two output groups in the generic kernel)
    (1, 1, 8, P8, 100, [0]),                    # RAID-5: parity ^= old ^ new
]


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("k,m,w,poly,B,idx", CASES)
def test_update_batch_matches_reencode(k, m, w, poly, B, idx, jit):
    S = 5
    old = encoded(k, m, w, poly, B, S, seed=31)
    new = old.copy()
    rng = np.random.default_rng(B + k)
    for j in idx:
        new[:, j] = rng.integers(0, 256, (S, B), dtype=np.uint8)
    want = new.copy()
    oracle.encode_bulk(want, k, m, w, poly, threads=8)
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    plan.set_jit(m_.RS_JIT_SYNC if jit else m_.RS_JIT_OFF)
    dev = torch.from_numpy(new).cuda()            # new data + OLD parity
    dev[:, k:] = torch.from_numpy(old[:, k:]).cuda()
    old_blocks = torch.from_numpy(np.ascontiguousarray(old[:, idx])).cuda()
    plan.update_batch(dev, idx, old_blocks)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy(), want)
    st = plan.stats()
    aligned = B % 32 == 0
    if jit and aligned and m <= (8 if w == 8 else 4):
        assert st["jit_launches"] >= 1


def test_update_single_stripe_pointer_api():
    k, m, B = 10, 4, 16384
    old = encoded(k, m, 8, P8, B, 1, seed=32)[0]
    new = old.copy()
    idx = [6, 1]
    rng = np.random.default_rng(5)
    for j in idx:
        new[j] = rng.integers(0, 256, B, dtype=np.uint8)
    want = new[None].copy()
    oracle.encode_bulk(want, k, m, 8, P8)
    m_ = rs()
    plan = m_.Plan(k, m)
    plan.set_jit(m_.RS_JIT_SYNC)
    d_new = [torch.from_numpy(new[j].copy()).cuda() for j in idx]
    d_old = [torch.from_numpy(old[j].copy()).cuda() for j in idx]
    d_par = [torch.from_numpy(old[k + i].copy()).cuda() for i in range(m)]
    plan.update(idx, d_old, d_new, d_par, B)
    torch.cuda.synchronize()
    for i in range(m):
        assert np.array_equal(d_par[i].cpu().numpy(), want[0, k + i])


def test_update_errors_and_noop():
    m_ = rs()
    plan = m_.Plan(10, 4)
    dev = torch.zeros((2, 14, 4096), dtype=torch.uint8, device="cuda")
    old = torch.zeros((2, 1, 4096), dtype=torch.uint8, device="cuda")
    for bad in ([10], [-1], [3, 3]):
        with pytest.raises(m_.RSError) as e:
            plan.update_batch(dev, bad, old if len(bad) == 1 else torch.zeros((2, 2, 4096), dtype=torch.uint8,
                                                                             device="cuda"))
        assert e.value.status == m_.RS_ERR_BAD_ERASURE
    n0 = m_.launch_count()
    plan.update_batch(dev, [], torch.zeros((2, 0, 4096), dtype=torch.uint8, device="cuda"))
    assert m_.launch_count() == n0


def test_prepare_update_compiles_before_the_first_call():
    k, m, B, S = 10, 4, 64 * 1024, 3
    m_ = rs()
    plan = m_.Plan(k, m)                       # background JIT mode
    plan.prepare_update([2, 7])
    st = plan.stats()
    assert st["jit_ready"] >= 1 and st["jit_pending"] == 0
    old = encoded(k, m, 8, P8, B, S, seed=33)
    new = old.copy()
    new[:, [2, 7]] ^= 0x5A
    want = new.copy()
    oracle.encode_bulk(want, k, m, 8, P8, threads=4)
    d = torch.from_numpy(new).cuda()
    d[:, k:] = torch.from_numpy(old[:, k:]).cuda()
    n0 = plan.stats()["jit_launches"]
    plan.update_batch(d, [7, 2], torch.from_numpy(np.ascontiguousarray(old[:, [7, 2]])).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), want)
    assert plan.stats()["jit_launches"] == n0 + 1      # the first call already used the JIT kernel
