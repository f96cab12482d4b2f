"""GPU verify (scrub): a stripe is flagged iff some column is not a codeword (some syndrome
at the roots of g is non-zero).  Codewords come from the oracle; corruptions are
single flipped bits anywhere (data or parity, body or ragged tail)."""
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


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("k,m,w,poly,B", [(10, 4, 8, P8, 64 * 1024 + 40), (12, 4, 16, P16, 16 * 1024 + 6),
                                          (6, 3, 8, P8, 4096), (1, 1, 8, P8, 777), (5, 2, 8, P8, 3000),
                                          (10, 6, 16, P16, 2048)])
def test_verify_flags_exactly_the_corrupted_stripes(k, m, w, poly, B, jit):
    S = 12
    ref = synth.stripes_array(90, range(S), k, m, B)
    oracle.encode_bulk(ref, k, m, w, poly, threads=4)
    # the oracle itself agrees these are codewords (root property, sampled columns)
    for c in range(0, B // (w // 8), max(1, B // 7)):
        col = [int.from_bytes(bytes(ref[0, b, c * (w // 8):(c + 1) * (w // 8)]), "little") for b in range(k + m)]
        for j in range(m):
            assert oracle.eval_codeword(col, k, m, oracle.gf_pow(2, j, w, poly), w, poly) == 0
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    plan.set_jit(m_.RS_JIT_SYNC if jit else m_.RS_JIT_OFF)
    d = torch.from_numpy(ref).cuda()
    flags = torch.full((S,), 7, dtype=torch.int32, device="cuda")
    plan.verify_batch(d, flags)
    torch.cuda.synchronize()
    assert flags.cpu().tolist() == [0] * S
    rng = np.random.default_rng(k + 31 * m)
    bad = sorted(rng.choice(S, 5, replace=False).tolist())
    bad_np = ref.copy()
    for s in bad:
        b = int(rng.integers(k + m))
        x = int(rng.integers(B)) if s % 2 else B - 1 - int(rng.integers(min(B, 40)))  # odd: anywhere; even: tail
        bad_np[s, b, x] ^= np.uint8(1 << int(rng.integers(8)))
    d = torch.from_numpy(bad_np).cuda()
    plan.verify_batch(d, flags)
    torch.cuda.synchronize()
    assert [i for i, f in enumerate(flags.cpu().tolist()) if f] == bad
    assert torch.equal(d.cpu(), torch.from_numpy(bad_np))   # verify writes nothing to the stripes
