"""GPU parity of the paper's optimisation study (NEXT-3): every Opt1/Opt2/Opt3
combination of the per-column table decode gives the oracle's bytes, for decoding and for
encoding through the decoder."""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P8 = 0x11D


def rs():
    import paper_1312_5155_b200 as m
    return m


@pytest.mark.parametrize("opt", range(8))
@pytest.mark.parametrize("k,m,er", [(10, 4, [0, 5, 11, 13]), (10, 4, [3]), (6, 3, [1, 2, 4]), (4, 3, [0, 1, 2]),
                                    (10, 6, [0, 2, 4, 9, 10, 15])])
def test_ablation_decode_matches_oracle(k, m, er, opt):
    S, B = 3, 4096 + 13
    ref = synth.stripes_array(40, range(S), k, m, B)
    oracle.encode_bulk(ref, k, m, 8, P8, threads=4)
    bad = ref.copy()
    bad[:, er] = 0x5A
    m_ = rs()
    plan = m_.Plan(k, m)
    d = torch.from_numpy(bad).cuda()
    plan.ablation_decode(d, er, opt)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)


@pytest.mark.parametrize("opt", [0, 7])
def test_ablation_encode_via_decode(opt):
    """Encoding = decoding the m parity positions (the symmetric use)."""
    k, m, S, B = 10, 2, 2, 8192
    ref = synth.stripes_array(41, range(S), k, m, B)
    oracle.encode_bulk(ref, k, m, 8, P8, threads=4)
    m_ = rs()
    plan = m_.Plan(k, m)
    d = torch.from_numpy(ref).cuda()
    d[:, k:] = 0
    plan.ablation_decode(d, list(range(k, k + m)), opt)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)


def test_ablation_limits():
    m_ = rs()
    d = torch.zeros((1, 14, 256), dtype=torch.uint8, device="cuda")
    with pytest.raises(m_.RSError):
        m_.Plan(10, 4, 16).ablation_decode(torch.zeros((1, 14, 256), dtype=torch.uint8, device="cuda"), [0], 7)
    with pytest.raises(m_.RSError):
        m_.Plan(10, 4).ablation_decode(d, [], 7)
    with pytest.raises(m_.RSError):
        m_.Plan(10, 4).ablation_decode(d, [0], 8)
