"""The seeded input generator (synth/) -- shared by the oracle and product sides."""
import numpy as np

import synth


def test_splitmix64_known_vector():
    # SplitMix64 seeded with 0: first output is 0xE220A8397B1DCDAF (published test vector
    # of the generator; its state is incremented by the golden gamma before mixing).
    assert synth.splitmix64_scalar(0) == 0xE220A8397B1DCDAF
    xs = np.array([0, 1, 2, 0xFFFFFFFFFFFFFFFF, 12345678901234], dtype=np.uint64)
    assert [int(v) for v in synth.splitmix64(xs)] == [synth.splitmix64_scalar(int(x)) for x in xs]


def test_data_block_counter_layout():
    b = synth.data_block(3, 5, 7, 24)
    words = b.view(np.uint64)
    for q in range(3):
        assert int(words[q]) == synth.splitmix64_scalar((3 << 48) | (5 << 32) | (7 << 24) | q)
    # odd lengths take a prefix of the same stream
    assert np.array_equal(synth.data_block(3, 5, 7, 13), b[:13])


def test_erasure_draw_properties():
    for s in range(200):
        e = synth.erasure_draw(0, s, range(14), 4)
        assert len(set(e)) == 4 and e == sorted(e) and all(0 <= x < 14 for x in e)
    # C3: even stripes are data-only
    for s in range(0, 64, 2):
        assert max(synth.erasure_pattern("C3", 0, s)) < 10
    tab = synth.erasure_table("C5", 1, 51)
    assert tab.shape == (51, 4) and (tab >= 0).all()
    # the draw is deterministic and depends on the seed
    assert synth.erasure_table("C5", 1, 51).tolist() == tab.tolist()
    assert synth.erasure_table("C5", 2, 51).tolist() != tab.tolist()


def test_c2_sweep_shape():
    sw = synth.c2_decode_sweep()
    assert len(sw) == 4 * (9 + 20)
    assert all(len(p) in (1, 3) for _, p in sw)
    assert all(max(p) < 6 for _, p in sw if len(p) == 3)
