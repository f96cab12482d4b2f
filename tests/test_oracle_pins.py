"""Pins for the CPU oracle (oracle/rs_oracle.c) against what the paper and the mathematics fix.

Each test names the plausible oracle mistake it would catch.  Nothing here uses
the CUDA library; expected values are the paper's (tests/golden/paper_example.json,
cited) or follow from closed forms, invariants, brute force, or an independent
multiply (tests/gfref.py).
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from tests import gfref

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_example.json")))
P8 = 0x11D
P16 = 0x1100B


# --------------------------------------------------------------------------
# Worked example of the paper -- strongest pins.
# --------------------------------------------------------------------------
def test_paper_alpha_powers():
    """P:255-278 print alpha^3..alpha^5 = 8,16,32, alpha^6=64, alpha^8=29, alpha^10=116.
    alpha^8 = 29 forces prim_poly 0x11D (reading G1); a wrong poly fails here."""
    V = GOLD["decode"]["V"]
    E = GOLD["decode"]["V_as_alpha_exponents"]
    for row_v, row_e in zip(V, E):
        for v, e in zip(row_v, row_e):
            assert oracle.gf_pow(2, e) == v


def test_paper_generator_polynomial():
    """g(x) = x^3 + 7x^2 + 14x + 8 for m=3 (catches a wrong root set or product order)."""
    assert oracle.gen_poly(3) == GOLD["gen_poly_k4_m3"]["coeffs_low_to_high"]


def test_paper_encode_example():
    """48,6,112,70 -> 243,125,142 (Eq. 1-2)."""
    e = GOLD["encode"]
    assert oracle.encode_column(e["data"], e["m"]) == e["parity"]


def test_paper_encode_data_order_is_pinned():
    """Reading G3: d_0 is the coefficient of x^m.  The reversed order must NOT give the paper's parity."""
    e = GOLD["encode"]
    assert oracle.encode_column(e["data"][::-1], e["m"]) != e["parity"]


def test_paper_decode_example():
    """erase d0..d2 of (48,6,112,70 | 243,125,142); Step 1 gives D = 70,91,171,
    Step 2's matrix is [[1,1,1],[8,16,32],[64,29,116]], the solution is 48,6,112."""
    d = GOLD["decode"]
    enc = GOLD["encode"]
    cw = list(d["received_data"]) + list(enc["parity"])  # API order: data then parity
    fixed, syn = oracle.decode_column(cw, 4, 3, d["erased_api_indices"], want_syndromes=True)
    assert syn == d["D_values"]
    assert fixed[:3] == d["recovered"]
    assert fixed == list(enc["data"]) + list(enc["parity"])
    V = oracle.decode_matrix(4, 3, d["erased_api_indices"])
    assert V.tolist() == d["V"]


# --------------------------------------------------------------------------
# Field GF(2^w)
# --------------------------------------------------------------------------
def _oracle_mul_table_w8():
    L = oracle.lib()
    return np.array([[L.orc_gf_mul(a, b, 8, P8) for b in range(256)] for a in range(256)], dtype=np.int64)


@pytest.fixture(scope="module")
def mul8():
    return _oracle_mul_table_w8()


def test_field_w8_multiply_matches_independent_definition(mul8):
    """All 65536 pairs vs carry-less product + polynomial reduction (tests/gfref.py)."""
    a, b = np.meshgrid(np.arange(256), np.arange(256), indexing="ij")
    ref = gfref.mul_np(a.ravel(), b.ravel(), 8, P8).reshape(256, 256)
    assert np.array_equal(mul8, ref)


def test_field_w8_axioms_exhaustive(mul8):
    """Commutativity, identity, zero, inverses on all elements; associativity and
    distributivity over all 2^24 triples."""
    M = mul8
    assert np.array_equal(M, M.T)
    assert np.array_equal(M[1], np.arange(256)) and not M[0].any()
    for a in range(1, 256):
        assert M[a, oracle.gf_inv(a)] == 1
    idx = np.arange(256)
    for a in range(256):
        ab = M[a][:, None]                     # (a*b) for all b
        lhs = M[ab, idx[None, :]]              # (a*b)*c
        rhs = M[a][M]                          # a*(b*c)
        assert np.array_equal(lhs, rhs)
        dist_l = M[a][idx[:, None] ^ idx[None, :]]       # a*(b+c)
        dist_r = M[a][:, None] ^ M[a][None, :]           # a*b + a*c
        assert np.array_equal(dist_l, dist_r)


def test_field_known_inverse_and_order():
    """2 * 142 = 1 under 0x11D (2*142 = 0x11C, reduced by 0x11D); ord(2) = 255 / 65535."""
    assert oracle.gf_mul(2, 142) == 1 and oracle.gf_inv(2) == 142
    assert oracle.gf_mul(2, 128) == 29          # alpha^8
    assert oracle.order_of_alpha(8, P8) == 255
    assert oracle.order_of_alpha(16, P16) == 65535
    # 0x11B (AES) is irreducible but 2 is not a generator: order 51 -> must be rejected
    assert oracle.order_of_alpha(8, 0x11B) == 51


def test_field_w16_multiply_sampled():
    rng = np.random.default_rng(1)
    a = rng.integers(0, 1 << 16, 4096)
    b = rng.integers(0, 1 << 16, 4096)
    L = oracle.lib()
    got = np.array([L.orc_gf_mul(int(x), int(y), 16, P16) for x, y in zip(a, b)])
    assert np.array_equal(got, gfref.mul_np(a, b, 16, P16))


def test_field_w16_axioms_sampled():
    rng = np.random.default_rng(2)
    T = gfref.Tables(16, P16)
    a, b, c = (rng.integers(0, 1 << 16, 200000) for _ in range(3))
    assert np.array_equal(T.mul(T.mul(a, b), c), T.mul(a, T.mul(b, c)))
    assert np.array_equal(T.mul(a, b ^ c), T.mul(a, b) ^ T.mul(a, c))
    for x in rng.integers(1, 1 << 16, 64):
        assert oracle.gf_mul(int(x), oracle.gf_inv(int(x), 16, P16), 16, P16) == 1


@pytest.mark.parametrize("w,poly", [(8, P8), (16, P16)])
def test_bulk_tables_match_shift_and_add(w, poly):
    """The bulk mode's log/exp multiply equals orc_gf_mul (all pairs for w=8, sampled for w=16)."""
    if w == 8:
        a, b = np.meshgrid(np.arange(256), np.arange(256), indexing="ij")
        a, b = a.ravel(), b.ravel()
    else:
        rng = np.random.default_rng(3)
        a = rng.integers(0, 1 << 16, 1 << 18)
        b = rng.integers(0, 1 << 16, 1 << 18)
        a[:256] = 0
        b[256:512] = 0
    got = oracle.bulk_table_mul(a, b, w, poly)
    assert np.array_equal(got, gfref.mul_np(a, b, w, poly))


# --------------------------------------------------------------------------
# Generator polynomial
# --------------------------------------------------------------------------
@pytest.mark.parametrize("w,poly", [(8, P8), (16, P16)])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 5, 6, 8])
def test_gen_poly_roots(w, poly, m):
    """g is monic of degree m with roots exactly alpha^0..alpha^{m-1} (g(alpha^m) != 0)."""
    g = oracle.gen_poly(m, w, poly)
    T = gfref.Tables(w, poly)
    assert len(g) == m + 1 and g[-1] == 1

    def ev(x):
        acc = 0
        for c in reversed(g):
            acc = int(T.mul(acc, x)) ^ c
        return acc

    for i in range(m):
        assert ev(T.pow_alpha(i)) == 0
    assert ev(T.pow_alpha(m)) != 0


# --------------------------------------------------------------------------
# Encode
# --------------------------------------------------------------------------
CODES = [(4, 3, 8, P8), (6, 3, 8, P8), (10, 4, 8, P8), (10, 2, 8, P8), (10, 6, 8, P8),
         (12, 4, 16, P16), (4, 3, 16, P16), (1, 1, 8, P8), (20, 8, 8, P8)]


def _rand_data(rng, k, w):
    return [int(x) for x in rng.integers(0, 1 << w, k)]


@pytest.mark.parametrize("k,m,w,poly", CODES)
def test_encode_root_property_and_systematic(k, m, w, poly):
    """Every codeword vanishes at alpha^0..alpha^{m-1}, evaluated with the
    independent multiply; data positions are the input (systematic)."""
    rng = np.random.default_rng(k * 100 + m + w)
    T = gfref.Tables(w, poly)
    for _ in range(20):
        d = _rand_data(rng, k, w)
        p = oracle.encode_column(d, m, w, poly)
        cw = d + p
        byp = gfref.by_position(cw, k, m)[:, None]
        for j in range(m):
            assert int(T.eval_positions(byp, T.pow_alpha(j))[0]) == 0
        assert cw[:k] == d


def test_encode_example_codeword_not_a_multiple_beyond_m():
    """The example codeword is a multiple of g only: c(alpha^3) != 0 (a wrong, larger g would zero it)."""
    e = GOLD["encode"]
    T = gfref.Tables(8, P8)
    byp = gfref.by_position(e["data"] + e["parity"], 4, 3)[:, None]
    assert int(T.eval_positions(byp, T.pow_alpha(3))[0]) != 0


@pytest.mark.parametrize("k,w,poly", [(1, 8, P8), (6, 8, P8), (10, 8, P8), (12, 16, P16)])
def test_encode_m1_is_raid5_xor(k, w, poly):
    """m=1: g = x+1, so the single parity is the XOR of the data (textbook RAID-5)."""
    rng = np.random.default_rng(5)
    for _ in range(50):
        d = _rand_data(rng, k, w)
        x = 0
        for v in d:
            x ^= v
        assert oracle.encode_column(d, 1, w, poly) == [x]


@pytest.mark.parametrize("k,m,w,poly", CODES)
def test_encode_linearity_diff_update(k, m, w, poly):
    """encoding data diff-blocks gives the parity diff-blocks (linearity over GF(2))."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        a, b = _rand_data(rng, k, w), _rand_data(rng, k, w)
        pa, pb = oracle.encode_column(a, m, w, poly), oracle.encode_column(b, m, w, poly)
        pab = oracle.encode_column([x ^ y for x, y in zip(a, b)], m, w, poly)
        assert pab == [x ^ y for x, y in zip(pa, pb)]


@pytest.mark.parametrize("k,m,w,poly", CODES)
def test_encode_equals_decode_with_parity_erased(k, m, w, poly):
    """P:306 symmetry: decoding with all m parity erased reproduces the encoder's parity."""
    rng = np.random.default_rng(11)
    for _ in range(10):
        d = _rand_data(rng, k, w)
        p = oracle.encode_column(d, m, w, poly)
        fixed = oracle.decode_column(d + [0] * m, k, m, list(range(k, k + m)), w, poly)
        assert fixed[k:] == p


@pytest.mark.parametrize("k,m,w,poly", [(10, 4, 8, P8), (6, 3, 8, P8), (12, 4, 16, P16)])
def test_parity_map_closed_forms(k, m, w, poly):
    """Parity map P[:, j] = encode(unit vector e_j).  Closed forms (x^{m+j} mod g):
    column 0 = (g_0..g_{m-1}) because x^m = g - (g - x^m); column j+1 = x * column j mod g."""
    g = oracle.gen_poly(m, w, poly)
    T = gfref.Tables(w, poly)
    cols = [oracle.encode_column([1 if i == j else 0 for i in range(k)], m, w, poly) for j in range(k)]
    assert cols[0] == g[:m]
    for j in range(k - 1):
        c = cols[j]
        top = c[m - 1]                       # coefficient that overflows into x^m
        shifted = [0] + c[: m - 1]           # x * c(x) without the x^m term
        nxt = [s ^ int(T.mul(top, g[i])) for i, s in enumerate(shifted)]
        assert cols[j + 1] == nxt


# --------------------------------------------------------------------------
# Decode
# --------------------------------------------------------------------------
def _codeword(rng, k, m, w, poly):
    d = _rand_data(rng, k, w)
    return d + oracle.encode_column(d, m, w, poly)


@pytest.mark.parametrize("k,m,w,poly", CODES)
def test_decode_single_erasure_is_xor_of_survivors(k, m, w, poly):
    """t=1: row j=0 of the system has alpha^0 = 1 everywhere, so the erased
    symbol is the XOR of the n-1 survivors (for every position, data or parity)."""
    rng = np.random.default_rng(13)
    n = k + m
    cw = _codeword(rng, k, m, w, poly)
    for e in range(n):
        bad = list(cw)
        bad[e] = 0x5A
        x = 0
        for b in range(n):
            if b != e:
                x ^= cw[b]
        assert oracle.decode_column(bad, k, m, [e], w, poly)[e] == x == cw[e]


@pytest.mark.parametrize("erased", [[0, 1], [0, 5], [2, 6], [5, 6], [3], [4]])
def test_decode_brute_force_small(erased):
    """RS(4,3) w=8: among all 256^t fillings of the erased slots exactly one makes
    the word vanish at alpha^0..alpha^2, and it is what the oracle returns."""
    k, m = 4, 3
    T = gfref.Tables(8, P8)
    rng = np.random.default_rng(17)
    cw = _codeword(rng, k, m, 8, P8)
    t = len(erased)
    cands = np.array(list(itertools.product(range(256), repeat=t)), dtype=np.int64)  # [256^t][t]
    words = np.tile(np.array(cw, dtype=np.int64), (cands.shape[0], 1))
    words[:, erased] = cands
    byp = np.zeros_like(words.T)
    for b, p in enumerate(gfref.positions(k, m)):
        byp[p] = words[:, b]
    ok = np.ones(cands.shape[0], dtype=bool)
    for j in range(m):
        ok &= T.eval_positions(byp, T.pow_alpha(j)) == 0
    sols = cands[ok]
    assert sols.shape[0] == 1
    got = oracle.decode_column([0 if b in erased else v for b, v in enumerate(cw)], k, m, erased)
    assert [got[e] for e in erased] == sols[0].tolist() == [cw[e] for e in erased]


def test_decode_brute_force_w16_t1():
    """RS(12,4) w=16: all 65536 candidates for one erased symbol; exactly one satisfies the roots."""
    k, m = 12, 4
    T = gfref.Tables(16, P16)
    rng = np.random.default_rng(19)
    cw = _codeword(rng, k, m, 16, P16)
    for e in (0, 7, 12, 15):
        cand = np.arange(1 << 16, dtype=np.int64)
        words = np.tile(np.array(cw, dtype=np.int64), (cand.size, 1))
        words[:, e] = cand
        byp = np.zeros_like(words.T)
        for b, p in enumerate(gfref.positions(k, m)):
            byp[p] = words[:, b]
        ok = np.ones(cand.size, dtype=bool)
        for j in range(m):
            ok &= T.eval_positions(byp, T.pow_alpha(j)) == 0
        assert ok.sum() == 1 and int(cand[ok][0]) == cw[e]
        assert oracle.decode_column([0 if b == e else v for b, v in enumerate(cw)], k, m, [e], 16, P16)[e] == cw[e]


@pytest.mark.parametrize("k,m,w,poly", CODES)
def test_decode_forney_equals_vandermonde(k, m, w, poly):
    """Forney's closed form (independent of Gauss-Jordan) agrees on random mixed patterns."""
    rng = np.random.default_rng(23)
    n = k + m
    for _ in range(60):
        cw = _codeword(rng, k, m, w, poly)
        t = int(rng.integers(1, m + 1))
        er = sorted(rng.choice(n, t, replace=False).tolist())
        bad = [0 if b in er else v for b, v in enumerate(cw)]
        a = oracle.decode_column(bad, k, m, er, w, poly)
        b = oracle.decode_column_forney(bad, k, m, er, w, poly)
        assert a == b == cw


@pytest.mark.parametrize("k,m,w,poly", [(4, 3, 8, P8), (6, 3, 8, P8), (10, 4, 8, P8), (12, 4, 16, P16)])
def test_decode_every_pattern_exhaustive(k, m, w, poly):
    """MDS: every erasure pattern of size <= m (1471 for (10,4), 2517 for (12,4)) recovers
    the codeword, with erased slots holding garbage and the list in any order."""
    rng = np.random.default_rng(29)
    n = k + m
    cw = _codeword(rng, k, m, w, poly)
    count = 0
    for t in range(0, m + 1):
        for er in itertools.combinations(range(n), t):
            bad = list(cw)
            for e in er:
                bad[e] = int(rng.integers(0, 1 << w))
            assert oracle.decode_column(bad, k, m, list(er)[::-1], w, poly) == cw
            count += 1
    assert count == sum(len(list(itertools.combinations(range(n), t))) for t in range(m + 1))


def test_decode_rejects_bad_erasure_lists():
    cw = [0] * 7
    with pytest.raises(ValueError):
        oracle.decode_column(cw, 4, 3, [0, 1, 2, 3])      # more than m
    with pytest.raises(ValueError):
        oracle.decode_column(cw, 4, 3, [1, 1])            # duplicate
    with pytest.raises(ValueError):
        oracle.decode_column(cw, 4, 3, [7])               # out of range


# --------------------------------------------------------------------------
# Bulk mode == column mode
# --------------------------------------------------------------------------
@pytest.mark.parametrize("k,m,w,poly,B", [(10, 4, 8, P8, 257), (6, 3, 8, P8, 64), (12, 4, 16, P16, 130)])
def test_bulk_matches_column_mode(k, m, w, poly, B):
    rng = np.random.default_rng(31)
    S, n = 5, k + m
    st = rng.integers(0, 256, (S, n, B), dtype=np.uint8)
    oracle.encode_bulk(st, k, m, w, poly, threads=3)
    sym = 1 if w == 8 else 2
    cols = B // sym
    def column(s, c):
        if w == 8:
            return [int(st[s, b, c]) for b in range(n)]
        return [int(st[s, b, 2 * c]) | (int(st[s, b, 2 * c + 1]) << 8) for b in range(n)]
    for s in range(S):
        for c in range(0, cols, max(1, cols // 17)):
            cw = column(s, c)
            assert cw[k:] == oracle.encode_column(cw[:k], m, w, poly)
    good = st.copy()
    er = np.full((S, m), -1, dtype=np.int32)
    for s in range(S):
        t = int(rng.integers(0, m + 1))
        e = rng.choice(n, t, replace=False)
        er[s, :t] = e
        st[s, e] = rng.integers(0, 256, (t, B), dtype=np.uint8)
    oracle.decode_bulk(st, er, k, m, w, poly, threads=2)
    assert np.array_equal(st, good)
