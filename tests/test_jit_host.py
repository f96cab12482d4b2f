"""The run-time generated (JIT) kernels, checked on the CPU.

rs_poly_jit_source returns the CUDA source the library would compile for an erasure
pattern (or for the encoder of a code without a compiled network).  Here its XOR
network is parsed and evaluated on random columns (as bit-planes) and compared with
the CPU oracle's decode/encode; one source per field is also compiled with nvcc for
sm_100a.  The GPU-side parity of the compiled kernels is in tests/test_gpu_jit.py.
"""
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import oracle

P8, P16 = 0x11D, 0x1100B


@pytest.fixture(scope="module")
def rs():
    import paper_1312_5155_b200 as m
    return m


def parse(src):
    ins = {int(i): int(b) for i, b in re.findall(r"uint8_t \*const bi(\d+) = blkp\(a, s, (\d+)\);", src)}
    outs = {int(i): int(b) for i, b in re.findall(r"uint8_t \*const bo(\d+) = blkp\(a, s, (\d+)\);", src)}
    w = int(re.search(r"const uint64_t off = unit_offset<(\d+), false>\(u, u1, h2\);", src).group(1))
    groups = []
    for body in re.findall(r"^    \{\n(.*?)\n    \}$", src, re.S | re.M):
        loads = [(int(i), int(base)) for i, base in re.findall(r"load_unit<\d+>\(bi(\d+) \+ off, &x\[(\d+)\], h2\);", body)]
        stmts = re.findall(r"^\s+(const uint32_t (t\d+)|y\[(\d+)\]) (\^?=) (.*);$", body, re.M)
        groups.append((loads, stmts))
    stores = [(int(i), int(base)) for i, base in re.findall(r"store_unit<\d+>\(bo(\d+) \+ off, &y\[(\d+)\], h2\);", src)]
    # pass-through inputs: bytes XORed into an output after its transpose back
    pins = {int(i): int(b) for i, b in re.findall(r"uint8_t \*const bp(\d+) = blkp\(a, s, (\d+)\);", src)}
    passes = [(int(base), pins[int(i)]) for base, i in re.findall(r"xor_unit<\d+>\(&y\[(\d+)\], bp(\d+) \+ off, h2\);", src)]
    return w, ins, outs, groups, stores, passes


def evaluate_horner(src, cw_cols):
    """Syndrome-form sources (w = 16): statements run in order on bit-planes -- the Horner
    steps are generated as plain XORs of plane snapshots (S_j <- S_j alpha^J + x spelled out
    as its GF(2) matrix), the output network as XORs -- and the stored outputs are compared
    with the oracle by the caller, so a wrong multiply, order or network fails."""
    ins = {int(i): int(b) for i, b in re.findall(r"uint8_t \*const bi(\d+) = blkp\(a, s, (\d+)\);", src)}
    outs = {int(i): int(b) for i, b in re.findall(r"uint8_t \*const bo(\d+) = blkp\(a, s, (\d+)\);", src)}
    w = int(re.search(r"const uint64_t off = unit_offset<(\d+), false>\(u, u1, h2\);", src).group(1))
    body = src[src.index("const uint64_t off = unit_offset<"):]
    C = cw_cols.shape[1]
    S, x, y, env, res = {}, {}, {}, {}, {}

    def planes(blk):
        return [sum(((int(cw_cols[blk][c]) >> b) & 1) << c for c in range(C)) for b in range(w)]

    def val(tok):
        tok = tok.strip()
        if tok == "0u":
            return 0
        mm = re.fullmatch(r"S\[(\d+)\]", tok)
        return S[int(mm.group(1))] if mm else env[tok]

    out_lines = [ln.strip() for ln in body.splitlines()]
    for line in out_lines:
        if mm := re.fullmatch(r"load_unit<\d+>\(blkp\(a, s, (\d+)\) \+ off, x, h2\);", line):
            x = dict(enumerate(planes(int(mm.group(1)))))
            continue
        if mm := re.fullmatch(r"uint32_t S\[(\d+)\];", line):
            S = {q: 0 for q in range(int(mm.group(1)))}
        elif mm := re.fullmatch(r"load_unit<\d+>\(bi(\d+) \+ off, x, h2\);", line):
            x = dict(enumerate(planes(ins[int(mm.group(1))])))
        elif mm := re.fullmatch(r"for \(int q = 0; q < (\d+); \+\+q\) S\[q\] = x\[q % (\d+)\];", line):
            for q in range(int(mm.group(1))):
                S[q] = x[q % int(mm.group(2))]
        elif mm := re.fullmatch(r"for \(int q = 0; q < (\d+); \+\+q\) S\[q\] = 0u;", line):
            for q in range(int(mm.group(1))):
                S[q] = 0
        elif line.startswith("{ const uint32_t h"):
            for name, q in re.findall(r"(h\d+) = S\[(\d+)\]", line):
                env[name] = S[int(q)]
        elif mm := re.fullmatch(r"S\[(\d+)\] \^= x\[(\d+)\];", line):
            S[int(mm.group(1))] ^= x[int(mm.group(2))]
        elif mm := re.fullmatch(r"S\[(\d+)\] = (.*);", line):
            v = 0
            for tok in mm.group(2).split("^"):
                tok = tok.strip()
                xm = re.fullmatch(r"x\[(\d+)\]", tok)
                v ^= x[int(xm.group(1))] if xm else val(tok)
            S[int(mm.group(1))] = v
        elif mm := re.fullmatch(r"const uint32_t (t\d+) = (.*);", line):
            v = 0
            for tok in mm.group(2).split("^"):
                v ^= val(tok)
            env[mm.group(1)] = v
        elif mm := re.fullmatch(r"y\[(\d+)\] = (.*);", line):
            v = 0
            for tok in mm.group(2).split("^"):
                v ^= val(tok)
            y[int(mm.group(1))] = v
        elif mm := re.fullmatch(r"store_unit<\d+>\(bo(\d+) \+ off, &y\[(\d+)\], h2\);", line):
            i, base = int(mm.group(1)), int(mm.group(2))
            res[outs[i]] = [sum(((y[base + o] >> c) & 1) << o for o in range(w)) for c in range(C)]
    return res


def evaluate(src, cw_cols):
    """cw_cols: [n][C] symbols (API order).  Returns {out_block: [C] symbols}."""
    if "uint32_t S[" in src:
        return evaluate_horner(src, cw_cols)
    w, ins, outs, groups, stores, passes = parse(src)
    C = cw_cols.shape[1]
    nout = len(outs)
    # y starts undefined unless the source zeroes it: a read of an unset plane fails
    zero = re.search(r"for \(int q = 0; q < \d+; \+\+q\) y\[q\] = 0u;", src) is not None
    y = [0 if zero else None] * (nout * w)
    for loads, stmts in groups:
        x = {}
        for i, base in loads:
            blk = ins[i]
            for b in range(w):
                x[base + b] = sum(((int(cw_cols[blk][c]) >> b) & 1) << c for c in range(C))
        env = {}

        def val(tok):
            tok = tok.strip()
            if tok.startswith("x["):
                return x[int(tok[2:-1])]
            if tok == "0u":
                return 0
            return env[tok]

        for _, tname, yidx, op, expr in stmts:
            v = 0
            for tok in expr.split("^"):
                v ^= val(tok)
            if tname:
                env[tname] = v
            elif op == "=":
                y[int(yidx)] = v
            else:
                assert y[int(yidx)] is not None, "accumulating into an unset output plane"
                y[int(yidx)] ^= v
    res = {}
    for i, base in stores:
        assert all(y[base + o] is not None for o in range(w)), "storing an unset output plane"
        res[outs[i]] = [sum(((y[base + o] >> c) & 1) << o for o in range(w)) for c in range(C)]
        for pbase, blk in passes:
            if pbase == base:
                res[outs[i]] = [v ^ int(cw_cols[blk][c]) for c, v in enumerate(res[outs[i]])]
    return res


def codewords(k, m, w, poly, C, seed):
    rng = np.random.default_rng(seed)
    cols = np.zeros((k + m, C), dtype=np.int64)
    for c in range(C):
        d = [int(v) for v in rng.integers(0, 1 << w, k)]
        cols[:, c] = d + oracle.encode_column(d, m, w, poly)
    return cols


@pytest.mark.parametrize("policy", [0, 1])
@pytest.mark.parametrize("k,m,w,poly", [(10, 4, 8, P8), (6, 3, 8, P8), (12, 4, 16, P16), (5, 2, 8, P8),
                                        (10, 6, 8, P8), (20, 8, 8, P8)])
def test_jit_decode_networks_match_oracle(rs, k, m, w, poly, policy):
    """policy 0: every survivor read (the paper's Step 1); 1: only k survivors read (NEXT-2)."""
    plan = rs.Plan(k, m, w, poly)
    plan.set_read_policy(policy)
    n = k + m
    rng = np.random.default_rng(k * 31 + m)
    cols = codewords(k, m, w, poly, 32, seed=k + m)
    pats = [list(range(m)), list(range(k, n)), [0, n - 1][: min(2, m)], [k - 1]]
    for _ in range(6):
        t = int(rng.integers(1, m + 1))
        pats.append(sorted(rng.choice(n, t, replace=False).tolist()))
    for er in pats:
        src = plan.jit_source(er)
        eligible = len(er) <= (8 if w == 8 else 4)
        assert bool(src) == eligible
        if not src:
            continue
        got = evaluate(src, cols)
        assert sorted(got) == sorted(er)
        for b in er:
            assert got[b] == [int(v) for v in cols[b]], (er, b)
        reads = set(re.findall(r"blkp\(a, s, (\d+)\)", src)) - {str(b) for b in er}
        assert len(reads) == (k if policy == 1 else k + m - len(er)), (er, sorted(reads))


@pytest.mark.parametrize("k,m,w,poly", [(5, 2, 8, P8), (10, 6, 8, P8), (10, 4, 16, P16), (3, 1, 8, P8)])
def test_jit_encoder_matches_oracle(rs, k, m, w, poly):
    plan = rs.Plan(k, m, w, poly)
    src = plan.jit_source([])
    assert src
    cols = codewords(k, m, w, poly, 32, seed=5)
    got = evaluate(src, cols)
    for i in range(m):
        assert got[k + i] == [int(v) for v in cols[k + i]]


def test_jit_not_eligible_when_too_many_outputs(rs):
    assert rs.Plan(10, 6, 16, P16).jit_source([0, 1, 2, 3, 4]) == ""   # w16: at most 4 outputs
    assert rs.Plan(20, 9, 8, P8).jit_source([]) == ""                  # w8: at most 8 outputs
    assert rs.Plan(10, 4).jit_source([0, 0]) == ""                      # invalid list


@pytest.mark.parametrize("k,m,w,poly,er", [(10, 4, 8, P8, [1, 4, 10, 13]), (12, 4, 16, P16, [0, 5, 12, 15])])
def test_jit_source_compiles_for_sm100a(rs, k, m, w, poly, er):
    src = rs.Plan(k, m, w, poly).jit_source(er)
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "jit.cu")
        open(f, "w").write(src)
        out = subprocess.run(["/usr/local/cuda/bin/nvcc", "-cubin", "-gencode", "arch=compute_100a,code=sm_100a",
                              "-std=c++17", "-Xptxas", "-v", "-o", os.path.join(d, "jit.cubin"), f],
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-3000:]
        assert "spill stores" in out.stderr


@pytest.mark.parametrize("k,m,w,poly,idx", [(10, 4, 8, P8, [3]), (10, 4, 8, P8, [7, 0, 9]), (6, 3, 8, P8, [5, 1]),
                                            (12, 4, 16, P16, [11, 2]), (5, 2, 8, P8, list(range(5)))])
def test_jit_update_network_matches_oracle(rs, k, m, w, poly, idx):
    """Diff-update: the generated network applied to (new, old, old parity) gives
    the oracle's encoding of the new data."""
    plan = rs.Plan(k, m, w, poly)
    src = plan.update_jit_source(idx)
    assert src
    C = 32
    rng = np.random.default_rng(len(idx) + k)
    old = rng.integers(0, 1 << w, (k, C))
    new = old.copy()
    for j in idx:
        new[j] = rng.integers(0, 1 << w, C)
    old_par = np.array([oracle.encode_column([int(v) for v in old[:, c]], m, w, poly) for c in range(C)]).T
    new_par = np.array([oracle.encode_column([int(v) for v in new[:, c]], m, w, poly) for c in range(C)]).T
    order = sorted(idx)
    virt = []                      # [new_0, old_0, new_1, old_1, ..., parity]
    for j in order:
        virt += [new[j], old[j]]
    virt += list(old_par)
    got = evaluate(src, np.array(virt, dtype=np.int64))
    for i in range(m):
        assert got[2 * len(order) + i] == [int(v) for v in new_par[i]]
