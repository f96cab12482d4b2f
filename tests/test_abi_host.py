"""Host-side checks of the product library (no GPU needed).

* the C-ABI library loads and exports every function include/*.h declares;
* argument validation returns the documented rs_status before any device work;
* the planner's g(x) and parity map equal the oracle's (different methods:
  shift-register recurrence in C++ vs literal long division in the oracle);
* the generated bit-sliced networks (csrc/rs_networks.cuh), evaluated here on
  random bit-planes, reproduce the oracle's parity for every column.
"""
import ctypes
import glob
import os
import re
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1312_5155_b200")
sys.path.insert(0, os.path.join(PKG, "csrc"))


@pytest.fixture(scope="module")
def rs():
    import paper_1312_5155_b200 as m
    return m


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(rs_\w+)\s*\(", src):
            names.add((os.path.basename(h), m.group(1)))
    return sorted(names)


def test_every_declared_symbol_is_exported(rs):
    libs = {"rs_poly.h": ctypes.CDLL(rs.LIB_PATH), "rs_synth.h": ctypes.CDLL(rs.SYNTH_PATH)}
    decl = declared_functions()
    assert len(decl) == 28  # 27 in rs_poly.h + rs_synth_fill
    for header, name in decl:
        assert hasattr(libs[header], name), f"{name} declared in {header} but not exported"


def test_abi_version_and_strerror(rs):
    assert rs.abi_version() == 2
    for s in range(8):
        assert rs.strerror(s)
    assert "unknown" in rs.strerror(99)


@pytest.mark.parametrize("k,m,w,poly,status", [
    (0, 4, 8, 0x11D, 1), (10, 0, 8, 0x11D, 1), (10, 33, 8, 0x11D, 1), (10, 4, 12, 0x11D, 1),
    (250, 6, 8, 0x11D, 1),            # n = 256 > 2^8 - 1 (reading G7)
    (10, 4, 16, 0x11D, 2),            # not of degree 16
    (10, 4, 8, 0x11B, 2),             # irreducible but alpha = 2 has order 51
    (10, 4, 8, 0x1FF, 2),             # not primitive
])
def test_plan_create_validation(rs, k, m, w, poly, status):
    with pytest.raises(rs.RSError) as e:
        rs.Plan(k, m, w, poly)
    assert e.value.status == status


@pytest.mark.parametrize("k,m,w,poly", [(4, 3, 8, 0x11D), (10, 4, 8, 0x11D), (6, 3, 8, 0x11D), (12, 4, 16, 0x1100B),
                                        (17, 5, 8, 0x11D), (1, 1, 8, 0x11D), (200, 32, 8, 0x11D), (30, 9, 16, 0x1100B)])
def test_plan_info_matches_oracle(rs, k, m, w, poly):
    g, P = rs.Plan(k, m, w, poly).info()
    assert g.tolist() == oracle.gen_poly(m, w, poly)
    for j in range(k):
        unit = [1 if i == j else 0 for i in range(k)]
        assert P[:, j].tolist() == oracle.encode_column(unit, m, w, poly)


def test_kernel_kind(rs):
    import gen_networks
    for (k, m, w, poly, _) in gen_networks.INSTANCES:
        assert rs.Plan(k, m, w, poly).kernel_kind == "bitsliced"
    assert rs.Plan(5, 2).kernel_kind == "generic"
    assert rs.Plan(10, 6).kernel_kind == "generic"


def test_validation_before_device_work(rs):
    """These calls must fail in validation (no CUDA device exists here)."""
    plan = rs.Plan(10, 4)
    fake = [0x10000 + 4096 * i for i in range(14)]
    with pytest.raises(rs.RSError) as e:
        plan.decode(fake, 4096, [0, 1, 2, 3, 4], stream=0)
    assert e.value.status == rs.RS_ERR_TOO_MANY_ERASURES
    with pytest.raises(rs.RSError) as e:
        plan.decode(fake, 4096, [3, 3], stream=0)
    assert e.value.status == rs.RS_ERR_BAD_ERASURE
    with pytest.raises(rs.RSError) as e:
        plan.decode(fake, 4096, [14], stream=0)
    assert e.value.status == rs.RS_ERR_BAD_ERASURE
    with pytest.raises(rs.RSError) as e:
        plan.encode(fake[:10], fake[10:], 0, stream=0)
    assert e.value.status == rs.RS_ERR_GEOMETRY
    p16 = rs.Plan(12, 4, 16)
    with pytest.raises(rs.RSError) as e:
        p16.encode([0x10000 + 4096 * i for i in range(12)], [0x90000 + 4096 * i for i in range(4)], 4095, stream=0)
    assert e.value.status == rs.RS_ERR_GEOMETRY
    with pytest.raises(rs.RSError) as e:       # misaligned symbol pointer for w=16
        p16.encode([0x10001] + [0x10000 + 4096 * i for i in range(1, 12)], [0x90000 + 4096 * i for i in range(4)],
                   4096, stream=0)
    assert e.value.status == rs.RS_ERR_GEOMETRY
    # batch: overlapping blocks, bad rows
    lib = rs.rs_poly._lib
    er = np.array([[0, 1, 2, 14]], dtype=np.int32)
    assert lib.rs_poly_decode_batch(plan._h, 0x10000, 1, 14 * 4096, 4096, 4096, er.ctypes.data, 0) == 5
    assert lib.rs_poly_encode_batch(plan._h, 0x10000, 2, 4096, 4096, 4096, 0) == rs.RS_ERR_GEOMETRY
    assert lib.rs_poly_encode_batch(None, 0x10000, 1, 4096, 4096, 4096, 0) == rs.RS_ERR_INVALID_ARG
    # empty work is a successful no-op without touching the device
    assert lib.rs_poly_encode_batch(plan._h, 0x10000, 0, 14 * 4096, 4096, 4096, 0) == 0
    plan.decode(fake, 4096, [], stream=0)


# --------------------------------------------------------------------------
# generated networks, evaluated on the CPU
# --------------------------------------------------------------------------
def parse_network(k, m, w, poly):
    src = open(os.path.join(PKG, "csrc", "rs_networks.cuh")).read()
    groups = []
    pat = re.compile(r"template <> struct RsNetGroup<%d, %d, %d, 0x%Xu, (\d+)> \{(.*?)\n\};" % (k, m, w, poly), re.S)
    for mt in pat.finditer(src):
        body = mt.group(2)
        first = int(re.search(r"kFirstBlock = (\d+)", body).group(1))
        nb = int(re.search(r"kBlocks = (\d+)", body).group(1))
        stmts = re.findall(r"^\s+(const uint32_t (t\d+)|y\[(\d+)\]) (\^?=) (.*);$", body, re.M)
        groups.append((first, nb, stmts))
    assert groups, "instance not found"
    return groups


def eval_network(groups, data_planes, m, w):
    """data_planes: [k*w] uint32 arrays; returns [m*w] parity planes."""
    y = [None] * (m * w)
    for first, nb, stmts in groups:
        x = data_planes[first * w:(first + nb) * w]
        env = {}

        def val(tok):
            tok = tok.strip()
            if tok.startswith("x["):
                return x[int(tok[2:-1])]
            if tok == "0u":
                return np.zeros_like(data_planes[0])
            return env[tok]

        for _, tname, yidx, op, expr in stmts:
            v = np.zeros_like(data_planes[0])
            for tok in expr.split("^"):
                v = v ^ val(tok)
            if tname:
                env[tname] = v
            elif op == "=":
                y[int(yidx)] = v
            else:
                y[int(yidx)] = y[int(yidx)] ^ v
    return y


def horner_parity(k, m, w, poly, data):
    """Syndrome-form instances (RsQNet): H_j = sum_b d_b alpha^{j b} computed here with
    tests/gfref.py (the Horner steps' contract), then the generated Q network."""
    from tests import gfref
    src = open(os.path.join(PKG, "csrc", "rs_networks.cuh")).read()
    mt = re.search(r"template <> struct RsQNet<%d, %d, %d, 0x%Xu> \{(.*?)\n\};" % (k, m, w, poly), src, re.S)
    assert mt, "instance not found"
    stmts = re.findall(r"^\s+(?:const uint32_t (t\d+)|y\[(\d+)\]) = (.*);$", mt.group(1), re.M)
    cols = data.shape[1]
    H = []
    for j in range(m):
        aj = 1
        for _ in range(j):
            aj = gfref.mul(aj, 2, poly)
        row = []
        for c in range(cols):
            acc = 0
            for b in range(k - 1, -1, -1):      # Horner from the highest data position down
                acc = gfref.mul(acc, aj, poly) ^ int(data[b, c])
            row.append(acc)
        H.append(row)
    h = [sum(((H[j][c] >> b) & 1) << c for c in range(cols)) for j in range(m) for b in range(w)]
    env, y = {}, {}

    def val(tok):
        tok = tok.strip()
        if tok.startswith("h["):
            return h[int(tok[2:-1])]
        return 0 if tok == "0u" else env[tok]

    for tname, yidx, expr in stmts:
        v = 0
        for tok in expr.split("^"):
            v ^= val(tok)
        if tname:
            env[tname] = v
        else:
            y[int(yidx)] = v
    return [[sum(((y[i * w + o] >> c) & 1) << o for o in range(w)) for i in range(m)] for c in range(cols)]


def test_generated_networks_match_oracle():
    import gen_networks
    rng = np.random.default_rng(41)
    for (k, m, w, poly, _) in gen_networks.INSTANCES:
        if w in gen_networks.HORNER_W:
            data = rng.integers(0, 1 << w, (k, 32))
            par = horner_parity(k, m, w, poly, data)
            for c in range(0, 32, 3):
                assert par[c] == oracle.encode_column([int(v) for v in data[:, c]], m, w, poly), (k, m, w, c)
            continue
        groups = parse_network(k, m, w, poly)
        cols = 32
        data = rng.integers(0, 1 << w, (k, cols))
        planes = [np.uint32(0)] * (k * w)
        planes = []
        for j in range(k):
            for b in range(w):
                bits = (data[j] >> b) & 1
                planes.append(np.uint32(sum(int(bits[c]) << c for c in range(cols))))
        planes = [np.array([p], dtype=np.uint32) for p in planes]
        y = eval_network(groups, planes, m, w)
        for c in range(0, cols, 3):
            par = [sum(((int(y[i * w + o][0]) >> c) & 1) << o for o in range(w)) for i in range(m)]
            assert par == oracle.encode_column([int(v) for v in data[:, c]], m, w, poly), (k, m, w, c)


def test_generator_parity_map_matches_oracle():
    import gen_networks
    for (k, m, w, poly, _) in gen_networks.INSTANCES:
        P = gen_networks.parity_map(k, m, w, poly)
        for j in range(k):
            assert [P[i][j] for i in range(m)] == oracle.encode_column([int(i == j) for i in range(k)], m, w, poly)


def test_generated_header_is_current():
    import gen_networks
    head = open(os.path.join(PKG, "csrc", "rs_networks.cuh")).read(4096)
    assert f"generator-digest: {gen_networks.source_digest()}" in head


def test_headers_are_plain_c_and_demo_links():
    """include/*.h compile as C99 (no C++ in the ABI), and the C demo links against the
    built libraries (tools/c_api_demo.c; it runs on the GPU in tests/test_gpu_c_api.py)."""
    import shutil
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    root = os.path.dirname(PKG)
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "h.c")
        open(src, "w").write('#include "rs_poly.h"\n#include "rs_synth.h"\nint main(void){return 0;}\n')
        r = subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-pedantic", "-fsyntax-only", "-I",
                            os.path.join(root, "include"), src], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
        r = subprocess.run([gcc, "-std=c99", "-O2", "-I", os.path.join(root, "include"), "-I",
                            "/usr/local/cuda/include", os.path.join(root, "tools", "c_api_demo.c"), "-L", PKG,
                            "-lrs_poly", "-lrs_synth", "-L", "/usr/local/cuda/lib64", "-lcudart",
                            "-o", os.path.join(d, "demo")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]


def test_prepare_all_enumerates_every_pattern_host_only(rs):
    """rs_poly_prepare_all: sum_t C(n, t) patterns; bounds checked before anything is built
    (JIT off here: only the host-side Opt1/Opt3 constants, no GPU needed)."""
    from math import comb
    plan = rs.Plan(10, 4, 8, 0x11D)
    plan.set_jit(rs.RS_JIT_OFF)
    with pytest.raises(rs.RSError):
        plan.prepare_all(5)                       # max_t > m
    with pytest.raises(rs.RSError):
        plan.prepare_all(4, max_patterns=1469)    # 1470 patterns for RS(10,4)
    assert plan.stats()["patterns"] == 0          # nothing prepared on a refused call
    plan.prepare_all(0)
    plan.prepare_all(2)
    assert plan.stats()["patterns"] == comb(14, 1) + comb(14, 2)
    plan.prepare_all()
    assert plan.stats()["patterns"] == sum(comb(14, t) for t in range(1, 5)) == 1470
    plan.close()


def test_binding_refuses_host_memory_on_device_entry_points(rs):
    """Device entry points take CUDA tensors on the current device: a numpy array or a CPU
    tensor would be an illegal address inside a kernel, so the binding refuses it before the
    call; negative strides are refused too."""
    import torch
    plan = rs.Plan(4, 2, 8, 0x11D)
    host = np.zeros((2, 6, 64), dtype=np.uint8)
    for bad in (host, torch.zeros((2, 6, 64), dtype=torch.uint8)):
        with pytest.raises(ValueError, match="CUDA tensor"):
            plan.encode_batch(bad)
        with pytest.raises(ValueError, match="CUDA tensor"):
            plan.decode_batch(bad, np.full((2, 2), -1, dtype=np.int32))
    with pytest.raises(ValueError, match="CUDA tensor"):
        plan.encode([host[0, j] for j in range(4)], [host[0, 4], host[0, 5]], 64)
    with pytest.raises(ValueError, match="negative strides"):
        rs.rs_poly._geometry(host[::-1], 6, device=False)
    plan.close()
