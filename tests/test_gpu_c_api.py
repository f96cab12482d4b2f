"""The library from plain C on the GPU (tools/c_api_demo.c): encode, erase, decode, verify and
per-call latency through include/rs_poly.h with no Python in the loop."""
import json
import os
import shutil
import subprocess
import tempfile

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_api_demo_runs():
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    pkg = os.path.join(ROOT, "paper_1312_5155_b200")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "demo")
        r = subprocess.run([gcc, "-std=c99", "-O2", "-I", os.path.join(ROOT, "include"), "-I",
                            "/usr/local/cuda/include", os.path.join(ROOT, "tools", "c_api_demo.c"), "-L", pkg,
                            "-lrs_poly", "-lrs_synth", "-L", "/usr/local/cuda/lib64", "-lcudart",
                            f"-Wl,-rpath,{pkg}", "-o", exe], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]
        out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert out.returncode == 0, out.stdout + out.stderr
        res = json.loads(out.stdout.strip().splitlines()[-1])
        assert res["restored"] and res["verify_flag"] == 0 and res["c1_encode_us"] > 0
