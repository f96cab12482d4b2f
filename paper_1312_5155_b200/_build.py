"""In-tree build of the native libraries (sm_100a only).

  librs_poly.so  -- the C-ABI library (include/rs_poly.h): kernels + planner
  librs_synth.so -- on-device input generator (include/rs_synth.h)

Both link the CUDA runtime statically, so they do not depend on torch's runtime.
Rebuilds only when a source is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
ROOT = os.path.dirname(PKG)
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-diag-suppress", "128",
                "-I", INCLUDE, "-cudart", "static", "--threads", "0"]

POLY_LIB = os.path.join(PKG, "librs_poly.so")
SYNTH_LIB = os.path.join(PKG, "librs_synth.so")


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    print("[build]", " ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def _embed(src: str, dst: str, name: str) -> None:
    """Write `src` as a C++ raw string literal (the JIT prepends it to generated kernels)."""
    text = open(src).read()
    body = f'static const char {name}[] = R"RSJIT({text})RSJIT";\n'
    if not os.path.exists(dst) or open(dst).read() != body:
        with open(dst, "w") as f:
            f.write(body)


def build(verbose_ptxas: bool = False) -> list[str]:
    sys.path.insert(0, CSRC)
    try:
        import gen_networks  # noqa: E402
        gen_networks.generate()
    finally:
        sys.path.pop(0)
    _embed(os.path.join(CSRC, "bitslice_device.cuh"), os.path.join(CSRC, "bitslice_device_src.inc"),
           "kBitsliceDeviceSrc")
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.inc")) + glob.glob(os.path.join(CSRC, "*.hpp")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    poly_src = [os.path.join(CSRC, f) for f in ("rs_kernels.cu", "polyrs_ablation.cu", "plan.cpp", "linear.cpp",
                                                 "host_pipeline.cpp", "jit.cpp")]
    extra = ["-Xptxas", "-v"] if verbose_ptxas else []
    if _stale(POLY_LIB, poly_src + headers + [__file__]):
        tmp = POLY_LIB + ".tmp%d" % os.getpid()
        _run([NVCC] + FLAGS + extra + ["-shared", "-o", tmp] + poly_src + ["-ldl"])
        os.replace(tmp, POLY_LIB)
    synth_src = [os.path.join(CSRC, "synth.cu")]
    if _stale(SYNTH_LIB, synth_src + [os.path.join(INCLUDE, "rs_synth.h"), __file__]):
        tmp = SYNTH_LIB + ".tmp%d" % os.getpid()
        _run([NVCC] + FLAGS + ["-shared", "-o", tmp] + synth_src)
        os.replace(tmp, SYNTH_LIB)
    return [POLY_LIB, SYNTH_LIB]


if __name__ == "__main__":
    for p in build(verbose_ptxas="-v" in sys.argv):
        print(p)
