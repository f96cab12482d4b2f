"""CPU oracle for polynomial Reed-Solomon (arXiv 1312.5155) -- TEST INFRASTRUCTURE ONLY.

This package wraps ``oracle/rs_oracle.c`` (plain scalar C, written from PAPER.md)
with ctypes.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it.  The product package
``paper_1312_5155_b200`` never imports it and shares no code with it.

Function -> passage:
  gf_mul, gf_pow, gf_inv, order_of_alpha ... GF(2^w) arithmetic, alpha=2 P:174
  gen_poly ................................. generator polynomial, P:170-177
  encode_column ............................ Eq. 1-2 long division, P:183-208
  eval_codeword ............................ root property c(alpha^j)=0
  decode_column ............................ two-step decode, P:213-303
  decode_matrix ............................ Step-2 Vandermonde matrix, P:244-263
  decode_column_forney ..................... independent textbook cross-check (not in the paper)
  encode_bulk / decode_bulk ................ the same steps over whole stripes, with
                                             Opt1/Opt3 and threads over stripes

Parity pins for every function live in tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u32, i32, sz, vp = ctypes.c_uint32, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p
        L.orc_field_ok.argtypes = [i32, u32]
        L.orc_gf_mul.argtypes = [u32, u32, i32, u32]; L.orc_gf_mul.restype = u32
        L.orc_gf_pow.argtypes = [u32, ctypes.c_uint64, i32, u32]; L.orc_gf_pow.restype = u32
        L.orc_gf_inv.argtypes = [u32, i32, u32]; L.orc_gf_inv.restype = u32
        L.orc_order_of_alpha.argtypes = [i32, u32]; L.orc_order_of_alpha.restype = u32
        L.orc_gen_poly.argtypes = [i32, i32, u32, vp]
        L.orc_encode_column.argtypes = [i32, i32, i32, u32, vp, vp]
        L.orc_eval_codeword.argtypes = [i32, i32, i32, u32, vp, u32]; L.orc_eval_codeword.restype = u32
        L.orc_decode_column.argtypes = [i32, i32, i32, u32, vp, vp, i32, vp]
        L.orc_decode_matrix.argtypes = [i32, i32, i32, u32, vp, i32, vp]
        L.orc_decode_column_forney.argtypes = [i32, i32, i32, u32, vp, vp, i32]
        L.orc_bulk_table_mul.argtypes = [i32, u32, vp, vp, vp, sz]
        L.orc_encode_bulk.argtypes = [i32, i32, i32, u32, vp, sz, sz, sz, sz, i32]
        L.orc_decode_bulk.argtypes = [i32, i32, i32, u32, vp, sz, sz, sz, sz, vp, i32]
        _lib = L
    return _lib


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


# ---- element arithmetic ---------------------------------------------------
def gf_mul(a: int, b: int, w: int = 8, poly: int = 0x11D) -> int:
    return int(lib().orc_gf_mul(a, b, w, poly))


def gf_pow(a: int, e: int, w: int = 8, poly: int = 0x11D) -> int:
    return int(lib().orc_gf_pow(a, e, w, poly))


def gf_inv(a: int, w: int = 8, poly: int = 0x11D) -> int:
    if a == 0:
        raise ZeroDivisionError("gf_inv(0)")
    return int(lib().orc_gf_inv(a, w, poly))


def order_of_alpha(w: int = 8, poly: int = 0x11D) -> int:
    return int(lib().orc_order_of_alpha(w, poly))


def bulk_table_mul(a, b, w: int = 8, poly: int = 0x11D) -> np.ndarray:
    a, b = _u32(a), _u32(b)
    out = np.zeros_like(a)
    if lib().orc_bulk_table_mul(w, poly, _ptr(a), _ptr(b), _ptr(out), a.size):
        raise ValueError("bad field")
    return out


# ---- polynomial / column level ---------------------------------------------
def gen_poly(m: int, w: int = 8, poly: int = 0x11D) -> list[int]:
    g = np.zeros(m + 1, dtype=np.uint32)
    if lib().orc_gen_poly(m, w, poly, _ptr(g)):
        raise ValueError("bad parameters")
    return [int(x) for x in g]


def encode_column(data, m: int, w: int = 8, poly: int = 0x11D) -> list[int]:
    d = _u32(data)
    p = np.zeros(m, dtype=np.uint32)
    if lib().orc_encode_column(d.size, m, w, poly, _ptr(d), _ptr(p)):
        raise ValueError("bad parameters")
    return [int(x) for x in p]


def eval_codeword(codeword, k: int, m: int, x: int, w: int = 8, poly: int = 0x11D) -> int:
    c = _u32(codeword)
    assert c.size == k + m
    return int(lib().orc_eval_codeword(k, m, w, poly, _ptr(c), x))


def decode_column(codeword, k: int, m: int, erasures, w: int = 8, poly: int = 0x11D,
                  want_syndromes: bool = False):
    """Return the repaired codeword (API order); optionally the Step-1 values D(alpha^j)."""
    c = _u32(codeword).copy()
    e = np.ascontiguousarray(np.asarray(list(erasures), dtype=np.int32))
    syn = np.zeros(max(1, e.size), dtype=np.uint32)
    rc = lib().orc_decode_column(k, m, w, poly, _ptr(c), _ptr(e), e.size, _ptr(syn))
    if rc:
        raise ValueError("decode failed rc=%d" % rc)
    out = [int(x) for x in c]
    if want_syndromes:
        return out, [int(x) for x in syn[: e.size]]
    return out


def decode_matrix(k: int, m: int, erasures, w: int = 8, poly: int = 0x11D) -> np.ndarray:
    e = np.ascontiguousarray(np.asarray(list(erasures), dtype=np.int32))
    V = np.zeros((e.size, e.size), dtype=np.uint32)
    if lib().orc_decode_matrix(k, m, w, poly, _ptr(e), e.size, _ptr(V)):
        raise ValueError("bad erasures")
    return V


def decode_column_forney(codeword, k: int, m: int, erasures, w: int = 8, poly: int = 0x11D) -> list[int]:
    c = _u32(codeword).copy()
    e = np.ascontiguousarray(np.asarray(list(erasures), dtype=np.int32))
    rc = lib().orc_decode_column_forney(k, m, w, poly, _ptr(c), _ptr(e), e.size)
    if rc:
        raise ValueError("forney failed rc=%d" % rc)
    return [int(x) for x in c]


# ---- bulk (whole stripes) ----------------------------------------------------
def encode_bulk(stripes: np.ndarray, k: int, m: int, w: int = 8, poly: int = 0x11D, threads: int = 1) -> None:
    """In place: ``stripes`` is uint8 ``[S][n][B]`` (C-contiguous); writes blocks k..n-1."""
    assert stripes.dtype == np.uint8 and stripes.flags.c_contiguous and stripes.shape[1] == k + m
    S, n, B = stripes.shape
    rc = lib().orc_encode_bulk(k, m, w, poly, _ptr(stripes), S, n * B, B, B, threads)
    if rc:
        raise ValueError("encode_bulk rc=%d" % rc)


def decode_bulk(stripes: np.ndarray, erasures: np.ndarray, k: int, m: int, w: int = 8, poly: int = 0x11D,
                threads: int = 1) -> None:
    """In place: recover the erased blocks listed per stripe in ``erasures`` ([S][m] int32, -1 padded)."""
    assert stripes.dtype == np.uint8 and stripes.flags.c_contiguous and stripes.shape[1] == k + m
    S, n, B = stripes.shape
    er = np.ascontiguousarray(erasures, dtype=np.int32)
    assert er.shape == (S, m)
    rc = lib().orc_decode_bulk(k, m, w, poly, _ptr(stripes), S, n * B, B, B, _ptr(er), threads)
    if rc:
        raise ValueError("decode_bulk rc=%d" % rc)
