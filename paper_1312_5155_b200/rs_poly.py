"""Thin ctypes binding of include/rs_poly.h (argument marshalling only).

Every computing call goes to librs_poly.so (hand-written sm_100a kernels).  There
is no CPU fallback: if the library is missing this module raises on import.
Names follow the C ABI; see the header for argument meaning, layout and errors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RS_POLY_LIB") or os.path.join(_PKG, "librs_poly.so")
SYNTH_PATH = os.path.join(_PKG, "librs_synth.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)
_vp, _sz, _i32, _u32, _u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64
_P = ctypes.POINTER

_lib.rs_poly_plan_create.argtypes = [_i32, _i32, _i32, _u32, _P(_vp)]
_lib.rs_poly_plan_destroy.argtypes = [_vp]
_lib.rs_poly_plan_destroy.restype = None
_lib.rs_poly_plan_info.argtypes = [_vp, _vp, _vp]
_lib.rs_poly_plan_kernel_kind.argtypes = [_vp]
_lib.rs_poly_encode.argtypes = [_vp, _vp, _vp, _sz, _vp]
_lib.rs_poly_decode.argtypes = [_vp, _vp, _sz, _vp, _i32, _vp]
_lib.rs_poly_encode_batch.argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp]
_lib.rs_poly_decode_batch.argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _vp]
_lib.rs_poly_encode_host.argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _P(_u64), _P(_u64)]
_lib.rs_poly_decode_host.argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _vp, _P(_u64), _P(_u64)]
_lib.rs_poly_strerror.argtypes = [_i32]
_lib.rs_poly_strerror.restype = ctypes.c_char_p
_lib.rs_poly_abi_version.restype = _i32
_lib.rs_poly_plan_set_jit.argtypes = [_vp, _i32]
_lib.rs_poly_plan_set_read_policy.argtypes = [_vp, _i32]
_lib.rs_poly_prepare.argtypes = [_vp, _vp, _sz]
_lib.rs_poly_plan_stats.argtypes = [_vp, _vp]
_lib.rs_poly_prepare_all.argtypes = [_vp, _i32, _sz]
_lib.rs_poly_jit_source.argtypes = [_vp, _vp, _i32, ctypes.c_char_p, _sz]
_lib.rs_poly_jit_source.restype = _sz
_lib.rs_poly_update.argtypes = [_vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp]
_lib.rs_poly_update_batch.argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _i32, _vp, _sz, _sz, _vp]
_lib.rs_poly_update_jit_source.argtypes = [_vp, _vp, _i32, ctypes.c_char_p, _sz]
_lib.rs_poly_update_jit_source.restype = _sz
_lib.rs_poly_prepare_update.argtypes = [_vp, _vp, _i32]
_lib.rs_poly_ablation_decode.argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _i32, _i32, _vp]
_lib.rs_poly_encode_partial.argtypes = [_vp, _vp, _i32, _vp, _vp, _sz, _sz, _i32, _vp]
_lib.rs_poly_xor_reduce.argtypes = [_vp, _vp, _vp, _i32, _sz, _sz, _vp]
_lib.rs_poly_verify_batch.argtypes = [_vp, _vp, _sz, _sz, _sz, _sz, _vp, _vp]


class Stats(ctypes.Structure):
    """rs_poly_stats"""
    _fields_ = [("patterns", _u64), ("jit_ready", _u64), ("jit_pending", _u64), ("jit_failed", _u64),
                ("jit_launches", _u64), ("table_launches", _u64), ("jit_available", _i32), ("jit_mode", _i32),
                ("jit_cache_hits", _u64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


RS_JIT_OFF, RS_JIT_BACKGROUND, RS_JIT_SYNC = 0, 1, 2
RS_READ_ALL_SURVIVORS, RS_READ_K_SURVIVORS = 0, 1
_lib.rs_poly_launch_count.restype = _u64

RS_OK, RS_ERR_INVALID_ARG, RS_ERR_NOT_PRIMITIVE, RS_ERR_GEOMETRY = 0, 1, 2, 3
RS_ERR_TOO_MANY_ERASURES, RS_ERR_BAD_ERASURE, RS_ERR_CUDA, RS_ERR_NOMEM = 4, 5, 6, 7
DEFAULT_POLY = {8: 0x11D, 16: 0x1100B}


class RSError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{what}: {strerror(status)} (rs_status {status})")


def strerror(status: int) -> str:
    return _lib.rs_poly_strerror(status).decode()


def abi_version() -> int:
    return int(_lib.rs_poly_abi_version())


def launch_count() -> int:
    """Kernels this library has launched since load."""
    return int(_lib.rs_poly_launch_count())


def _check(status: int, what: str) -> None:
    if status != RS_OK:
        raise RSError(status, what)


def _stream(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if hasattr(stream, "cuda_stream"):
        return stream.cuda_stream
    return int(stream)


def _ptr(x) -> int:
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if isinstance(x, np.ndarray):
        return int(x.ctypes.data)
    return int(x)


def _where(x, device: bool):
    """Device entry points take CUDA tensors on the current device; host ones numpy arrays or
    CPU tensors.  A mismatch would be an illegal address inside a kernel (a sticky context
    error) or a kernel on another GPU's stream, so it is refused here."""
    if hasattr(x, "is_cuda"):
        if device:
            if not x.is_cuda:
                raise ValueError("expected a CUDA tensor (this entry point reads device memory)")
            import torch
            if x.device.index != torch.cuda.current_device():
                raise ValueError(f"tensor is on cuda:{x.device.index} but the current device is "
                                 f"cuda:{torch.cuda.current_device()} (use torch.cuda.device(...))")
        elif x.is_cuda:
            raise ValueError("expected host memory (numpy array or CPU tensor), got a CUDA tensor")
    elif isinstance(x, np.ndarray) and device:
        raise ValueError("expected a CUDA tensor, got a numpy (host) array")


def _dptr(x) -> int:
    """Address of a device buffer (tensor checked by _where; raw ints are taken as given)."""
    _where(x, True)
    return _ptr(x)


def _geometry(stripes, n: int, device: bool = True):
    """(ptr, S, stripe_stride, block_stride, block_bytes) of a [S][n][B] uint8 array/tensor."""
    _where(stripes, device)
    shape = tuple(stripes.shape)
    if len(shape) != 3 or shape[1] != n:
        raise ValueError(f"expected a [S][{n}][B] uint8 array, got shape {shape}")
    if hasattr(stripes, "element_size"):
        if stripes.element_size() != 1:
            raise ValueError("expected uint8")
        st = stripes.stride()
    else:
        if stripes.dtype != np.uint8:
            raise ValueError("expected uint8")
        st = stripes.strides
    if st[2] != 1:
        raise ValueError("blocks must be contiguous (last stride 1)")
    if st[0] < 0 or st[1] < 0:
        raise ValueError("negative strides are not supported")
    return _ptr(stripes), shape[0], st[0], st[1], shape[2]


def _erasure_table(erasures, S: int, m: int) -> np.ndarray:
    er = np.ascontiguousarray(np.asarray(erasures, dtype=np.int32))
    if er.shape != (S, m):
        raise ValueError(f"erasures must be int32 [{S}][{m}] (-1 padded)")
    return er


class Plan:
    """An RS(k, m) code over GF(2^w) with alpha = 2 (rs_poly_plan_create)."""

    def __init__(self, k: int, m: int, w: int = 8, prim_poly: int | None = None):
        self.k, self.m, self.w = k, m, w
        self.n = k + m
        self.prim_poly = DEFAULT_POLY.get(w, 0) if prim_poly is None else prim_poly
        h = _vp()
        _check(_lib.rs_poly_plan_create(k, m, w, self.prim_poly, ctypes.byref(h)), "rs_poly_plan_create")
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.rs_poly_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ---- run-time specialised kernels ------------------------------------------
    def set_jit(self, mode: int) -> None:
        """RS_JIT_OFF / RS_JIT_BACKGROUND (default) / RS_JIT_SYNC."""
        _check(_lib.rs_poly_plan_set_jit(self._h, mode), "rs_poly_plan_set_jit")

    def set_read_policy(self, policy: int) -> None:
        """RS_READ_ALL_SURVIVORS (default, the paper's Step 1) / RS_READ_K_SURVIVORS."""
        _check(_lib.rs_poly_plan_set_read_policy(self._h, policy), "rs_poly_plan_set_read_policy")

    def prepare(self, erasures) -> None:
        """Precompute decode constants and compile JIT kernels for these patterns ([rows][m], -1 padded)."""
        er = np.ascontiguousarray(np.asarray(erasures, dtype=np.int32)).reshape(-1, self.m)
        _check(_lib.rs_poly_prepare(self._h, er.ctypes.data, er.shape[0]), "rs_poly_prepare")

    def prepare_all(self, max_t: int | None = None, max_patterns: int = 8192) -> None:
        """Compile the decode kernel of every pattern of 1..max_t (default m) erasures now
        (rs_poly_prepare_all): no decode call then waits on, or falls back from, a JIT compile."""
        t = self.m if max_t is None else max_t
        _check(_lib.rs_poly_prepare_all(self._h, t, max_patterns), "rs_poly_prepare_all")

    def stats(self) -> dict:
        st = Stats()
        _check(_lib.rs_poly_plan_stats(self._h, ctypes.byref(st)), "rs_poly_plan_stats")
        return st.as_dict()

    def jit_source(self, erasures=()) -> str:
        """CUDA source the JIT generates for an erasure list (empty = the encoder); '' if not eligible."""
        er = list(erasures)
        e = (ctypes.c_int * max(1, len(er)))(*er)
        n = _lib.rs_poly_jit_source(self._h, e, len(er), None, 0)
        if n == 0:
            return ""
        buf = ctypes.create_string_buffer(n + 1)
        _lib.rs_poly_jit_source(self._h, e, len(er), buf, n + 1)
        return buf.value.decode()

    @property
    def kernel_kind(self) -> str:
        return "bitsliced" if _lib.rs_poly_plan_kernel_kind(self._h) == 1 else "generic"

    def info(self):
        """(g low->high, parity map [m][k]) -- host-only."""
        g = np.zeros(self.m + 1, dtype=np.uint32)
        P = np.zeros((self.m, self.k), dtype=np.uint32)
        _check(_lib.rs_poly_plan_info(self._h, g.ctypes.data, P.ctypes.data), "rs_poly_plan_info")
        return g, P

    # ---- single stripe -------------------------------------------------------
    def encode(self, data, parity, block_bytes: int, stream=None) -> None:
        d = (ctypes.c_void_p * self.k)(*[_dptr(x) for x in data])
        p = (ctypes.c_void_p * self.m)(*[_dptr(x) for x in parity])
        _check(_lib.rs_poly_encode(self._h, d, p, block_bytes, _stream(stream)), "rs_poly_encode")

    def decode(self, blocks, block_bytes: int, erasures, stream=None) -> None:
        b = (ctypes.c_void_p * self.n)(*[_dptr(x) for x in blocks])
        er = list(erasures)
        e = (ctypes.c_int * max(1, len(er)))(*er)
        _check(_lib.rs_poly_decode(self._h, b, block_bytes, e, len(er), _stream(stream)), "rs_poly_decode")

    # ---- batched (device memory) ----------------------------------------------
    def encode_batch(self, stripes, stream=None) -> None:
        ptr, S, ss, bs, B = _geometry(stripes, self.n)
        _check(_lib.rs_poly_encode_batch(self._h, ptr, S, ss, bs, B, _stream(stream)), "rs_poly_encode_batch")

    def decode_batch(self, stripes, erasures, stream=None) -> None:
        ptr, S, ss, bs, B = _geometry(stripes, self.n)
        er = _erasure_table(erasures, S, self.m)
        _check(_lib.rs_poly_decode_batch(self._h, ptr, S, ss, bs, B, er.ctypes.data, _stream(stream)),
               "rs_poly_decode_batch")

    # ---- diff-update ----------------------------------------------------
    def update(self, data_idx, old_data, new_data, parity, block_bytes: int, stream=None) -> None:
        """parity ^= P[:, data_idx] (old ^ new), in place (rs_poly_update)."""
        idx = list(data_idx)
        c = len(idx)
        ix = (ctypes.c_int * max(1, c))(*idx)
        o = (ctypes.c_void_p * max(1, c))(*[_dptr(x) for x in old_data])
        nw = (ctypes.c_void_p * max(1, c))(*[_dptr(x) for x in new_data])
        p = (ctypes.c_void_p * self.m)(*[_dptr(x) for x in parity])
        _check(_lib.rs_poly_update(self._h, ix, c, o, nw, p, block_bytes, _stream(stream)), "rs_poly_update")

    def update_batch(self, stripes, data_idx, old_blocks, stream=None) -> None:
        """stripes [S][n][B]: new data + old parity (updated in place); old_blocks [S][c][B]."""
        ptr, S, ss, bs, B = _geometry(stripes, self.n)
        idx = list(data_idx)
        c = len(idx)
        ix = (ctypes.c_int * max(1, c))(*idx)
        shape = tuple(old_blocks.shape)
        if c and (len(shape) != 3 or shape[0] != S or shape[1] != c or shape[2] != B):
            raise ValueError(f"old_blocks must be [{S}][{c}][{B}]")
        _where(old_blocks, True)
        ost = old_blocks.stride() if hasattr(old_blocks, "stride") else old_blocks.strides
        if ost[0] < 0 or ost[1] < 0:
            raise ValueError("negative strides are not supported")
        _check(_lib.rs_poly_update_batch(self._h, ptr, S, ss, bs, B, ix, c, _ptr(old_blocks), ost[0], ost[1],
                                         _stream(stream)), "rs_poly_update_batch")

    def prepare_update(self, data_idx) -> None:
        """Compile the diff-update kernel for this changed set now (rs_poly_prepare_update)."""
        idx = list(data_idx)
        ix = (ctypes.c_int * max(1, len(idx)))(*idx)
        _check(_lib.rs_poly_prepare_update(self._h, ix, len(idx)), "rs_poly_prepare_update")

    def update_jit_source(self, data_idx) -> str:
        idx = list(data_idx)
        ix = (ctypes.c_int * max(1, len(idx)))(*idx)
        n = _lib.rs_poly_update_jit_source(self._h, ix, len(idx), None, 0)
        if n == 0:
            return ""
        buf = ctypes.create_string_buffer(n + 1)
        _lib.rs_poly_update_jit_source(self._h, ix, len(idx), buf, n + 1)
        return buf.value.decode()

    # ---- cross-GPU placement pieces (NEXT-4) ----------------------------------------
    def encode_partial(self, data_idx, data, partial, block_bytes: int, accumulate: bool = False,
                       stream=None) -> None:
        """partial[s][i] (^)= sum_q P[i][data_idx[q]] data[s][q]; data [S][c], partial [S][m] (pointers/tensors)."""
        idx = list(data_idx)
        c, S = len(idx), len(partial)
        ix = (ctypes.c_int * max(1, c))(*idx)
        d = (ctypes.c_void_p * max(1, S * c))(*[_dptr(x) for row in data for x in row])
        p = (ctypes.c_void_p * (S * self.m))(*[_dptr(x) for row in partial for x in row])
        _check(_lib.rs_poly_encode_partial(self._h, ix, c, d, p, S, block_bytes, int(accumulate), _stream(stream)),
               "rs_poly_encode_partial")

    def xor_reduce(self, dst, srcs, nbytes: int, stream=None) -> None:
        """dst[s] = XOR of srcs[s][*] (lists of pointers/tensors; dst may alias a source)."""
        S, n_src = len(dst), len(srcs[0])
        dp = (ctypes.c_void_p * S)(*[_dptr(x) for x in dst])
        sp = (ctypes.c_void_p * (S * n_src))(*[_dptr(x) for row in srcs for x in row])
        _check(_lib.rs_poly_xor_reduce(self._h, dp, sp, n_src, S, nbytes, _stream(stream)), "rs_poly_xor_reduce")

    # ---- the paper's optimisation study (NEXT-3) -----------------------------------
    def ablation_decode(self, stripes, erasures, opt_mask: int, stream=None) -> None:
        """Per-column table decode with Opt1/2/3 = opt_mask bits 0/1/2 (0 = PolyRS, 7 = OptPolyRS)."""
        ptr, S, ss, bs, B = _geometry(stripes, self.n)
        er = list(erasures)
        e = (ctypes.c_int * max(1, len(er)))(*er)
        _check(_lib.rs_poly_ablation_decode(self._h, ptr, S, ss, bs, B, e, len(er), opt_mask, _stream(stream)),
               "rs_poly_ablation_decode")

    def verify_batch(self, stripes, flags, stream=None) -> None:
        """flags[s] = 0 if every column of stripe s is a codeword, else 1 (flags: int32 device [S])."""
        ptr, S, ss, bs, B = _geometry(stripes, self.n)
        _where(flags, True)
        if tuple(flags.shape) != (S,) or flags.element_size() != 4:
            raise ValueError(f"flags must be a 32-bit device tensor [{S}]")
        _check(_lib.rs_poly_verify_batch(self._h, ptr, S, ss, bs, B, _ptr(flags), _stream(stream)),
               "rs_poly_verify_batch")

    # ---- end to end from host memory --------------------------------------------
    def encode_host(self, host_stripes, stream=None):
        ptr, S, ss, bs, B = _geometry(host_stripes, self.n, device=False)
        h2d, d2h = _u64(), _u64()
        _check(_lib.rs_poly_encode_host(self._h, ptr, S, ss, bs, B, _stream(stream), ctypes.byref(h2d),
                                        ctypes.byref(d2h)), "rs_poly_encode_host")
        return int(h2d.value), int(d2h.value)

    def decode_host(self, host_stripes, erasures, stream=None):
        ptr, S, ss, bs, B = _geometry(host_stripes, self.n, device=False)
        er = _erasure_table(erasures, S, self.m)
        h2d, d2h = _u64(), _u64()
        _check(_lib.rs_poly_decode_host(self._h, ptr, S, ss, bs, B, er.ctypes.data, _stream(stream),
                                        ctypes.byref(h2d), ctypes.byref(d2h)), "rs_poly_decode_host")
        return int(h2d.value), int(d2h.value)


# ---- on-device input generator (librs_synth.so; not the method) ---------------
_synth = None


def synth_fill(stripes, k: int, seed: int, stripe0: int = 0, stream=None) -> None:
    """Fill data blocks 0..k-1 of a [S][n][B] device array with the synth/ recipe."""
    global _synth
    if _synth is None:
        _synth = ctypes.CDLL(SYNTH_PATH)
        _synth.rs_synth_fill.argtypes = [_vp, _sz, _sz, _sz, _sz, _i32, _u32, _u32, _vp]
    _where(stripes, True)
    shape = tuple(stripes.shape)
    ptr, S, ss, bs, B = _ptr(stripes), shape[0], stripes.stride()[0], stripes.stride()[1], shape[2]
    rc = _synth.rs_synth_fill(ptr, S, ss, bs, B, k, seed, stripe0, _stream(stream))
    if rc != 0:
        raise RuntimeError(f"rs_synth_fill failed ({rc})")
