"""Thin ctypes binding of libptucker.so (include/ptucker.h) -- argument marshalling only.

Every computation runs in the library's CUDA kernels; there is no Python or CPU
fallback: if the shared library is missing this module raises at load time.
Function names and argument order follow the C-ABI (see include/ptucker.h for
the meaning, layout, ownership and error behaviour of each call).
"""
from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# PTUCKER_LIB: a tools-only experiment build (build.py --variant) loaded instead of the
# in-tree product library; unset in tests, smoke() and the bench
LIB_PATH = os.environ.get("PTUCKER_LIB") or os.path.join(_HERE, "libptucker.so")

PTUCKER_OK, PTUCKER_EINVAL, PTUCKER_ENUMERIC, PTUCKER_ERESOURCE = 0, 1, 2, 3
PTUCKER_ECUDA, PTUCKER_ENCCL, PTUCKER_ESTATE = 4, 5, 6
PTUCKER_F32, PTUCKER_F64 = 0, 1

_SIGS = {
    "ptucker_version": (C.c_int32, []),
    "ptucker_last_error": (C.c_char_p, []),
    "ptucker_get_unique_id": (C.c_int, [C.c_void_p]),
    "ptucker_comm_init": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p]),
    "ptucker_partition_rows": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "ptucker_peer_handles": (C.c_int, [C.c_void_p, C.c_int32]),
    "ptucker_open_peers": (C.c_int, [C.c_void_p, C.c_int32]),
    "ptucker_set_stream": (C.c_int, [C.c_void_p]),
    "ptucker_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                               C.c_double, C.c_uint64]),
    "ptucker_update_mode": (C.c_int, [C.c_int32]),
    "ptucker_sweep": (C.c_int, []),
    "ptucker_error": (C.c_int, [C.POINTER(C.c_double)]),
    "ptucker_error_literal": (C.c_int, [C.POINTER(C.c_double)]),
    "ptucker_orthogonalize": (C.c_int, []),
    "ptucker_core_scores": (C.c_int, [C.c_void_p]),
    "ptucker_truncate_core": (C.c_int, [C.c_double, C.POINTER(C.c_int64)]),
    "ptucker_core_nnz": (C.c_int, [C.POINTER(C.c_int64)]),
    "ptucker_predict": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p]),
    "ptucker_test_rmse": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double)]),
    "ptucker_run": (C.c_int, [C.c_int32, C.c_double, C.c_double, C.c_int32, C.c_void_p, C.POINTER(C.c_int32)]),
    "ptucker_get_factor": (C.c_int, [C.c_int32, C.c_void_p]),
    "ptucker_set_factor": (C.c_int, [C.c_int32, C.c_void_p]),
    "ptucker_get_core": (C.c_int, [C.c_void_p]),
    "ptucker_set_core": (C.c_int, [C.c_void_p]),
    "ptucker_get_mode_index": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p]),
    "ptucker_get_partition": (C.c_int, [C.c_int32, C.c_void_p]),
    "ptucker_set_option": (C.c_int, [C.c_char_p, C.c_int64]),
    "ptucker_kernel_stats": (C.c_int, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "ptucker_reset_kernel_stats": (C.c_int, []),
    "ptucker_info": (C.c_int, [C.c_char_p, C.c_int32]),
    "ptucker_debug_trace": (C.c_int, [C.c_void_p, C.c_int32]),
    "ptucker_synchronize": (C.c_int, []),
    "ptucker_finalize": (C.c_int, []),
}
EXPORTS = tuple(_SIGS)


class PTuckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def load():
    """Load the in-tree libptucker.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1710_02261_b200.build` "
                              "(there is no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _check(rc: int):
    if rc != PTUCKER_OK:
        raise PTuckerError(rc, load().ptucker_last_error().decode())


def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


_state = {"dims": None, "J": None, "dtype": None}


def ptucker_version() -> int:
    return int(load().ptucker_version())


def ptucker_last_error() -> str:
    return load().ptucker_last_error().decode()


def ptucker_get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(load().ptucker_get_unique_id(buf))
    return bytes(buf)


def ptucker_peer_handles() -> bytes:
    n = ptucker_info()["N"]
    buf = C.create_string_buffer(64 * n)
    _check(load().ptucker_peer_handles(buf, 64 * n))
    return buf.raw


def ptucker_open_peers(handles: bytes, world: int):
    buf = C.create_string_buffer(bytes(handles), len(handles))
    _check(load().ptucker_open_peers(buf, world))


def ptucker_comm_init(rank: int, world: int, uid: bytes | None):
    buf = (C.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
    _check(load().ptucker_comm_init(rank, world, buf))


def ptucker_partition_rows(row_ptr, world: int) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    out = np.zeros(world + 1, np.int64)
    _check(load().ptucker_partition_rows(_ptr(row_ptr), row_ptr.size - 1, world, _ptr(out)))
    return out


def ptucker_set_stream(stream: int | None):
    _check(load().ptucker_set_stream(C.c_void_p(stream) if stream else None))


def ptucker_init(coords, vals, dims, core_dims, lam: float, seed: int):
    """coords: int32 [nnz, N] (0-based); vals: float32 or float64 [nnz] (selects the precision)."""
    coords = np.ascontiguousarray(coords, np.int32)
    vals = np.ascontiguousarray(vals)
    if vals.dtype not in (np.float32, np.float64):
        raise TypeError("vals must be float32 or float64")
    dims = np.ascontiguousarray(dims, np.int64)
    core_dims = np.ascontiguousarray(core_dims, np.int32)
    N = int(dims.size)
    if coords.ndim != 2 or coords.shape[1] != N or coords.shape[0] != vals.size:
        raise ValueError("coords must be [nnz, N] with nnz == vals.size")
    dt = PTUCKER_F64 if vals.dtype == np.float64 else PTUCKER_F32
    _check(load().ptucker_init(_ptr(coords), _ptr(vals), dt, vals.size, N, _ptr(dims), _ptr(core_dims),
                               float(lam), int(seed)))
    _state.update(dims=[int(d) for d in dims], J=[int(j) for j in core_dims], dtype=vals.dtype)


def ptucker_update_mode(n: int):
    _check(load().ptucker_update_mode(n))


def ptucker_sweep():
    _check(load().ptucker_sweep())


def ptucker_error() -> float:
    out = C.c_double()
    _check(load().ptucker_error(C.byref(out)))
    return out.value


def ptucker_error_literal() -> float:
    out = C.c_double()
    _check(load().ptucker_error_literal(C.byref(out)))
    return out.value


def ptucker_orthogonalize():
    _check(load().ptucker_orthogonalize())


def ptucker_core_scores() -> np.ndarray:
    """Eq. 13 partial reconstruction error of every core entry (C order, NaN = truncated)."""
    out = np.empty(tuple(_state["J"]), np.float64)
    _check(load().ptucker_core_scores(_ptr(out)))
    return out


def ptucker_truncate_core(p: float) -> int:
    """Alg. 4: zero the top floor(p|G|) core entries by R(beta); returns the number removed."""
    k = C.c_int64()
    _check(load().ptucker_truncate_core(float(p), C.byref(k)))
    return int(k.value)


def ptucker_core_nnz() -> int:
    k = C.c_int64()
    _check(load().ptucker_core_nnz(C.byref(k)))
    return int(k.value)


def ptucker_predict(coords) -> np.ndarray:
    """Eq. 4 predictions for query coordinates (n x N int32)."""
    coords = np.ascontiguousarray(coords, np.int32)
    out = np.empty(coords.shape[0], np.float64)
    _check(load().ptucker_predict(_ptr(coords), coords.shape[0], _ptr(out)))
    return out


def ptucker_test_rmse(coords, vals) -> float:
    """Held-out RMSE of the test entries (values converted to the context's precision)."""
    coords = np.ascontiguousarray(coords, np.int32)
    vals = np.ascontiguousarray(vals, _state["dtype"])
    out = C.c_double()
    dt = PTUCKER_F64 if vals.dtype == np.float64 else PTUCKER_F32
    _check(load().ptucker_test_rmse(_ptr(coords), _ptr(vals), dt, coords.shape[0], C.byref(out)))
    return out.value


def ptucker_run(max_iters: int, tol: float = 1e-4, approx_p: float = 0.0, orthogonalize: bool = True):
    """Alg. 2 driver: returns (errors e_0..e_T, T)."""
    errs = np.zeros(max_iters + 1, np.float64)
    it = C.c_int32()
    _check(load().ptucker_run(int(max_iters), float(tol), float(approx_p), int(orthogonalize), _ptr(errs),
                              C.byref(it)))
    return errs[: it.value + 1], int(it.value)


def ptucker_get_factor(n: int, out: np.ndarray | None = None) -> np.ndarray:
    if out is None:
        out = np.empty((_state["dims"][n], _state["J"][n]), _state["dtype"])
    _check(load().ptucker_get_factor(n, _ptr(out)))
    return out


def ptucker_set_factor(n: int, a):
    a = np.ascontiguousarray(a, _state["dtype"])
    assert a.shape == (_state["dims"][n], _state["J"][n])
    _check(load().ptucker_set_factor(n, _ptr(a)))


def ptucker_get_core() -> np.ndarray:
    out = np.empty(tuple(_state["J"]), _state["dtype"])
    _check(load().ptucker_get_core(_ptr(out)))
    return out


def ptucker_set_core(G):
    G = np.ascontiguousarray(G, _state["dtype"])
    assert G.shape == tuple(_state["J"])
    _check(load().ptucker_set_core(_ptr(G)))


def ptucker_get_mode_index(n: int):
    nnz = ptucker_info()["nnz"]
    row_ptr = np.empty(_state["dims"][n] + 1, np.int64)
    perm = np.empty(nnz, np.int64)
    _check(load().ptucker_get_mode_index(n, _ptr(row_ptr), _ptr(perm)))
    return row_ptr, perm


def ptucker_get_partition(n: int) -> np.ndarray:
    world = ptucker_info()["world"]
    out = np.empty(world + 1, np.int64)
    _check(load().ptucker_get_partition(n, _ptr(out)))
    return out


def ptucker_set_option(key: str, value: int):
    _check(load().ptucker_set_option(key.encode(), int(value)))


def ptucker_kernel_stats(name: str):
    ms, cnt = C.c_double(), C.c_int64()
    _check(load().ptucker_kernel_stats(name.encode(), C.byref(ms), C.byref(cnt)))
    return ms.value, cnt.value


def ptucker_reset_kernel_stats():
    _check(load().ptucker_reset_kernel_stats())


def ptucker_info() -> dict:
    buf = C.create_string_buffer(1 << 16)
    _check(load().ptucker_info(buf, len(buf)))
    return json.loads(buf.value.decode())


def ptucker_debug_trace(n: int = 4096) -> np.ndarray:
    out = np.zeros(n, np.int64)
    _check(load().ptucker_debug_trace(_ptr(out), n))
    return out


def ptucker_synchronize():
    _check(load().ptucker_synchronize())


def ptucker_finalize():
    _check(load().ptucker_finalize())
