"""Python (ctypes) front end of the FP64 CPU oracle in ptucker_oracle.c.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py
(cpu_baseline / --impl reference) may import this module.  The product path
(paper_1710_02261_b200/) never imports it, and it imports nothing from there.

All arithmetic lives in ptucker_oracle.c (plain C, FP64, the paper's algorithm
step by step; see that file's header for the P:<line> citations).  This module
only marshals numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ptucker_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (OpenMP for the paper's dynamic row loop)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.c_void_p
        i64, i32, f64, u64 = C.c_int64, C.c_int32, C.c_double, C.c_uint64
        sig = {
            "or_mix64": (u64, [u64]),
            "or_rng_word": (u64, [u64, u64, u64]),
            "or_uniform": (f64, [u64, u64, u64, C.c_int]),
            "or_init": (None, [C.c_int, P, P, u64, C.c_int, P, P]),
            "or_mode_index": (C.c_int, [C.c_int, i64, P, P, C.c_int, P, P]),
            "or_partition": (None, [P, i64, C.c_int, P]),
            "or_delta": (None, [C.c_int, P, P, P, P, P, C.c_int, P]),
            "or_predict": (f64, [C.c_int, P, P, P, P, P]),
            "or_row_system": (None, [C.c_int, P, P, P, P, P, P, C.c_int, P, P, i64, P, P, P]),
            "or_solve": (C.c_int, [C.c_int, P, P, f64, P]),
            "or_update_row": (C.c_int, [C.c_int, P, P, P, P, P, P, C.c_int, P, P, i64, f64]),
            "or_update_mode": (C.c_int, [C.c_int, P, P, P, P, P, P, C.c_int, P, P, f64, C.c_int]),
            "or_sse": (f64, [C.c_int, P, P, P, P, P, P, i64, C.c_int]),
            "or_loss": (f64, [C.c_int, P, P, P, P, P, P, i64, f64, C.c_int]),
            "or_thin_qr": (C.c_int, [i64, C.c_int, P, P]),
            "or_core_mode_product": (None, [C.c_int, P, P, C.c_int, P]),
            "or_orthogonalize": (C.c_int, [C.c_int, P, P, P, P, P]),
            "or_partial_errors": (None, [C.c_int, P, P, P, P, P, P, i64, P, P, C.c_int]),
            "or_truncate": (i64, [i64, P, P, P, f64]),
            "or_predict_many": (None, [C.c_int, P, P, P, P, P, i64, P]),
            "or_test_rmse": (f64, [C.c_int, P, P, P, P, P, P, i64]),
            "or_pres_init": (None, [C.c_int, P, P, P, P, P, i64, P, C.c_int]),
            "or_delta_cache": (None, [C.c_int, P, P, P, P, P, P, C.c_int, P]),
            "or_update_mode_cache": (C.c_int, [C.c_int, P, P, P, P, P, P, i64, C.c_int, P, P, f64, P, C.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


class Tensor:
    """Observed entries Omega (Table 2): 0-based int32 coords (nnz x N),
    FP64 values (FP32 inputs are widened exactly), dims I_1..I_N."""

    def __init__(self, coords, vals, dims):
        self.coords = np.ascontiguousarray(coords, dtype=np.int32)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.dims = np.ascontiguousarray(dims, dtype=np.int64)
        self.N = int(self.dims.size)
        self.nnz = int(self.vals.size)
        assert self.coords.shape == (self.nnz, self.N)
        self._index = {}

    def mode_index(self, n: int):
        """Stable per-mode CSR of Omega^(n)_{i_n}: (row_ptr[I_n+1], perm[nnz]), int64."""
        if n not in self._index:
            I = int(self.dims[n])
            row_ptr = np.zeros(I + 1, np.int64)
            perm = np.zeros(max(self.nnz, 1), np.int64)
            rc = lib().or_mode_index(self.N, self.nnz, _p(self.coords), _p(self.dims), n, _p(row_ptr), _p(perm))
            if rc:
                raise ValueError("coordinate out of range")
            self._index[n] = (row_ptr, perm[: self.nnz])
        return self._index[n]


class Model:
    """Core G (C-order, J_1 x ... x J_N) and factors A^(n) (I_n x J_n row-major), FP64."""

    def __init__(self, G, A):
        self.J = np.ascontiguousarray([a.shape[1] for a in A], dtype=np.int32)
        self.G = np.ascontiguousarray(G, dtype=np.float64).reshape(tuple(int(j) for j in self.J))
        self.A_all = np.ascontiguousarray(np.concatenate([np.asarray(a, np.float64).ravel() for a in A]))
        self.dims = np.ascontiguousarray([a.shape[0] for a in A], dtype=np.int64)
        self._off = np.concatenate([[0], np.cumsum(self.dims * self.J.astype(np.int64))])

    @property
    def N(self):
        return int(self.J.size)

    def A(self, n: int) -> np.ndarray:
        """View of A^(n) inside the flat buffer (writes go through)."""
        return self.A_all[self._off[n]: self._off[n + 1]].reshape(int(self.dims[n]), int(self.J[n]))

    @property
    def factors(self):
        return [self.A(n).copy() for n in range(self.N)]

    def copy(self) -> "Model":
        return Model(self.G.copy(), self.factors)


def init_model(dims, J, seed: int, prec: int) -> Model:
    """Alg. 2 line 1: G, A^(n) ~ U[0,1) from the counter RNG.
    prec=0 gives the values an FP32 library stores (exact in f32), prec=1 FP64."""
    dims = np.ascontiguousarray(dims, np.int64)
    J = np.ascontiguousarray(J, np.int32)
    G = np.zeros(int(np.prod(J)), np.float64)
    A_all = np.zeros(int(np.sum(dims * J)), np.float64)
    lib().or_init(len(dims), _p(dims), _p(J), seed, prec, _p(G), _p(A_all))
    A, off = [], 0
    for I, j in zip(dims, J):
        A.append(A_all[off: off + I * j].reshape(I, j))
        off += I * j
    return Model(G, A)


def rng_word(seed, stream, idx) -> int:
    return int(lib().or_rng_word(seed, stream, idx))


def mix64(z) -> int:
    return int(lib().or_mix64(z))


def uniform(seed, stream, idx, prec) -> float:
    return float(lib().or_uniform(seed, stream, idx, prec))


def delta(t: Tensor, m: Model, entry: int, n: int) -> np.ndarray:
    """Eq. 12 for entry `entry` (index into t) and mode n."""
    out = np.zeros(int(m.J[n]), np.float64)
    coord = np.ascontiguousarray(t.coords[entry])
    lib().or_delta(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(coord), n, _p(out))
    return out


def predict(m: Model, coord) -> float:
    """Eq. 4."""
    coord = np.ascontiguousarray(coord, np.int32)
    return float(lib().or_predict(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(coord)))


def row_system(t: Tensor, m: Model, n: int, row: int):
    """Eq. 10-11: B (J x J), c (J), sum x^2 over Omega^(n)_row."""
    row_ptr, perm = t.mode_index(n)
    Jn = int(m.J[n])
    B = np.zeros((Jn, Jn), np.float64)
    c = np.zeros(Jn, np.float64)
    s2 = np.zeros(1, np.float64)
    lib().or_row_system(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), _p(t.vals), n,
                        _p(row_ptr), _p(perm), row, _p(B), _p(c), _p(s2))
    return B, c, float(s2[0])


def solve(B, c, lam: float) -> np.ndarray:
    """Eq. 9: a = c [B + lambda I]^-1 (Cholesky)."""
    B = np.ascontiguousarray(B, np.float64)
    c = np.ascontiguousarray(c, np.float64)
    a = np.zeros(c.size, np.float64)
    rc = lib().or_solve(int(c.size), _p(B), _p(c), float(lam), _p(a))
    if rc:
        raise FloatingPointError("non-positive pivot")
    return a


def update_row(t: Tensor, m: Model, n: int, row: int, lam: float) -> None:
    row_ptr, perm = t.mode_index(n)
    rc = lib().or_update_row(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), _p(t.vals), n,
                             _p(row_ptr), _p(perm), row, float(lam))
    if rc:
        raise FloatingPointError("non-positive pivot")


def update_mode(t: Tensor, m: Model, n: int, lam: float, threads: int = 0) -> None:
    """Alg. 3 lines 6-15 for every row of A^(n), in place."""
    row_ptr, perm = t.mode_index(n)
    rc = lib().or_update_mode(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), _p(t.vals), n,
                              _p(row_ptr), _p(perm), float(lam), int(threads))
    if rc:
        raise FloatingPointError("non-positive pivot")


def sse(t: Tensor, m: Model, threads: int = 0) -> float:
    """Squared Eq. 5."""
    return float(lib().or_sse(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), _p(t.vals),
                              t.nnz, int(threads)))


def error(t: Tensor, m: Model, threads: int = 0) -> float:
    """Eq. 5: sqrt of the SSE over Omega."""
    return float(np.sqrt(sse(t, m, threads)))


def loss(t: Tensor, m: Model, lam: float, threads: int = 0) -> float:
    """Eq. 6."""
    return float(lib().or_loss(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), _p(t.vals),
                               t.nnz, float(lam), int(threads)))


def thin_qr(A):
    """Eq. 7: Householder thin QR with diag(R) > 0."""
    Q = np.ascontiguousarray(A, np.float64).copy()
    I, Jn = Q.shape
    R = np.zeros((Jn, Jn), np.float64)
    rc = lib().or_thin_qr(I, Jn, _p(Q), _p(R))
    if rc == 1:
        raise ValueError("I < J")
    if rc == 2:
        raise FloatingPointError("rank deficient")
    return Q, R


def core_mode_product(G, n: int, R) -> np.ndarray:
    """Eq. 2 with U = R, as in Eq. 8."""
    G = np.ascontiguousarray(G, np.float64).copy()
    J = np.ascontiguousarray(G.shape, np.int32)
    R = np.ascontiguousarray(R, np.float64)
    lib().or_core_mode_product(len(J), _p(J), _p(G), n, _p(R))
    return G


def orthogonalize(m: Model):
    """Alg. 2 lines 8-11, in place; returns the R^(n)."""
    R_all = np.zeros(int(np.sum(m.J.astype(np.int64) ** 2)), np.float64)
    rc = lib().or_orthogonalize(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(R_all))
    if rc == 1:
        raise ValueError("I < J")
    if rc == 2:
        raise FloatingPointError("rank deficient")
    Rs, off = [], 0
    for j in m.J:
        Rs.append(R_all[off: off + j * j].reshape(j, j))
        off += j * j
    return Rs


def partition(row_ptr, world: int) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    b = np.zeros(world + 1, np.int64)
    lib().or_partition(_p(row_ptr), row_ptr.size - 1, int(world), _p(b))
    return b


def als(t: Tensor, m: Model, lam: float, iters: int, threads: int = 0):
    """Alg. 2 lines 2-4: `iters` sweeps of Alg. 3 over n = 1..N
    (ascending), error Eq. 5 after each sweep.  Returns (errors, losses)
    with index 0 = the state before the first sweep (reading R10)."""
    errs = [error(t, m, threads)]
    losses = [loss(t, m, lam, threads)]
    for _ in range(iters):
        for n in range(m.N):
            update_mode(t, m, n, lam, threads)
        errs.append(error(t, m, threads))
        losses.append(loss(t, m, lam, threads))
    return np.array(errs), np.array(losses)


# ---------------------------------------------------------------------- P-Tucker-Approx
def partial_errors(t: Tensor, m: Model, present=None, threads: int = 0) -> np.ndarray:
    """Eq. 13 for every core entry (C order); 0 for absent entries."""
    gsize = int(np.prod(m.J))
    pres = np.ones(gsize, np.uint8) if present is None else np.ascontiguousarray(present, np.uint8)
    R = np.zeros(gsize, np.float64)
    lib().or_partial_errors(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), _p(t.vals), t.nnz,
                            _p(pres), _p(R), int(threads))
    return R


def truncate(m: Model, R, present, p: float) -> int:
    """Alg. 4 lines 3-4: zero the top floor(p|G|) present entries of G by R
    (descending, ties by ascending index; at least one entry stays).  `present` (uint8,
    C order) and m.G are updated in place.  Returns the number removed."""
    assert present.dtype == np.uint8 and present.flags["C_CONTIGUOUS"]
    R = np.ascontiguousarray(R, np.float64)
    G = m.G.reshape(-1)
    k = int(lib().or_truncate(G.size, _p(G), _p(present), _p(R), float(p)))
    return k


def truncate_core(t: Tensor, m: Model, present, p: float, threads: int = 0):
    """Alg. 4: scores, then truncation.  Returns (R, removed)."""
    R = partial_errors(t, m, present, threads)
    return R, truncate(m, R, present, p)


# ---------------------------------------------------------------------- prediction, test RMSE, Alg. 2 driver
def predict_many(m: Model, coords) -> np.ndarray:
    """Eq. 4 for query coordinates (n x N)."""
    coords = np.ascontiguousarray(coords, np.int32)
    out = np.zeros(coords.shape[0], np.float64)
    lib().or_predict_many(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(coords), coords.shape[0], _p(out))
    return out


def test_rmse(m: Model, coords, vals) -> float:
    """Held-out RMSE (§4.4)."""
    coords = np.ascontiguousarray(coords, np.int32)
    vals = np.ascontiguousarray(vals, np.float64)
    assert coords.shape[0] >= 1
    return float(lib().or_test_rmse(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(coords), _p(vals),
                                    coords.shape[0]))


def converged(e_prev: float, e: float, tol: float, xnorm: float) -> bool:
    """Alg. 2 line 2 "until ... ||X - X'|| converges", reading R30: the relative
    change of the error falls below tol, |e_t - e_(t-1)| < tol * e_(t-1), or the fit is
    already within tol of the data scale, e_t <= tol * ||x||."""
    return abs(e - e_prev) < tol * e_prev or e <= tol * xnorm


def run(t: Tensor, m: Model, lam: float, max_iters: int, tol: float, approx_p: float = 0.0,
        orthogonalize: bool = True, threads: int = 0):
    """Alg. 2: e_0 = error; repeat {update A^(1..N) (line 3); e_t = error (line 4);
    if Approx: truncate the core (lines 5-6)} until t = max_iters or
    |e_t - e_(t-1)| < tol * e_(t-1) or e_t <= tol ||x|| (reading R30); then QR + core update
    (lines 8-11).  Returns (errors e_0..e_T, T, present mask)."""
    present = np.ones(int(np.prod(m.J)), np.uint8)
    xnorm = float(np.sqrt(t.vals @ t.vals))
    errs = [error(t, m, threads)]
    it = 0
    while it < max_iters:
        for n in range(m.N):
            update_mode(t, m, n, lam, threads)
        e = error(t, m, threads)
        it += 1
        errs.append(e)
        if approx_p > 0:
            truncate_core(t, m, present, approx_p, threads)
        if converged(errs[-2], e, tol, xnorm):
            break
    if orthogonalize:
        globals()["orthogonalize"](m)
        present[:] = 1
    return np.array(errs), it, present


# ---------------------------------------------------------------------- P-Tucker-Cache
def pres_init(t: Tensor, m: Model, threads: int = 0) -> np.ndarray:
    """Alg. 3 lines 1-4: Pres[alpha][beta] = G_beta prod_k a^(k)_{i_k j_k},
    |Omega| x |G| (beta in C order)."""
    gsize = int(np.prod(m.J))
    pres = np.zeros((t.nnz, gsize), np.float64)
    lib().or_pres_init(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), t.nnz, _p(pres), int(threads))
    return pres


def delta_cache(t: Tensor, m: Model, pres, entry: int, n: int) -> np.ndarray:
    """Alg. 3 line 12: delta of one entry for mode n from its cache row."""
    out = np.zeros(int(m.J[n]), np.float64)
    coord = np.ascontiguousarray(t.coords[entry])
    row = np.ascontiguousarray(pres[entry])
    lib().or_delta_cache(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(coord), _p(row), n, _p(out))
    return out


def update_mode_cache(t: Tensor, m: Model, pres, n: int, lam: float, threads: int = 0) -> None:
    """Alg. 3 lines 6-19, TOP branch: every row of A^(n) from the cached
    products, then Pres rescaled by a_new / a_old (in place, both m and pres)."""
    assert pres.flags["C_CONTIGUOUS"] and pres.dtype == np.float64
    row_ptr, perm = t.mode_index(n)
    rc = lib().or_update_mode_cache(m.N, _p(m.J), _p(m.G), _p(m.A_all), _p(m.dims), _p(t.coords), _p(t.vals),
                                    t.nnz, n, _p(row_ptr), _p(perm), float(lam), _p(pres), int(threads))
    if rc:
        raise FloatingPointError("non-positive pivot")
