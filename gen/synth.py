"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module is the ONLY code shared by the oracle side (tests/, bench.py's
cpu_baseline) and the CUDA side (tests/, bench.py, smoke): it draws the
observed entries Omega (coordinates and values) and holds none of P-Tucker's
arithmetic.  The method's own random numbers (the U[0,1) init of G and A^(n),
P:466) are NOT drawn here: the oracle and the library each implement the
counter-based init generator (reading R2).

Recipe per config:
  c1  N=3, 100^3, 10,000 DISTINCT coords uniform, values U[0,1) f64, J=5
  c2  N=3, 1e4^3, 1e6 coords uniform (deduplicated), values U[0,1) f32, J=10
  c3  N=4, 138000 x 27000 x 21 x 24 (MovieLens shape, PAPER Table 4),
      2e7 entries, modes 1/2 finite Zipf(1.1) with seeded ID permutations,
      modes 3/4 uniform, values uniform over {0.5, 1.0, ..., 5.0} (f32),
      duplicates kept (multiset, reading R14), J=10
  c4  N=5, 1e5^5, 1e7 coords uniform; values = planted rank-(5,...,5) Tucker
      model (orthonormal factors, N(0,1) core) rescaled to unit RMS (reading
      R17) + N(0, 0.01^2) noise, f32, J=5, lambda=0.001
  c5  N=3, 1e6^3, 1e8 coords uniform, values U[0,1) f32, J=10
The paper's synthetic tensors are "random tensors ... with real-valued entries
between 0 and 1" with uniform coordinates; c3 stands in for the
MovieLens dataset, which is not available (no network, no data files).
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class Config:
    name: str
    dims: tuple
    nnz: int
    J: int
    lam: float
    iters: int
    dtype: str          # "f32" | "f64"  (value/factor storage precision)
    values: str         # "uniform" | "ratings" | "planted"
    coords: str         # "uniform" | "zipf12"
    distinct: bool      # redraw duplicates (c1/c2) or keep (multiset)
    seed: int = 0


CONFIGS = {
    "c1": Config("c1", (100, 100, 100), 10_000, 5, 0.01, 5, "f64", "uniform", "uniform", True),
    "c2": Config("c2", (10_000,) * 3, 1_000_000, 10, 0.01, 10, "f32", "uniform", "uniform", True),
    "c3": Config("c3", (138_000, 27_000, 21, 24), 20_000_000, 10, 0.01, 10, "f32", "ratings", "zipf12", False),
    "c4": Config("c4", (100_000,) * 5, 10_000_000, 5, 0.001, 10, "f32", "planted", "uniform", False),
    "c5": Config("c5", (1_000_000,) * 3, 100_000_000, 10, 0.01, 10, "f32", "uniform", "uniform", False),
}


def config(name: str, **over) -> Config:
    return dataclasses.replace(CONFIGS[name], **over)


def _zipf_indices(rng: np.random.Generator, I: int, n: int, s: float = 1.1) -> np.ndarray:
    """Finite Zipf(s) over ranks 1..I by inverse-CDF sampling, rank k mapped to
    index pi(k-1) with pi a seeded permutation (reading R15)."""
    w = np.arange(1, I + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    perm = rng.permutation(I).astype(np.int32)
    out = np.empty(n, np.int32)
    step = 1 << 22
    for a in range(0, n, step):
        u = rng.random(min(step, n - a))
        r = np.searchsorted(cdf, u, side="right")
        np.minimum(r, I - 1, out=r)
        out[a:a + r.size] = perm[r]
    return out


def _uniform_coords(rng, dims, n) -> np.ndarray:
    c = np.empty((n, len(dims)), np.int32)
    for k, I in enumerate(dims):
        c[:, k] = rng.integers(0, I, size=n, dtype=np.int64).astype(np.int32)
    return c


def _dedupe_redraw(rng, dims, coords) -> np.ndarray:
    """Distinct coordinates: duplicates are redrawn in generation order."""
    mult = np.cumprod([1] + list(dims[::-1]))[:-1][::-1].astype(np.int64)  # C-order strides
    assert float(np.prod([float(d) for d in dims])) < 9.2e18
    while True:
        key = coords.astype(np.int64) @ mult
        _, first = np.unique(key, return_index=True)
        dup = np.ones(key.size, bool)
        dup[first] = False
        nd = int(dup.sum())
        if nd == 0:
            return coords
        coords[dup] = _uniform_coords(rng, dims, nd)


def _planted_values(rng, dims, J, coords, noise=0.01) -> np.ndarray:
    """c4: x0 = sum_beta G*_beta prod_n A*^(n)_{i_n j_n} with orthonormal A*
    (Q of a Gaussian matrix) and an N(0,1) core, rescaled to unit RMS, plus
    N(0, noise^2).  Evaluated with numpy einsum chains in chunks (reading R17)."""
    N = len(dims)
    A = [np.linalg.qr(rng.standard_normal((I, J)))[0] for I in dims]
    G = rng.standard_normal((J,) * N)
    x0 = np.empty(coords.shape[0], np.float64)
    step = 20_000
    for a in range(0, coords.shape[0], step):
        c = coords[a:a + step]
        T = np.einsum("ej,j...->e...", A[0][c[:, 0]], G)
        for k in range(1, N):
            T = np.einsum("ej,ej...->e...", A[k][c[:, k]], T)
        x0[a:a + step] = T
    scale = 1.0 / np.sqrt(np.mean(x0 ** 2))
    return x0 * scale + noise * rng.standard_normal(x0.size)


def generate(cfg: Config):
    """Returns (coords int32 [nnz, N] row-major 0-based, vals f32|f64 [nnz])."""
    rng = np.random.default_rng(cfg.seed)
    dims, n = cfg.dims, cfg.nnz
    if cfg.coords == "zipf12":
        coords = np.empty((n, len(dims)), np.int32)
        coords[:, 0] = _zipf_indices(rng, dims[0], n)
        coords[:, 1] = _zipf_indices(rng, dims[1], n)
        for k in range(2, len(dims)):
            coords[:, k] = rng.integers(0, dims[k], size=n, dtype=np.int64).astype(np.int32)
    else:
        coords = _uniform_coords(rng, dims, n)
    if cfg.distinct:
        coords = _dedupe_redraw(rng, dims, coords)
    vdt = np.float64 if cfg.dtype == "f64" else np.float32
    if cfg.values == "uniform":
        vals = rng.random(n, dtype=vdt)
    elif cfg.values == "ratings":
        vals = (0.5 * rng.integers(1, 11, size=n)).astype(vdt)
    elif cfg.values == "planted":
        vals = _planted_values(rng, dims, cfg.J, coords).astype(vdt)
    else:
        raise ValueError(cfg.values)
    return np.ascontiguousarray(coords), np.ascontiguousarray(vals)


def small(name: str, scale: float, seed: int = 0) -> Config:
    """A reduced copy of config `name` with |Omega| and I_n scaled down but the
    same order, rank, value recipe and (for c3) skew, for oracle-speed tests."""
    c = CONFIGS[name]
    dims = tuple(max(d if d <= 64 else int(d * scale), 2) for d in c.dims)
    return dataclasses.replace(c, dims=dims, nnz=max(int(c.nnz * scale), 1), seed=seed)


def order(N: int, J: int = 3, I: int = 100, nnz: int = 1000, dtype: str = "f64", seed: int = 0) -> Config:
    """The order-scaling workload of P:1013-1014 (Fig. 8b): N-way, I = 100 per mode,
    |Omega| = 10^3 uniform coordinates, values U[0,1), J = 3.  Coordinates are
    deduplicated while the C-order key fits int64 (I^N < 2^63), else kept as drawn (a
    collision among 10^3 draws from 100^10 cells has probability ~5e-15)."""
    distinct = N * np.log2(max(I, 2)) < 62
    return Config(f"order{N}", (I,) * N, nnz, J, 0.01, 5, dtype, "uniform", "uniform", bool(distinct), seed)
