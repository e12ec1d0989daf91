"""P-Tucker-Cache (Alg. 3 TOP branch) through the C-ABI
(option "cache") against the oracle's Cache implementation (oracle.update_mode_cache,
pinned in test_oracle_pins.test_cache_variant) and against plain P-Tucker:
  * one mode update from an identical state: 1e-10 (FP64) / 1e-5 (FP32) per row;
  * 4 sweeps: the error trajectory of the Cache variant = P-Tucker's (the same ALS);
  * a zero factor value (the P:639 fallback), orders up to 10 (the order-scaling shapes
    of P:1070, Fig. 8), unequal J_n, multi-segment rows, QR / truncation rebuilding Pres.
"""
import numpy as np
import pytest

from gen import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pt():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    torch.cuda.set_device(0)
    from paper_1710_02261_b200 import build, ptucker
    build.build()
    ptucker.load()
    yield ptucker
    ptucker.ptucker_finalize()
    ptucker.ptucker_set_option("cache", 0)


def init(pt, coords, vals, dims, J, lam, seg=256):
    pt.ptucker_finalize()
    pt.ptucker_set_option("seg_len", seg)
    pt.ptucker_set_option("cache", 1)
    try:
        pt.ptucker_init(coords, vals, dims, list(J), lam, 0)
    finally:
        pt.ptucker_set_option("cache", 0)   # the option is read at init; later inits are plain
    assert pt.ptucker_info()["cache"]


def rel_rows(a_gpu, a_ref):
    num = np.linalg.norm(np.asarray(a_gpu, np.float64) - a_ref, axis=1)
    den = np.linalg.norm(a_ref, axis=1)
    assert np.all(num[den == 0] == 0)
    return num[den > 0] / den[den > 0]


CASES = [
    ("c1", None, 256),
    ("c1", None, 8),
    ("c2@0.005", None, 256),
    ("order6", None, 256),
    ("order10", None, 256),
    ("mixed", (3, 2, 4, 2), 3),
]


def workload(name, J):
    if name.startswith("order"):
        cfg = synth.order(int(name[5:]))
        coords, vals = synth.generate(cfg)
        return coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, cfg.dtype
    if name == "mixed":
        rng = np.random.default_rng(3)
        dims = (16, 12, 10, 9)
        coords = np.stack([rng.integers(0, d, 1500) for d in dims], 1).astype(np.int32)
        return coords, rng.random(1500), dims, list(J), 0.02, "f64"
    base, _, sc = name.partition("@")
    cfg = synth.config(base) if not sc else synth.small(base, float(sc))
    coords, vals = synth.generate(cfg)
    return coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, cfg.dtype


@pytest.mark.parametrize("name,J,seg", CASES)
def test_cache_mode_updates_and_trajectory(pt, orc, name, J, seg):
    coords, vals, dims, Js, lam, dtype = workload(name, J)
    N = len(dims)
    prec = 1 if dtype == "f64" else 0
    dt = np.float64 if prec else np.float32
    # FP64: 1e-10 on the compiled-size shapes; the order-scaling shapes (K = J^(N-1) terms per
    # delta component, kappa up to ~1e6) take reading R31's conditioning-aware bound, of which
    # 2e-9 is a small fraction (4 kappa sqrt(K) u ~ 6e-8 at order 10)
    tol = (1e-10 if N <= 5 else 2e-9) if prec else 1e-5
    init(pt, coords, vals, dims, Js, lam, seg)
    t = orc.Tensor(coords, vals, dims)
    # the same ALS on both sides, mode by mode: oracle Cache from its own init, rows compared
    m = orc.init_model(dims, Js, seed=0, prec=prec)
    pres = orc.pres_init(t, m)
    m_plain = m.copy()
    worst = 0.0
    for sweep in range(2):
        for n in range(N):
            orc.update_mode_cache(t, m, pres, n, lam)
            orc.update_mode(t, m_plain, n, lam)
            pt.ptucker_update_mode(n)
            a = pt.ptucker_get_factor(n)
            err = rel_rows(a, m.A(n))
            worst = max(worst, float(err.max()))
            assert err.max() <= tol, (name, sweep, n, float(err.max()))
            # Cache and P-Tucker are the same update (the oracle's two implementations)
            assert rel_rows(m.A(n), m_plain.A(n)).max() <= tol
            # every side continues from the GPU's stored state: each mode is compared from an
            # identical state (reading R20), the tables rebuilt from it
            m.A(n)[:] = a.astype(np.float64)
            m_plain.A(n)[:] = a.astype(np.float64)
            pres[:] = orc.pres_init(t, m)
    e_gpu = pt.ptucker_error_literal()
    e_ref = orc.error(t, m)   # the same (GPU-synced) state: Eq. 5 on both sides
    assert abs(e_gpu - e_ref) <= 1e-9 * e_ref
    print(f"{name}: worst row rel err over 2 sweeps {worst:.2e}; error {e_gpu:.6g}")


def test_cache_zero_factor_and_rebuilds(pt, orc):
    """A factor value of exactly 0 (line 12 takes the product loop, lines 16-19 recompute,
    P:639), then QR and truncation (the table is rebuilt from the new state)."""
    cfg = synth.config("c1")
    coords, vals = synth.generate(cfg)
    init(pt, coords, vals, cfg.dims, [cfg.J] * 3, cfg.lam)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * 3, seed=0, prec=1)
    A1 = m.A(1)
    A1[coords[:40, 1], 2] = 0.0            # zeros under the first 40 entries' mode-1 rows
    pt.ptucker_set_factor(1, A1)
    pres = orc.pres_init(t, m)
    for n in range(3):
        orc.update_mode_cache(t, m, pres, n, cfg.lam)
        pt.ptucker_update_mode(n)
        assert rel_rows(pt.ptucker_get_factor(n), m.A(n)).max() <= 1e-10, n
    pt.ptucker_truncate_core(0.2)
    pt.ptucker_orthogonalize()
    g = orc.Model(pt.ptucker_get_core().astype(np.float64), [pt.ptucker_get_factor(n) for n in range(3)])
    ref = g.copy()
    pres = orc.pres_init(t, ref)
    orc.update_mode_cache(t, ref, pres, 0, cfg.lam)
    pt.ptucker_update_mode(0)
    assert rel_rows(pt.ptucker_get_factor(0), ref.A(0)).max() <= 1e-10


def test_cache_too_large(pt):
    from paper_1710_02261_b200.ptucker import PTuckerError
    cfg = synth.config("c5")
    coords, vals = synth.generate(synth.small("c5", 0.01))   # 10^6 entries x 1000 x 8 B = 8 GB: fits
    pt.ptucker_finalize()
    pt.ptucker_set_option("cache", 1)
    try:
        with pytest.raises(PTuckerError) as e:
            big = np.repeat(coords, 40, axis=0)             # 4e7 x 1000 x 8 B = 320 GB: does not
            pt.ptucker_init(big, np.repeat(vals, 40), synth.small("c5", 0.01).dims, [10] * 3, 0.01, 0)
        assert e.value.code == 3   # PTUCKER_ERESOURCE
    finally:
        pt.ptucker_set_option("cache", 0)
        pt.ptucker_finalize()
    del cfg
