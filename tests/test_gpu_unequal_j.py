"""Unequal core dimensionality J_1..J_N (Alg. 2's input "core tensor dimensionality
J_1, ..., J_N") through the C-ABI against the FP64 oracle,
which takes per-mode J everywhere:
  * init (G of J_1 x ... x J_N, A^(n) of I_n x J_n) bit-exact;
  * one mode update from an identical oracle-made state: 1e-10 (FP64) / 1e-5 (FP32)
    relative per factor row (reading R20), with and without multi-segment (heavy) rows;
  * 5 sweeps: error trajectory, fused = literal Eq. 5;
  * QR + core update (Eq. 7-8), Eq. 4 predictions and the Approx scores (Eq. 13).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [  # (dims, J, nnz, dtype)
    ((40, 30, 20), (2, 3, 4), 3000, "f64"),
    ((40, 30, 20), (4, 2, 3), 3000, "f32"),
    ((16, 12, 10, 9), (3, 2, 4, 2), 2500, "f64"),
    ((12, 10, 9, 8, 7), (2, 3, 2, 3, 2), 2000, "f64"),
    ((30, 25, 20), (10, 5, 8), 4000, "f64"),
]


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


def make(dims, nnz, dtype, seed=5):
    rng = np.random.default_rng(seed)
    coords = np.stack([rng.integers(0, d, nnz) for d in dims], 1).astype(np.int32)
    vals = rng.random(nnz).astype(np.float64 if dtype == "f64" else np.float32)
    return coords, vals


def init(pt, dims, J, coords, vals, seg=256):
    pt.ptucker_finalize()
    pt.ptucker_set_option("seg_len", seg)
    pt.ptucker_init(coords, vals, dims, list(J), 0.01, 0)


def rel_rows(a_gpu, a_ref):
    num = np.linalg.norm(np.asarray(a_gpu, np.float64) - a_ref, axis=1)
    den = np.linalg.norm(a_ref, axis=1)
    assert np.all(num[den == 0] == 0)
    return num[den > 0] / den[den > 0]


@pytest.mark.parametrize("dims,J,nnz,dtype", SHAPES)
@pytest.mark.parametrize("seg", [256, 3])
def test_unequal_j_mode_updates(pt, orc, dims, J, nnz, dtype, seg):
    coords, vals = make(dims, nnz, dtype)
    init(pt, dims, J, coords, vals, seg)
    info = pt.ptucker_info()
    assert info["core_dims"] == list(J) and info["generic"]
    prec = 1 if dtype == "f64" else 0
    dt = np.float64 if prec else np.float32
    ref = orc.init_model(dims, list(J), seed=0, prec=prec)
    assert np.array_equal(pt.ptucker_get_core().astype(np.float64), ref.G)
    for n in range(len(dims)):
        assert np.array_equal(pt.ptucker_get_factor(n).astype(np.float64), ref.A(n))
    t = orc.Tensor(coords, vals, dims)
    for sweeps in (0, 1):
        s0 = orc.init_model(dims, list(J), seed=0, prec=prec)
        for _ in range(sweeps):
            for n in range(len(dims)):
                orc.update_mode(t, s0, n, 0.01)
        s0 = orc.Model(s0.G.astype(dt).astype(np.float64), [a.astype(dt).astype(np.float64) for a in s0.factors])
        for n in range(len(dims)):
            m = s0.copy()
            pt.ptucker_set_core(m.G.astype(dt))
            for k in range(len(dims)):
                pt.ptucker_set_factor(k, m.A(k).astype(dt))
            orc.update_mode(t, m, n, 0.01)
            pt.ptucker_update_mode(n)
            err = rel_rows(pt.ptucker_get_factor(n), m.A(n))
            assert err.max() <= (1e-10 if prec else 1e-5), (dims, J, n, sweeps, float(err.max()))


@pytest.mark.parametrize("dims,J,nnz,dtype", SHAPES)
def test_unequal_j_trajectory_qr_predict_scores(pt, orc, dims, J, nnz, dtype):
    coords, vals = make(dims, nnz, dtype)
    init(pt, dims, J, coords, vals)
    N = len(dims)
    prec = 1 if dtype == "f64" else 0
    t = orc.Tensor(coords, vals, dims)
    m = orc.init_model(dims, list(J), seed=0, prec=prec)
    ref, _ = orc.als(t, m, 0.01, 5)
    gpu = [pt.ptucker_error()]
    for _ in range(5):
        pt.ptucker_sweep()
        e = pt.ptucker_error()
        el = pt.ptucker_error_literal()
        assert abs(e - el) <= 1e-9 * el
        gpu.append(e)
    rel = np.abs(np.array(gpu) - ref) / ref
    assert rel.max() <= (1e-9 if prec else 1e-4), rel
    # Eq. 4 predictions and Eq. 13 scores on the GPU's own state, the oracle from the same state
    g = orc.Model(pt.ptucker_get_core().astype(np.float64), [pt.ptucker_get_factor(n).astype(np.float64)
                                                              for n in range(N)])
    q = coords[:200]
    np.testing.assert_allclose(pt.ptucker_predict(q), orc.predict_many(g, q), rtol=1e-9, atol=1e-9)
    R = pt.ptucker_core_scores()
    R_ref = orc.partial_errors(t, g).reshape(J)
    assert np.abs(R - R_ref).max() <= 1e-9 * np.abs(R_ref).max()
    # QR + core update: Q^T Q = I per mode, predictions unchanged
    before = orc.predict_many(g, q)
    pt.ptucker_orthogonalize()
    g2 = orc.Model(pt.ptucker_get_core().astype(np.float64), [pt.ptucker_get_factor(n).astype(np.float64)
                                                               for n in range(N)])
    for n in range(N):
        Q = g2.A(n)
        assert np.abs(Q.T @ Q - np.eye(J[n])).max() <= (1e-12 if prec else 1e-5)
    np.testing.assert_allclose(orc.predict_many(g2, q), before, rtol=1e-8 if prec else 1e-4,
                               atol=1e-8 if prec else 1e-4)
    mo = g.copy()
    orc.orthogonalize(mo)
    np.testing.assert_allclose(g2.G, mo.G, rtol=0, atol=(1e-9 if prec else 1e-3) * np.abs(mo.G).max())


def test_unequal_j_invalid(pt):
    from paper_1710_02261_b200.ptucker import PTuckerError
    coords, vals = make((5, 5, 5), 10, "f64")
    pt.ptucker_finalize()
    with pytest.raises(PTuckerError):
        pt.ptucker_init(coords, vals, (5, 5, 5), [2, 17, 3], 0.01, 0)   # J_n > 16
    with pytest.raises(PTuckerError):
        pt.ptucker_init(coords, vals, (5, 5, 5), [2, 0, 3], 0.01, 0)
