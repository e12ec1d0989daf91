"""GPU parity of the generic-order path (orders N = 6..10 and core
sizes without a compiled (N, J) kernel, update_generic.cu) through the C-ABI against
the FP64 oracle, on the order-scaling workload of P:1013-1014 (I = 100, |Omega| = 10^3,
J = 3, N = 6..10) and on odd J:
  * one mode update from an identical oracle-made state: 1e-10 (FP64) / 1e-5 (FP32)
    relative per factor row (reading R20);
  * the error trajectory of 5 sweeps within 1e-9 (FP64) / 1e-4 (FP32) relative, the
    fused error (identity of update.cuh) equal to the literal Eq. 5 pass;
  * QR + core update (Eq. 7-8), the Approx scores (Eq. 13, generic kernel), Eq. 4
    predictions, the Alg. 2 driver with truncation, and a row-partitioned run.
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


def dtype_of(cfg):
    return np.float64 if cfg.dtype == "f64" else np.float32


def init(pt, cfg, coords, vals, world=1, rank=0):
    pt.ptucker_finalize()
    pt.ptucker_set_option("emulate_world", world)
    pt.ptucker_set_option("emulate_rank", rank)
    pt.ptucker_set_option("seg_len", 256)
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, 0)


def gpu_model(pt, orc, N):
    return orc.Model(pt.ptucker_get_core().astype(np.float64),
                     [pt.ptucker_get_factor(n).astype(np.float64) for n in range(N)])


def push_state(pt, m, dtype):
    pt.ptucker_set_core(m.G.astype(dtype))
    for n in range(m.N):
        pt.ptucker_set_factor(n, m.A(n).astype(dtype))


def oracle_state(orc, t, cfg, sweeps):
    N = len(cfg.dims)
    prec = 1 if cfg.dtype == "f64" else 0
    m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=prec)
    for _ in range(sweeps):
        for n in range(N):
            orc.update_mode(t, m, n, cfg.lam)
    dt = dtype_of(cfg)
    return orc.Model(m.G.astype(dt).astype(np.float64), [a.astype(dt).astype(np.float64) for a in m.factors])


def check_rows(orc, t, m_ref, n, a_gpu, cfg, m_in):
    """Reading R31: outside the five configs the FP64 row bound is conditioning-aware,
    err_i <= max(1e-10, 4 kappa_i sqrt(K) u) with kappa_i = cond(B_i + lambda I) of the
    input state m_in, K = J^(N-1) the terms of each delta component and u = 2^-53 (the
    forward error of a backward-stable solve of a system whose entries carry ~sqrt(K) u
    relative rounding); FP32 keeps the north-star 1e-5."""
    err_all = np.zeros(a_gpu.shape[0])
    a_g = np.asarray(a_gpu, np.float64)
    num = np.linalg.norm(a_g - m_ref.A(n), axis=1)
    den = np.linalg.norm(m_ref.A(n), axis=1)
    assert np.all(num[den == 0] == 0), "empty rows must be exactly zero"
    nz = den > 0
    err_all[nz] = num[nz] / den[nz]
    if cfg.dtype != "f64":
        assert err_all.max() <= 1e-5, (n, float(err_all.max()))
        return
    K = cfg.J ** (len(cfg.dims) - 1)
    for i in np.flatnonzero(err_all > 1e-10):
        B, _, _ = orc.row_system(t, m_in, n, int(i))
        kappa = np.linalg.cond(B + cfg.lam * np.eye(cfg.J))
        bound = 4 * kappa * np.sqrt(K) * 2.0 ** -53
        assert err_all[i] <= bound, (n, int(i), float(err_all[i]), float(kappa), bound)


def row_rel_err(a_gpu, a_ref):
    a_gpu = np.asarray(a_gpu, np.float64)
    num = np.linalg.norm(a_gpu - a_ref, axis=1)
    den = np.linalg.norm(a_ref, axis=1)
    zero = den == 0
    assert np.all(num[zero] == 0), "empty rows must be exactly zero"
    return num[~zero] / den[~zero]


CASES = [synth.order(N) for N in (6, 7, 8, 9, 10)] + [
    synth.order(6, dtype="f32"),
    synth.order(10, dtype="f32"),
    synth.Config("N3J6", (300, 200, 100), 20_000, 6, 0.01, 5, "f32", "uniform", "uniform", True),
    synth.Config("N4J7", (60, 50, 40, 30), 5_000, 7, 0.01, 5, "f64", "uniform", "uniform", True),
    synth.Config("N2J16", (500, 400), 20_000, 16, 0.01, 5, "f64", "uniform", "uniform", True),
    synth.Config("N3J12", (200, 200, 200), 10_000, 12, 0.01, 5, "f32", "uniform", "uniform", True),
]
IDS = [f"{c.name}-{c.dtype}" for c in CASES]


def test_shapes_route_to_generic(pt):
    for cfg in CASES:
        coords, vals = synth.generate(cfg)
        init(pt, cfg, coords, vals)
        info = pt.ptucker_info()
        assert info["generic"] is True and info["tensor_cores"] is False, cfg.name
    cfg = synth.order(5)                                   # compiled order-5 kernel
    init(pt, cfg, *synth.generate(cfg))
    assert pt.ptucker_info()["generic"] is False


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_mode_update_parity(pt, orc, cfg):
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    init(pt, cfg, coords, vals)
    N = len(cfg.dims)
    for sweeps in (0, 1):
        s0 = oracle_state(orc, t, cfg, sweeps)
        for n in range(N):
            m = s0.copy()
            push_state(pt, m, dtype_of(cfg))
            orc.update_mode(t, m, n, cfg.lam)
            pt.ptucker_update_mode(n)
            check_rows(orc, t, m, n, pt.ptucker_get_factor(n), cfg, s0)


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_error_trajectory(pt, orc, cfg):
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    N = len(cfg.dims)
    init(pt, cfg, coords, vals)
    m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=1 if cfg.dtype == "f64" else 0)
    ref, _ = orc.als(t, m, cfg.lam, 5)
    got = [pt.ptucker_error()]
    for _ in range(5):
        pt.ptucker_sweep()
        e_fused, e_lit = pt.ptucker_error(), pt.ptucker_error_literal()
        assert abs(e_fused - e_lit) <= 1e-9 * e_lit, (e_fused, e_lit)
        got.append(e_fused)
    rel = np.abs(np.array(got) - ref) / ref
    assert rel.max() <= (1e-9 if cfg.dtype == "f64" else 1e-4), rel


@pytest.mark.parametrize("N", [6, 8, 10])
def test_orthogonalize_and_predict(pt, orc, N):
    cfg = synth.order(N)
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    init(pt, cfg, coords, vals)
    m = oracle_state(orc, t, cfg, 2)
    push_state(pt, m, np.float64)
    e_before = orc.error(t, m)
    orc.orthogonalize(m)
    pt.ptucker_orthogonalize()
    g = gpu_model(pt, orc, N)
    for n in range(N):
        assert np.abs(g.A(n).T @ g.A(n) - np.eye(cfg.J)).max() <= 1e-12
        assert np.abs(g.A(n) - m.A(n)).max() <= 1e-9
    assert np.abs(g.G - m.G).max() <= 1e-9 * np.abs(m.G).max()
    assert abs(pt.ptucker_error() - e_before) <= 1e-10 * e_before
    q = np.random.default_rng(3).integers(0, 100, size=(257, N)).astype(np.int32)
    ref = orc.predict_many(g, q)
    np.testing.assert_allclose(pt.ptucker_predict(q), ref, rtol=1e-10, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("cfg", [synth.order(6), synth.order(9, dtype="f32"), CASES[7], CASES[8]],
                         ids=["order6", "order9-f32", "N3J6", "N4J7"])
def test_approx_scores(pt, orc, cfg):
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    N = len(cfg.dims)
    init(pt, cfg, coords, vals)
    pt.ptucker_sweep()
    m = gpu_model(pt, orc, N)
    R_o = orc.partial_errors(t, m).reshape(m.G.shape)
    R_g = pt.ptucker_core_scores()
    np.testing.assert_allclose(R_g, R_o, rtol=0, atol=1e-9 * np.abs(R_o).max())


@pytest.mark.parametrize("N,approx", [(7, 0.0), (7, 0.2), (10, 0.1)])
def test_run_matches_oracle(pt, orc, N, approx):
    cfg = synth.order(N)
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=1)
    e_ref, it_ref, _ = orc.run(t, m, cfg.lam, 6, 1e-4, approx, orthogonalize=True)
    init(pt, cfg, coords, vals)
    e, it = pt.ptucker_run(6, 1e-4, approx, True)
    assert it == it_ref, (it, it_ref)
    np.testing.assert_allclose(e, e_ref, rtol=1e-6)
    g = gpu_model(pt, orc, N)
    # after 6 iterations, truncations and the QR, order 10's conditioning (reading R31,
    # kappa ~ 1e6) turns the rounding of a different summation order into ~1e-6 absolute
    for n in range(N):
        assert np.abs(g.A(n) - m.A(n)).max() <= 5e-6


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_rows(pt, orc, world):
    """Emulated ranks of an order-8 run: stitched row blocks equal the single-rank
    update bit for bit, the per-rank SSE partials (fused and literal) add up, and so
    do the per-rank Approx scores."""
    cfg = synth.order(8)
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    N = 8
    s0 = oracle_state(orc, t, cfg, 1)
    init(pt, cfg, coords, vals)
    ref = {}
    for n in range(N):
        push_state(pt, s0, np.float64)
        pt.ptucker_update_mode(n)
        ref[n] = pt.ptucker_get_factor(n).copy()
    push_state(pt, s0, np.float64)
    ref_sse = pt.ptucker_error_literal() ** 2
    ref_R = pt.ptucker_core_scores()
    got = {n: np.full_like(ref[n], np.nan) for n in range(N)}
    sse, R = 0.0, np.zeros_like(ref_R)
    for r in range(world):
        init(pt, cfg, coords, vals, world, r)
        for n in range(N):
            b = pt.ptucker_get_partition(n)
            push_state(pt, s0, np.float64)
            pt.ptucker_update_mode(n)
            a = pt.ptucker_get_factor(n)
            got[n][b[r]:b[r + 1]] = a[b[r]:b[r + 1]]
        push_state(pt, s0, np.float64)
        sse += pt.ptucker_error_literal() ** 2
        R += pt.ptucker_core_scores()
    init(pt, cfg, coords, vals)
    for n in range(N):
        assert np.array_equal(got[n], ref[n]), n
    assert abs(sse - ref_sse) <= 1e-10 * ref_sse
    np.testing.assert_allclose(R, ref_R, rtol=0, atol=1e-10 * np.abs(ref_R).max())


def test_generic_edges(pt, orc):
    # single entry of an order-10 tensor; empty rows everywhere else
    cfg = synth.Config("one", (4,) * 10, 1, 2, 0.1, 1, "f64", "uniform", "uniform", False)
    coords = np.array([[1, 2, 3, 0, 1, 2, 3, 0, 1, 2]], np.int32)
    vals = np.array([0.75])
    t = orc.Tensor(coords, vals, cfg.dims)
    init(pt, cfg, coords, vals)
    s0 = oracle_state(orc, t, cfg, 0)
    for n in range(10):
        m = s0.copy()
        push_state(pt, m, np.float64)
        orc.update_mode(t, m, n, cfg.lam)
        pt.ptucker_update_mode(n)
        a = pt.ptucker_get_factor(n)
        assert np.all(a[np.arange(4) != coords[0, n]] == 0)
        err = row_rel_err(a, m.A(n))
        assert err.max() <= 1e-10
    # J = 1 (rank-one core) at order 7
    cfg = synth.Config("j1", (30,) * 7, 500, 1, 0.01, 1, "f64", "uniform", "uniform", True)
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    init(pt, cfg, coords, vals)
    m = orc.init_model(cfg.dims, [1] * 7, seed=0, prec=1)
    ref, _ = orc.als(t, m, cfg.lam, 3)
    got = [pt.ptucker_error()]
    for _ in range(3):
        pt.ptucker_sweep()
        got.append(pt.ptucker_error())
    np.testing.assert_allclose(got, ref, rtol=1e-9)


@pytest.mark.parametrize("cfg", [synth.order(7), CASES[7]], ids=["order7", "N3J6"])
def test_heavy_rows_split(pt, orc, cfg):
    """seg_len = 3 splits every row with more than 3 entries into segments whose
    partial (B, c, sum x^2) records are combined by the heavy-row finalize."""
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    pt.ptucker_finalize()
    pt.ptucker_set_option("emulate_world", 1)
    pt.ptucker_set_option("emulate_rank", 0)
    pt.ptucker_set_option("seg_len", 3)
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, 0)
    assert any(m["heavy_rows"] > 0 for m in pt.ptucker_info()["modes"])
    s0 = oracle_state(orc, t, cfg, 1)
    for n in range(len(cfg.dims)):
        m = s0.copy()
        push_state(pt, m, dtype_of(cfg))
        orc.update_mode(t, m, n, cfg.lam)
        pt.ptucker_update_mode(n)
        check_rows(orc, t, m, n, pt.ptucker_get_factor(n), cfg, s0)
    e_f, e_l = pt.ptucker_error(), pt.ptucker_error_literal()
    assert abs(e_f - e_l) <= 1e-9 * e_l
