"""GPU parity of P-Tucker-Approx through the C-ABI against the FP64 oracle:
  * R(beta) of every core entry (Eq. 13) from an identical state: within 1e-9 of max |R|
    (both sides fp64 from the same stored values; only the summation order differs);
  * Alg. 4 truncation inside the ALS loop (Alg. 2 lines 3-6): the removed set of every
    iteration equals the oracle's (its scores computed from the GPU's state), |G| follows
    max(1, |G| - floor(p|G|)), the truncated entries are exactly zero;
  * scores of a row-partitioned run (emulated ranks) add up to the single-rank scores;
  * edge cases: invalid p, a core truncated down to one entry.
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


def gpu_model(pt, orc, N):
    G = pt.ptucker_get_core().astype(np.float64)
    A = [pt.ptucker_get_factor(n).astype(np.float64) for n in range(N)]
    return orc.Model(G, A)


def init(pt, cfg, **opts):
    coords, vals = synth.generate(cfg)
    pt.ptucker_finalize()
    for k, v in opts.items():
        pt.ptucker_set_option(k, v)
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, 0)
    return coords, vals


CASES = [("c1", 1.0), ("c2", 0.005), ("c3", 0.002), ("c4", 0.002)]


@pytest.mark.parametrize("name,scale", CASES)
def test_scores_match_oracle(pt, orc, name, scale):
    cfg = synth.small(name, scale) if scale < 1 else synth.config(name)
    coords, vals = init(pt, cfg)
    N = len(cfg.dims)
    t = orc.Tensor(coords, vals, cfg.dims)
    for sweeps in (0, 1):
        if sweeps:
            pt.ptucker_sweep()
        m = gpu_model(pt, orc, N)
        R_o = orc.partial_errors(t, m).reshape(m.G.shape)
        R_g = pt.ptucker_core_scores()
        scale_r = np.abs(R_o).max()
        np.testing.assert_allclose(R_g, R_o, rtol=0, atol=1e-9 * scale_r)


@pytest.mark.parametrize("name,scale,p", [("c1", 1.0, 0.2), ("c2", 0.005, 0.2), ("c4", 0.002, 0.3)])
def test_truncation_sequence(pt, orc, name, scale, p):
    cfg = synth.small(name, scale) if scale < 1 else synth.config(name)
    coords, vals = init(pt, cfg)
    N = len(cfg.dims)
    t = orc.Tensor(coords, vals, cfg.dims)
    gsize = cfg.J ** N
    present = np.ones(gsize, np.uint8)
    n_present = gsize
    for it in range(5):
        pt.ptucker_sweep()
        m = gpu_model(pt, orc, N)                     # the GPU's state, read back
        before = present.copy()
        R_o, k_o = orc.truncate_core(t, m, present, p)  # oracle truncation from that state
        k_g = pt.ptucker_truncate_core(p)
        G_g = pt.ptucker_get_core().astype(np.float64).reshape(-1)
        removed_g = set(np.flatnonzero((G_g == 0) & (before == 1)).tolist())
        removed_o = set(np.flatnonzero(before & ~present).tolist())
        assert k_g == k_o == min(int(np.floor(p * n_present)), n_present - 1)
        if removed_g != removed_o:
            # only admissible at an exact-in-rounding tie at the threshold
            diff = removed_g ^ removed_o
            thr = np.sort(R_o[before == 1])[::-1][k_o - 1]
            assert np.all(np.abs(R_o[list(diff)] - thr) <= 1e-9 * np.abs(R_o).max()), (it, diff)
        n_present -= k_g
        assert pt.ptucker_core_nnz() == n_present == int(present.sum())
        assert np.all(G_g[present == 0] == 0.0)
        # the error after truncation is the literal Eq. 5 of the truncated model
        e = pt.ptucker_error()
        e_ref = orc.error(t, gpu_model(pt, orc, N))
        assert abs(e - e_ref) <= 1e-6 * e_ref


def test_scores_add_over_ranks(pt, orc):
    """U and V are sums over entries, and R is linear in them: the scores of the
    row blocks of a 3-way partition of mode 0 add up to the single-rank scores."""
    cfg = synth.small("c2", 0.005)
    coords, vals = synth.generate(cfg)
    N = 3
    pt.ptucker_finalize()
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
    G, A = pt.ptucker_get_core(), [pt.ptucker_get_factor(n) for n in range(N)]
    R_full = pt.ptucker_core_scores()
    acc = np.zeros_like(R_full)
    for r in range(3):
        pt.ptucker_finalize()
        pt.ptucker_set_option("emulate_world", 3)
        pt.ptucker_set_option("emulate_rank", r)
        pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * N, cfg.lam, 0)
        pt.ptucker_set_core(G)
        for n in range(N):
            pt.ptucker_set_factor(n, A[n])
        acc += pt.ptucker_core_scores()
    pt.ptucker_finalize()
    pt.ptucker_set_option("emulate_world", 1)
    pt.ptucker_set_option("emulate_rank", 0)
    np.testing.assert_allclose(acc, R_full, rtol=0, atol=1e-10 * np.abs(R_full).max())


def test_truncation_edges(pt, orc):
    coords = np.array([[0, 0], [1, 2], [2, 1], [3, 3]], np.int32)
    vals = np.array([1.0, 0.5, 2.0, 1.5])
    pt.ptucker_finalize()
    pt.ptucker_init(coords, vals, [4, 4], [2, 2], 0.1, 0)
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_truncate_core(0.0)
    assert e.value.code == pt.PTUCKER_EINVAL
    with pytest.raises(pt.PTuckerError):
        pt.ptucker_truncate_core(1.0)
    counts = []
    for _ in range(6):
        pt.ptucker_truncate_core(0.5)
        counts.append(pt.ptucker_core_nnz())
    assert counts == [2, 1, 1, 1, 1, 1]              # 4 -> 2 -> 1, then never below one
    assert np.count_nonzero(pt.ptucker_get_core()) == 1
    pt.ptucker_sweep()                                # still a valid model
    assert np.isfinite(pt.ptucker_error())


def test_truncation_ties_lower_index_first(pt, orc):
    """Reading R28 on the device path: two core entries with bit-identical scores (equal
    G values, identical factor columns, so every term of U and V is the same) are removed
    lower C-order index first, as the oracle's stable sort does."""
    rng = np.random.default_rng(7)
    I0, I1, J = 40, 30, 3
    coords = np.stack([rng.integers(0, I0, 400), rng.integers(0, I1, 400)], 1).astype(np.int32)
    vals = rng.random(400)
    pt.ptucker_finalize()
    pt.ptucker_set_option("emulate_world", 1)
    pt.ptucker_set_option("emulate_rank", 0)
    pt.ptucker_init(coords, vals, [I0, I1], [J, J], 0.1, 0)
    A0 = rng.random((I0, J))
    col = rng.random(I1)
    A1 = np.stack([col, col, rng.random(I1)], 1)       # columns 0 and 1 identical
    G = rng.random((J, J))
    G[:, 1] = G[:, 0]                                  # beta = (j, 0) and (j, 1) tie for every j
    G *= 10.0                                          # make the tied pairs the top scores
    G[:, 2] = 0.01
    pt.ptucker_set_core(G)
    pt.ptucker_set_factor(0, A0)
    pt.ptucker_set_factor(1, A1)
    R = pt.ptucker_core_scores().reshape(-1)
    assert R[0] == R[1] and R[3] == R[4] and R[6] == R[7]
    t = orc.Tensor(coords, vals, [I0, I1])
    m = orc.Model(G.astype(np.float64).copy(), [A0.copy(), A1.copy()])
    present = np.ones(J * J, np.uint8)
    for p in (0.15, 0.2, 0.3):                         # removes 1 (a tie split), then 1, then 2
        before = present.copy()
        _, k_o = orc.truncate_core(t, m, present, p)
        k_g = pt.ptucker_truncate_core(p)
        assert k_g == k_o
        G_g = pt.ptucker_get_core().reshape(-1)
        removed_g = set(np.flatnonzero((G_g == 0) & (before == 1)).tolist())
        removed_o = set(np.flatnonzero(before & ~present).tolist())
        assert removed_g == removed_o, (p, removed_g, removed_o)
