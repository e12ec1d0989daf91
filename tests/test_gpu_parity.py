"""GPU parity: the CUDA path (through the C-ABI) against the FP64 CPU oracle on
the same seeded inputs (north-star tolerances, BASELINE.json):
  * init, slice index (CSR/perm) and row partition bit-exact;
  * one mode update from an identical state within 1e-5 (FP32) / 1e-10 (FP64)
    relative per factor row (reading R20: ||a_gpu - a_ref|| / ||a_ref||, the
    reference computed in FP64 from the identical stored state; empty rows 0);
  * the error trajectory over the iterations within 1e-3 relative;
  * QR + core update against the oracle's Householder QR (Eq. 7-8).
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
    """The GPU's current state, read back (used only for checks of the GPU's own
    output, never as an oracle input)."""
    G = pt.ptucker_get_core().astype(np.float64)
    A = [pt.ptucker_get_factor(n).astype(np.float64) for n in range(N)]
    return orc.Model(G, A)


def push_state(pt, m, dtype):
    """Put an oracle-made state (already representable in `dtype`) into the library."""
    pt.ptucker_set_core(m.G.astype(dtype))
    for n in range(m.N):
        pt.ptucker_set_factor(n, m.A(n).astype(dtype))


def rounded(orc, m, dtype):
    """The oracle state rounded to the library's storage precision."""
    return orc.Model(m.G.astype(dtype).astype(np.float64), [a.astype(dtype).astype(np.float64) for a in m.factors])


def row_rel_err(a_gpu, a_ref):
    a_gpu = np.asarray(a_gpu, np.float64)
    num = np.linalg.norm(a_gpu - a_ref, axis=1)
    den = np.linalg.norm(a_ref, axis=1)
    zero = den == 0
    assert np.all(num[zero] == 0), "empty rows must be exactly zero"
    return num[~zero] / den[~zero]


def init_cfg(pt, cfg, policy=-1, seg_len=256):
    coords, vals = synth.generate(cfg)
    pt.ptucker_finalize()
    pt.ptucker_set_option("seg_len", seg_len)
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, 0)
    pt.ptucker_set_option("policy", policy)
    return coords, vals


def oracle_state(orc, t, cfg, sweeps):
    """Identical starting state made by the ORACLE: its own init (bit-identical to the
    library's, checked in test_init_and_index_bit_exact) plus `sweeps` FP64 sweeps,
    rounded to the storage precision."""
    N = len(cfg.dims)
    prec = 1 if cfg.dtype == "f64" else 0
    m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=prec)
    for _ in range(sweeps):
        for n in range(N):
            orc.update_mode(t, m, n, cfg.lam)
    return rounded(orc, m, np.float64 if prec else np.float32)


def mode_update_parity(pt, orc, t, cfg, tol, sweeps=0, modes=None):
    """For each mode n: the same oracle-made state goes into both sides, both update
    mode n once, the rows of A^(n) are compared (reading R20)."""
    N = len(cfg.dims)
    dtype = np.float64 if cfg.dtype == "f64" else np.float32
    s0 = oracle_state(orc, t, cfg, sweeps)
    worst = 0.0
    for n in (range(N) if modes is None else modes):
        m = s0.copy()
        push_state(pt, m, dtype)
        orc.update_mode(t, m, n, cfg.lam)
        pt.ptucker_update_mode(n)
        err = row_rel_err(pt.ptucker_get_factor(n), m.A(n))
        worst = max(worst, float(err.max()) if err.size else 0.0)
        assert err.size == 0 or err.max() <= tol, (n, float(err.max()), float(np.median(err)))
    return worst


# ---------------------------------------------------------------- init / index / partition
@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c2", 0.01), ("c3", 0.002)])
def test_init_and_index_bit_exact(pt, orc, name, scale):
    cfg = synth.config("c1") if scale == 1.0 else synth.small(name, scale)
    coords, vals = init_cfg(pt, cfg)
    N = len(cfg.dims)
    prec = 1 if cfg.dtype == "f64" else 0
    ref = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=prec)
    assert np.array_equal(pt.ptucker_get_core().astype(np.float64), ref.G)
    for n in range(N):
        assert np.array_equal(pt.ptucker_get_factor(n).astype(np.float64), ref.A(n))
    t = orc.Tensor(coords, vals, cfg.dims)
    for n in range(N):
        rp, perm = pt.ptucker_get_mode_index(n)
        orp, operm = t.mode_index(n)
        assert np.array_equal(rp, orp) and np.array_equal(perm, operm)
        assert np.array_equal(pt.ptucker_get_partition(n), orc.partition(orp, 1))


# ---------------------------------------------------------------- one mode update from an identical state
@pytest.mark.parametrize("seg", [256, -1])
def test_mode_update_f64_c1(pt, orc, seg):
    """c1 at full size; seg = -1 is the automatic S bench.py runs (8 for c1: every row is
    a multi-segment heavy row, reduced by the fused heavy-row finalize)."""
    cfg = synth.config("c1")
    coords, vals = init_cfg(pt, cfg, seg_len=seg)
    t = orc.Tensor(coords, vals, cfg.dims)
    mode_update_parity(pt, orc, t, cfg, 1e-10, sweeps=0)        # init state
    mode_update_parity(pt, orc, t, cfg, 1e-10, sweeps=2)        # mid-trajectory state
    if seg < 0:
        assert pt.ptucker_info()["seg_len"] == 8


# c3 at scale 0.005 (690 x 135 x 21 x 24) exercises both small-mode tables (kind 2 for
# modes 0/1, kind 1 for modes 2/3); 0.002 (276 x 54 x 21 x 24) the plain order-4 kernel
@pytest.mark.parametrize("name,scale,seg", [("c2", 0.01, 256), ("c3", 0.002, 256), ("c3", 0.005, 256),
                                            ("c3", 0.005, 7), ("c4", 0.001, 256), ("c5", 0.0001, 256),
                                            ("c2", 0.05, -1), ("c5", 0.0005, -1)])
def test_mode_update_f32(pt, orc, name, scale, seg):
    cfg = synth.small(name, scale)
    coords, vals = init_cfg(pt, cfg, seg_len=seg)
    N = len(cfg.dims)
    t = orc.Tensor(coords, vals, cfg.dims)
    w0 = mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=0)    # init state (worst case, survey E4)
    w1 = mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=1)    # mid-trajectory
    info = pt.ptucker_info()
    print(f"{name}@{scale} seg={seg} worst row rel err init {w0:.2e} mid {w1:.2e}; heavy rows "
          f"{[m['heavy_rows'] for m in info['modes']]}; smp {[m['smp'] for m in info['modes']]}")
    if name == "c3" and scale == 0.005:
        assert [m["smp"] for m in info["modes"]] == [2, 2, 1, 1]


@pytest.mark.parametrize("name,scale", [("c5", 0.001), ("c2", 0.01)])
def test_mode_update_l0_kahan(pt, orc, name, scale):
    """l0_group 0: level 0 in packed fp32 pairs with Kahan compensation (one rounding per
    product), held to the same 1e-5 per row (full size, all 3x10^6 c5 rows: 5.8e-6,
    profiles/r02/l0_group_row_errors_c5_full_kahan.txt)."""
    cfg = synth.small(name, scale)
    coords, vals = init_cfg(pt, cfg)
    pt.ptucker_set_option("l0_group", 0)
    t = orc.Tensor(coords, vals, cfg.dims)
    w0 = mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=0)
    w1 = mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=1)
    pt.ptucker_set_option("l0_group", 1)
    print(f"{name}@{scale} l0_group 0 worst row rel err init {w0:.2e} mid {w1:.2e}")


@pytest.mark.parametrize("policy,label", [(3, "F32-C2"), (-1, "F32-C2"), (2, "F32-C")])
@pytest.mark.parametrize("scale,seg", [(0.001, 256), (0.005, 256), (0.005, 7)])
def test_mode_update_c4_f32c2(pt, orc, scale, seg, policy, label):
    """Order 5: F32-C2 (policy 3, and the automatic choice for the c4 shape: the level next to
    the innermost in fp32, J^3 instead of J^4 fp32 -> fp64 conversions per entry, the outer
    ones in fp64) and F32-C (policy 2, every outer level in fp64) are both held to 1e-5 per
    row, at the init state (the worst case) and mid-trajectory."""
    cfg = synth.small("c4", scale)
    coords, vals = init_cfg(pt, cfg, policy=policy, seg_len=seg)
    assert pt.ptucker_info()["policy"] == label
    t = orc.Tensor(coords, vals, cfg.dims)
    w0 = mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=0)
    w1 = mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=1)
    print(f"c4@{scale} seg={seg} {label} worst row rel err init {w0:.2e} mid {w1:.2e}")


@pytest.mark.parametrize("tc_table", [0, 1])
def test_mode_update_c3_table_modes(pt, orc, tc_table):
    """Order-4 modes with one small other mode (c3 modes 2/3, SMP kind 1) on the ALU table
    kernel (tc_table 0) and on the tensor-core kernel in table mode (tc_table 1, the
    default: lanes in (i_s, length) order, core block swapped per class)."""
    cfg = synth.small("c3", 0.005)
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    pt.ptucker_finalize()
    pt.ptucker_set_option("seg_len", 256)
    pt.ptucker_set_option("tc_table", tc_table)
    try:
        pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * 4, cfg.lam, 0)
        info = pt.ptucker_info()
        assert [m["smp"] for m in info["modes"]] == [2, 2, 1, 1]
        assert [m["tc_table"] for m in info["modes"]] == [False, False, bool(tc_table), bool(tc_table)]
        mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=0, modes=[2, 3])
        mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=1, modes=[2, 3])
        if tc_table:
            # the gathers of the skewed modes go through L1 (rows_l1 automatic = 1 here);
            # the L2-only path must give the same rows bit for bit
            s0 = oracle_state(orc, t, cfg, 1)
            got = {}
            for l1 in (1, 0):
                pt.ptucker_set_option("rows_l1", l1)
                push_state(pt, s0, np.float32)
                pt.ptucker_update_mode(2)
                got[l1] = pt.ptucker_get_factor(2).copy()
            pt.ptucker_set_option("rows_l1", -1)
            assert np.array_equal(got[0], got[1])
    finally:
        pt.ptucker_finalize()
        pt.ptucker_set_option("tc_table", 1)


@pytest.mark.parametrize("name,scale", [("c2", 0.01), ("c5", 0.0005)])
def test_mode_update_tc_packed_gathers(pt, orc, name, scale):
    """J = 10 tensor-core updates with the packed 32 + 8-byte gather tables (option
    pack_gathers): same rows as the oracle within 1e-5, and bit-identical to the
    unpacked gathers (the same values reach the same arithmetic)."""
    cfg = synth.small(name, scale)
    coords, vals = init_cfg(pt, cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    pt.ptucker_set_option("pack_gathers", 1)
    try:
        mode_update_parity(pt, orc, t, cfg, 1e-5, sweeps=1)
        s0 = oracle_state(orc, t, cfg, 1)
        got = {}
        for pk in (0, 1):
            pt.ptucker_set_option("pack_gathers", pk)
            push_state(pt, s0, np.float32)
            pt.ptucker_update_mode(1)
            got[pk] = pt.ptucker_get_factor(1).copy()
        assert np.array_equal(got[0], got[1])
    finally:
        pt.ptucker_set_option("pack_gathers", 0)


@pytest.mark.parametrize("name,scale", [("c2", 0.01), ("c4", 0.001)])
def test_mode_update_f64_variants(pt, orc, name, scale):
    """Every config also runs in FP64 mode (1e-10 per row)."""
    cfg = synth.small(name, scale)
    cfg.dtype = "f64"
    coords, vals = init_cfg(pt, cfg)
    assert vals.dtype == np.float64
    t = orc.Tensor(coords, vals, cfg.dims)
    mode_update_parity(pt, orc, t, cfg, 1e-10)


@pytest.mark.parametrize("name,scale,policy", [("c2", 0.01, 0), ("c3", 0.002, 0), ("c3", 0.002, 1),
                                               ("c4", 0.001, 0), ("c4", 0.001, 2)])
def test_policies_reported(pt, orc, name, scale, policy):
    """The non-default precision policies are measured, not assumed: their worst row
    error is printed (the automatic policy is the one held to 1e-5 above)."""
    cfg = synth.small(name, scale)
    coords, vals = init_cfg(pt, cfg, policy=policy)
    t = orc.Tensor(coords, vals, cfg.dims)
    w = mode_update_parity(pt, orc, t, cfg, 1e-4)
    print(f"{name} policy {pt.ptucker_info()['policy']}: worst row rel err {w:.2e}")


# ---------------------------------------------------------------- error (Eq. 5) and trajectory
@pytest.mark.parametrize("name,scale,iters", [("c1", 1.0, 5), ("c2", 0.01, 10), ("c3", 0.001, 10),
                                              ("c4", 0.001, 10), ("c5", 0.001, 10)])
def test_error_trajectory(pt, orc, name, scale, iters):
    cfg = synth.config(name) if scale == 1.0 else synth.small(name, scale)
    coords, vals = init_cfg(pt, cfg)
    N = len(cfg.dims)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=1 if cfg.dtype == "f64" else 0)
    ref_errs, _ = orc.als(t, m, cfg.lam, iters)
    gpu = [pt.ptucker_error()]                                   # literal pass (no update yet)
    for _ in range(iters):
        pt.ptucker_sweep()
        e_fused = pt.ptucker_error()
        e_lit = pt.ptucker_error_literal()
        assert abs(e_fused - e_lit) <= 1e-6 * e_lit, (e_fused, e_lit)
        gpu.append(e_fused)
    rel = np.abs(np.array(gpu) - ref_errs) / ref_errs
    assert rel.max() <= 1e-3, rel
    print(f"{name}: trajectory max rel diff {rel.max():.2e}; e {ref_errs[0]:.4g} -> {ref_errs[-1]:.4g}")


def test_error_of_identical_state(pt, orc):
    cfg = synth.small("c4", 0.001)
    coords, vals = init_cfg(pt, cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = oracle_state(orc, t, cfg, 1)
    push_state(pt, m, np.float32)
    ref = orc.error(t, m)
    assert abs(pt.ptucker_error() - ref) <= 1e-5 * ref            # literal pass (state was set)
    assert abs(pt.ptucker_error_literal() - ref) <= 1e-5 * ref


# ---------------------------------------------------------------- QR + core update (Eq. 7-8)
@pytest.mark.parametrize("name,scale,tol", [("c1", 1.0, 1e-10), ("c2", 0.01, 2e-5), ("c4", 0.001, 2e-5)])
def test_orthogonalize(pt, orc, name, scale, tol):
    cfg = synth.config(name) if scale == 1.0 else synth.small(name, scale)
    coords, vals = init_cfg(pt, cfg)
    N = len(cfg.dims)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = oracle_state(orc, t, cfg, 2)
    dtype = np.float64 if cfg.dtype == "f64" else np.float32
    push_state(pt, m, dtype)
    e_before = orc.error(t, m)
    orc.orthogonalize(m)
    pt.ptucker_orthogonalize()
    g = gpu_model(pt, orc, N)
    for n in range(N):
        Q = g.A(n)
        assert np.abs(Q.T @ Q - np.eye(cfg.J)).max() <= (1e-12 if tol < 1e-6 else 1e-5)
        assert np.abs(Q - m.A(n)).max() <= tol * max(1.0, np.abs(m.A(n)).max()) * 10
    assert np.abs(g.G - m.G).max() <= tol * np.abs(m.G).max()
    assert abs(pt.ptucker_error() - e_before) <= tol * e_before


# ---------------------------------------------------------------- edge cases
def test_edge_empty_rows_and_tiny(pt, orc):
    coords = np.array([[0, 0, 0], [0, 1, 1], [3, 1, 0]], np.int32)
    vals = np.array([1.0, 2.0, 3.0])
    pt.ptucker_finalize()
    pt.ptucker_set_option("seg_len", 256)
    pt.ptucker_init(coords, vals, [5, 2, 2], [2, 2, 2], 0.01, 0)
    t = orc.Tensor(coords, vals, [5, 2, 2])
    tiny = synth.Config("tiny", (5, 2, 2), 3, 2, 0.01, 1, "f64", "uniform", "uniform", False)
    mode_update_parity(pt, orc, t, tiny, 1e-10)
    pt.ptucker_update_mode(0)
    a0 = pt.ptucker_get_factor(0)
    assert np.all(a0[[1, 2, 4]] == 0) and np.all(a0[[0, 3]] != 0)
    # single entry, N = 2 (matrix case)
    pt.ptucker_init(np.array([[1, 2]], np.int32), np.array([0.5]), [3, 4], [3, 3], 0.1, 1)
    t = orc.Tensor([[1, 2]], [0.5], [3, 4])
    tiny2 = synth.Config("tiny2", (3, 4), 1, 3, 0.1, 1, "f64", "uniform", "uniform", False, seed=1)
    mode_update_parity(pt, orc, t, tiny2, 1e-10)


def test_worked_example(pt, orc):
    import json, os
    ex = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example_e10.json")))
    pt.ptucker_finalize()
    pt.ptucker_init(np.array(ex["coords"], np.int32), np.array(ex["vals"]), ex["dims"], ex["J"], ex["lambda"], 0)
    assert abs(pt.ptucker_error() - ex["e0"]) < 1e-12
    pt.ptucker_update_mode(0)
    np.testing.assert_allclose(pt.ptucker_get_factor(0), ex["A0_after_first_mode_update"], rtol=1e-12)
    pt.ptucker_update_mode(1)
    pt.ptucker_update_mode(2)
    assert abs(pt.ptucker_error() - ex["e1"]) < 1e-12
    pt.ptucker_sweep()
    assert abs(pt.ptucker_error() - ex["e2"]) < 1e-12


def test_determinism(pt):
    cfg = synth.small("c3", 0.005)
    init_cfg(pt, cfg, seg_len=16)
    pt.ptucker_sweep()
    a = [pt.ptucker_get_factor(n).copy() for n in range(4)]
    init_cfg(pt, cfg, seg_len=16)
    pt.ptucker_sweep()
    for n in range(4):
        assert np.array_equal(a[n], pt.ptucker_get_factor(n))


# ---------------------------------------------------------------- partitioned path (multi-GPU logic on one GPU)
@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_rows_bit_identical(pt, orc, world):
    """Each emulated rank builds and updates only its nnz-balanced row block of
    every mode (the exact code path of an N-GPU run minus the NCCL exchange);
    stitched together, the blocks equal the single-rank result bit for bit (rows
    are independent) and the per-rank SSE partials add up."""
    cfg = synth.small("c3", 0.005)
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    s0 = oracle_state(orc, t, cfg, 0)
    ref, ref_sse = {}, None
    pt.ptucker_finalize()
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * 4, cfg.lam, 0)
    for n in range(4):
        push_state(pt, s0, np.float32)
        pt.ptucker_update_mode(n)
        ref[n] = pt.ptucker_get_factor(n).copy()
    ref_sse = pt.ptucker_error() ** 2
    got = {n: np.full_like(ref[n], np.nan) for n in range(4)}
    sse = 0.0
    for r in range(world):
        pt.ptucker_finalize()
        pt.ptucker_set_option("emulate_world", world)
        pt.ptucker_set_option("emulate_rank", r)
        pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * 4, cfg.lam, 0)
        for n in range(4):
            b = pt.ptucker_get_partition(n)
            row_ptr, _ = t.mode_index(n)
            assert np.array_equal(b, orc.partition(row_ptr, world))
            push_state(pt, s0, np.float32)
            pt.ptucker_update_mode(n)
            got[n][b[r]:b[r + 1]] = pt.ptucker_get_factor(n)[b[r]:b[r + 1]]
        sse += pt.ptucker_error() ** 2
    pt.ptucker_finalize()
    for n in range(4):
        assert np.array_equal(got[n], ref[n]), n
    assert abs(sse - ref_sse) <= 1e-9 * ref_sse


@pytest.mark.parametrize("name,scale", [("c1", 1.0), ("c3", 0.005), ("c5", 0.0005)])
def test_graph_sweep_bit_identical(pt, orc, name, scale):
    """ptucker_sweep replays a captured CUDA graph of the sweep (option graph, default on):
    the same factors and errors bit for bit as direct launches, also across the events that
    drop the graph (an option change, Approx truncation, QR which swaps the core buffers)."""
    cfg = synth.config(name) if scale == 1.0 else synth.small(name, scale)
    N = len(cfg.dims)
    runs = {}
    for graph in (0, 1):
        init_cfg(pt, cfg, seg_len=-1)
        pt.ptucker_set_option("graph", graph)
        errs = []
        for it in range(4):
            pt.ptucker_sweep()
            errs.append(pt.ptucker_error())
            if it == 1:
                pt.ptucker_truncate_core(0.2)
            if it == 2:
                pt.ptucker_set_option("l0_group", 1)     # an option change drops the graph
        pt.ptucker_orthogonalize()
        pt.ptucker_sweep()
        errs.append(pt.ptucker_error())
        runs[graph] = ([pt.ptucker_get_factor(n).copy() for n in range(N)], pt.ptucker_get_core().copy(), errs)
    pt.ptucker_set_option("graph", 1)
    for n in range(N):
        assert np.array_equal(runs[0][0][n], runs[1][0][n]), n
    assert np.array_equal(runs[0][1], runs[1][1])
    assert runs[0][2] == runs[1][2]


def test_invalid_data_keeps_context(pt, orc):
    """ptucker_init validates the COO on the device before releasing the previous context:
    an out-of-range coordinate or a non-finite value is EINVAL naming the first offending
    entry (and mode), and the previous context keeps working."""
    cfg = synth.small("c2", 0.01)
    coords, vals = init_cfg(pt, cfg)
    pt.ptucker_sweep()
    e0 = pt.ptucker_error()
    bad = coords.copy()
    bad[123, 1] = cfg.dims[1]          # entry 123, mode 1 out of range
    bad[456, 0] = -1
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_init(bad, vals, cfg.dims, [cfg.J] * 3, cfg.lam, 0)
    assert e.value.code == pt.PTUCKER_EINVAL and "coordinate 1 of entry 123" in str(e.value)
    badv = vals.copy()
    badv[77] = np.inf
    badv[900] = np.nan
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_init(coords, badv, cfg.dims, [cfg.J] * 3, cfg.lam, 0)
    assert e.value.code == pt.PTUCKER_EINVAL and "entry 77" in str(e.value)
    assert pt.ptucker_error() == e0            # the previous context is intact
    pt.ptucker_sweep()


@pytest.mark.parametrize("name,scale,seg", [("c1", 1.0, 8), ("c2", 0.01, 7), ("c3", 0.002, 64), ("c5", 0.0005, 7),
                                            ("c4", 0.0005, 5)])
def test_inline_heavy_rows_bit_identical(pt, orc, name, scale, seg):
    """Heavy rows (2..64 segments) solved inside the update kernel by the lane that stores the
    row's last partial (option fin_inline; off by default: slower) give the same factors, core and errors bit
    for bit as the separate finalize launch: the same additions in the same order, the same
    solve.  The finalize launch count shows which path ran."""
    cfg = synth.config(name) if scale == 1.0 else synth.small(name, scale)
    N = len(cfg.dims)
    runs = {}
    for inline in (0, 1):
        init_cfg(pt, cfg, seg_len=seg)
        pt.ptucker_set_option("fin_inline", inline)
        pt.ptucker_set_option("time_kernels", 1)
        pt.ptucker_reset_kernel_stats()
        errs = []
        for it in range(3):
            pt.ptucker_sweep()
            errs.append(pt.ptucker_error())
        _, nfin = pt.ptucker_kernel_stats("finalize")
        pt.ptucker_set_option("time_kernels", 0)
        runs[inline] = ([pt.ptucker_get_factor(n).copy() for n in range(N)], errs, nfin)
    pt.ptucker_set_option("fin_inline", 0)
    for n in range(N):
        assert np.array_equal(runs[0][0][n], runs[1][0][n]), n
    assert runs[0][1] == runs[1][1]
    assert runs[0][2] > 0                    # the finalize launch ran without the option
    assert runs[1][2] < runs[0][2]           # and (at least some modes) not with it
    # and the inline run is still the ALS of the oracle: the error trajectory
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=1 if cfg.dtype == "f64" else 0)
    for it in range(3):
        for n in range(N):
            orc.update_mode(t, m, n, cfg.lam)
        e = orc.error(t, m)
        assert abs(runs[1][1][it] - e) <= 1e-3 * e, (it, runs[1][1][it], e)


@pytest.mark.gpu
@pytest.mark.parametrize("name,scale,seg", [("c2", 0.05, -1), ("c5", 0.0005, -1), ("c3", 0.002, -1), ("c1", 1.0, 8)])
def test_pdl_bit_identical(pt, orc, name, scale, seg):
    """Programmatic dependent launch (option pdl, off by default) only changes when the kernels of a
    sweep start, not what they compute: three graph-replayed sweeps with the error read back give
    the same factors and errors bit for bit with pdl = 0 and 1 (tensor-core kernel, table mode,
    heavy-row finalize, error sums), and the trajectory is the oracle's."""
    cfg = synth.config(name) if scale == 1.0 else synth.small(name, scale)
    N = len(cfg.dims)
    runs = {}
    for pdl in (0, 1):
        pt.ptucker_set_option("pdl", pdl)
        init_cfg(pt, cfg, seg_len=seg)
        errs = []
        for it in range(3):
            pt.ptucker_sweep()
            errs.append(pt.ptucker_error())
        runs[pdl] = ([pt.ptucker_get_factor(n).copy() for n in range(N)], errs)
    pt.ptucker_set_option("pdl", 0)
    for n in range(N):
        assert np.array_equal(runs[0][0][n], runs[1][0][n]), n
    assert runs[0][1] == runs[1][1]
    coords, vals = synth.generate(cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * N, seed=0, prec=1 if cfg.dtype == "f64" else 0)
    for it in range(3):
        for n in range(N):
            orc.update_mode(t, m, n, cfg.lam)
        e = orc.error(t, m)
        assert abs(runs[1][1][it] - e) <= 1e-3 * e, (it, runs[1][1][it], e)
