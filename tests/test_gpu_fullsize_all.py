"""Full-size parity beyond sampled rows (VERDICT r01 "What's missing" 3, "What's weak" 1):

  * c2 at BASELINE.json's full size: the 10-iteration reconstruction-error trajectory
    (Alg. 2 lines 2-4) within 1e-3 of the FP64 oracle's;
  * c5 at full size (the bench workload): one mode update of EVERY mode compared on ALL
    10^6 rows (reading R20, 1e-5) at the init state and at a mid-trajectory state made by
    one FP64 oracle sweep (Eq. 9-12);
  * c3 at full size: the Zipf head rows of modes 0 and 1 (2.7M / 2.9M entries, the heavy
    multi-segment path), recomputed by the oracle's row system (Eq. 10-11) over chunks of
    the row's entries summed here in fp64.

Every expected value comes from oracle/ (its own init, bit-identical to the library's by
test_gpu_parity.test_init_and_index_bit_exact, its own slice index and its own sweeps).
"""
import concurrent.futures as cf
import os

import numpy as np
import pytest

from gen import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def pt():
    import torch
    assert torch.cuda.is_available()
    torch.cuda.set_device(0)
    from paper_1710_02261_b200 import build, ptucker
    build.build()
    ptucker.load()
    yield ptucker
    ptucker.ptucker_finalize()


def _init(pt, cfg):
    coords, vals = synth.generate(cfg)
    pt.ptucker_finalize()
    pt.ptucker_set_option("seg_len", -1)   # automatic, as bench.py runs it
    pt.ptucker_init(coords, vals, cfg.dims, [cfg.J] * len(cfg.dims), cfg.lam, cfg.seed)
    pt.ptucker_set_option("policy", -1)    # the automatic precision policy (what bench.py runs)
    return coords, vals


def _row_err(a_gpu, a_ref):
    num = np.linalg.norm(np.asarray(a_gpu, np.float64) - a_ref, axis=1)
    den = np.linalg.norm(a_ref, axis=1)
    assert np.all(num[den == 0] == 0), "empty rows must be exactly zero"
    return num[den > 0] / den[den > 0]


def test_c2_full_trajectory(pt, orc):
    cfg = synth.config("c2")
    coords, vals = _init(pt, cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * 3, seed=cfg.seed, prec=0)
    ref, _ = orc.als(t, m, cfg.lam, 10)
    gpu = [pt.ptucker_error()]
    for _ in range(10):
        pt.ptucker_sweep()
        gpu.append(pt.ptucker_error())
    rel = np.abs(np.array(gpu) - ref) / ref
    print(f"c2 full: trajectory max rel diff {rel.max():.2e}; e {ref[0]:.6g} -> {ref[-1]:.6g}")
    assert rel.max() <= 1e-3, rel


def test_c5_full_all_rows(pt, orc):
    cfg = synth.config("c5")
    coords, vals = _init(pt, cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m0 = orc.init_model(cfg.dims, [cfg.J] * 3, seed=cfg.seed, prec=0)
    report = []
    for state in ("init", "mid"):
        if state == "mid":   # one FP64 oracle sweep, rounded to the fp32 storage
            for n in range(3):
                orc.update_mode(t, m0, n, cfg.lam)
            m0 = orc.Model(m0.G.astype(np.float32).astype(np.float64),
                           [a.astype(np.float32).astype(np.float64) for a in m0.factors])
        for n in range(3):
            m = m0.copy()
            pt.ptucker_set_core(m.G.astype(np.float32))
            for k in range(3):
                pt.ptucker_set_factor(k, m.A(k).astype(np.float32))
            orc.update_mode(t, m, n, cfg.lam)
            pt.ptucker_update_mode(n)
            err = _row_err(pt.ptucker_get_factor(n), m.A(n))
            report.append(f"{state} mode {n}: max {err.max():.2e} p99.99 {np.quantile(err, 0.9999):.2e} "
                          f"median {np.median(err):.2e} over {err.size} rows")
            assert err.size == 10**6 and err.max() <= 1e-5, report[-1]
    print("c5 full, all rows: " + "; ".join(report))


def _row_system_chunked(orc, t, m, n, row, chunk=65536):
    """B, c of one (huge) row by the oracle's literal Eq. 10-11 pass over consecutive
    chunks of the row's entries (slice order), the chunk sums added in fp64."""
    row_ptr, perm = t.mode_index(n)
    p0, p1 = int(row_ptr[row]), int(row_ptr[row + 1])
    J = int(m.J[n])
    lib = orc.lib()

    def part(a):
        b = min(a + chunk, p1)
        rp = np.array([a, b], np.int64)
        B = np.zeros((J, J))
        c = np.zeros(J)
        s2 = np.zeros(1)
        lib.or_row_system(m.N, orc._p(m.J), orc._p(m.G), orc._p(m.A_all), orc._p(m.dims), orc._p(t.coords),
                          orc._p(t.vals), n, orc._p(rp), orc._p(perm), 0, orc._p(B), orc._p(c), orc._p(s2))
        return B, c

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        parts = list(ex.map(part, range(p0, p1, chunk)))
    return sum(p[0] for p in parts), sum(p[1] for p in parts), p1 - p0


def test_c3_full_head_rows(pt, orc):
    cfg = synth.config("c3")
    coords, vals = _init(pt, cfg)
    t = orc.Tensor(coords, vals, cfg.dims)
    m = orc.init_model(cfg.dims, [cfg.J] * 4, seed=cfg.seed, prec=0)
    out = []
    for n in (0, 1):
        if n:
            pt.ptucker_set_factor(n - 1, m.A(n - 1).astype(np.float32))
        pt.ptucker_update_mode(n)
        a_gpu = pt.ptucker_get_factor(n).astype(np.float64)
        row_ptr, _ = t.mode_index(n)
        lens = np.diff(row_ptr)
        for row in np.argsort(-lens, kind="stable")[:2]:
            B, c, ln = _row_system_chunked(orc, t, m, n, int(row))
            a = orc.solve(B, c, cfg.lam)
            err = np.linalg.norm(a_gpu[row] - a) / np.linalg.norm(a)
            out.append(f"mode {n} row {row} ({ln} entries): {err:.2e}")
            assert ln >= 10**6 and err <= 1e-5, out[-1]
    print("c3 full head rows: " + "; ".join(out))
