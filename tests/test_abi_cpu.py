"""C-ABI checks that need no GPU: the library loads, exports every symbol that
include/ptucker.h declares, and its pure host logic (row partition, argument
validation) behaves; compute calls are never made here."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def pt():
    from paper_1710_02261_b200 import build, ptucker
    build.build()
    ptucker.load()
    return ptucker


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ptucker.h")).read()
    return sorted(set(re.findall(r"\b(ptucker_\w+)\s*\(", src)))


def test_exports_every_header_symbol(pt):
    lib = pt.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(pt.EXPORTS)
    assert pt.ptucker_version() >= 100


def test_partition_rows_matches_oracle(pt, orc):
    rng = np.random.default_rng(0)
    for trial in range(30):
        I = int(rng.integers(1, 200))
        lens = rng.integers(0, 50, I) * (rng.random(I) < 0.9)
        if trial % 5 == 0:
            lens[rng.integers(0, I)] = 5000  # a Zipf-like head row
        row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        for W in (1, 2, 3, 4, 8):
            assert np.array_equal(pt.ptucker_partition_rows(row_ptr, W), orc.partition(row_ptr, W))


def test_validation_without_gpu(pt):
    # argument errors are detected on the host before any device work
    c = np.zeros((4, 3), np.int32)
    v = np.ones(4, np.float32)
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_init(c, v, [2, 2, 2], [2, 2, 2], 0.0, 0)      # lambda must be > 0
    assert e.value.code == pt.PTUCKER_EINVAL
    # coordinates and values are validated on the device (a GPU test checks EINVAL): without
    # a GPU the call fails in the device setup instead
    with pytest.raises(pt.PTuckerError):
        pt.ptucker_init(c + 5, v, [2, 2, 2], [2, 2, 2], 0.1, 0)  # coordinate out of range
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_init(c, v, [2, 2, 2], [17, 17, 17], 0.1, 0)   # J > 16 (no kernel at all)
    assert e.value.code == pt.PTUCKER_EINVAL
    c11 = np.zeros((4, 11), np.int32)
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_init(c11, v, [2] * 11, [2] * 11, 0.1, 0)      # N > 10
    assert e.value.code == pt.PTUCKER_EINVAL
    c8 = np.zeros((4, 8), np.int32)
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_init(c8, v, [2] * 8, [10] * 8, 0.1, 0)        # core 10^8 > 2^26 entries
    assert e.value.code == pt.PTUCKER_EINVAL
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_init(c, v, [2, 2, 2], [2, 17, 2], 0.1, 0)     # a J_n above 16 (unequal J_n are valid)
    assert e.value.code == pt.PTUCKER_EINVAL
    with pytest.raises(pt.PTuckerError):
        pt.ptucker_init(c, np.array([1, np.nan, 1, 1], np.float32), [2, 2, 2], [2, 2, 2], 0.1, 0)
    with pytest.raises(pt.PTuckerError) as e:
        pt.ptucker_update_mode(0)                                # before init
    assert e.value.code == pt.PTUCKER_ESTATE
    with pytest.raises(pt.PTuckerError):
        pt.ptucker_set_option("no_such_option", 1)
    pt.ptucker_set_option("time_kernels", 0)
