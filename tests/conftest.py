import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu under gpurun)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle as o
    o.build()
    return o


# Library options live in the process-wide context and survive ptucker_finalize (they
# are the caller's settings): a test that changes one (policy, tc_table, cache, ...) must
# not leak it into the next test, so every test ends with the library finalized and its
# options back at the documented defaults (include/ptucker.h).
_OPTION_DEFAULTS = [("policy", -1), ("tc", 1), ("l0_group", 1), ("pack_gathers", 0), ("rows_l1", -1),
                    ("tc_table", 1), ("smp", 1), ("smp_table", 2), ("seg_len", -1), ("exchange", 1),
                    ("graph", 1), ("sparse_core", -1), ("cache", 0), ("time_kernels", 0),
                    ("emulate_world", 1), ("emulate_rank", 0), ("fin_inline", 0), ("pdl", 0)]


@pytest.fixture(autouse=True)
def _reset_library_options():
    yield
    mod = sys.modules.get("paper_1710_02261_b200.ptucker")
    if mod is None or getattr(mod, "_lib", None) is None:
        return
    try:
        mod.ptucker_finalize()
    except Exception:
        pass
    for k, v in _OPTION_DEFAULTS:
        try:
            mod.ptucker_set_option(k, v)
        except Exception:
            pass
