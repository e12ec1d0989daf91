"""Input generators (gen/synth.py): shapes, ranges, determinism and the c3 skew."""
import numpy as np

from gen import synth


def test_c1_distinct_and_ranges():
    cfg = synth.config("c1")
    c, v = synth.generate(cfg)
    assert c.shape == (10_000, 3) and c.dtype == np.int32 and v.dtype == np.float64
    key = (c[:, 0].astype(np.int64) * 100 + c[:, 1]) * 100 + c[:, 2]
    assert np.unique(key).size == 10_000
    assert (c >= 0).all() and (c < 100).all() and (v >= 0).all() and (v < 1).all()
    c2, v2 = synth.generate(cfg)
    assert np.array_equal(c, c2) and np.array_equal(v, v2)


def test_c3_small_skew_and_values():
    cfg = synth.small("c3", 0.01)
    c, v = synth.generate(cfg)
    assert cfg.dims == (1380, 270, 21, 24) and c.shape == (200_000, 4)
    assert set(np.unique(v).tolist()) <= {0.5 * k for k in range(1, 11)}
    cnt = np.bincount(c[:, 0], minlength=1380)
    # finite Zipf(1.1): the head row holds ~1/H(1380) of the entries (H ~ 5.7)
    assert 0.12 < cnt.max() / c.shape[0] < 0.22
    assert (np.bincount(c[:, 2], minlength=21) > 0).all()


def test_c4_small_planted_unit_rms():
    cfg = synth.small("c4", 0.001)
    c, v = synth.generate(cfg)
    assert c.shape == (10_000, 5) and v.dtype == np.float32
    assert 0.8 < np.sqrt(np.mean(v.astype(np.float64) ** 2)) < 1.2
