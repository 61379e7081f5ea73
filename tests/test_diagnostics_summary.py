"""summarize_hist (the host half of the device replay diagnostics) against the
reference's own summarize() (metrics.cpp:185-202, through oracle/_ref): for
integer-valued metrics a histogram carries the same mean, nearest-rank
quartiles and histogram exactly."""
import numpy as np
import pytest

from paper_2604_08706_b200.replay import summarize_hist


@pytest.mark.parametrize("seed", range(6))
def test_summarize_hist_matches_reference(reference, seed):
    r = np.random.default_rng(seed)
    n = int(r.integers(1, 3000))
    top = int(r.integers(1, 40))
    vals = r.integers(0, top, n)
    if seed == 0:
        vals = np.array([7])
    hist = np.bincount(vals, minlength=64).astype(np.uint64)
    got = summarize_hist(hist, int(vals.sum()))
    want = reference.summarize(vals.astype(np.float64))
    assert got == want


def test_summarize_hist_empty():
    with pytest.raises(ValueError, match="at least one value"):
        summarize_hist(np.zeros(8, np.uint64))
