"""Host logic of bench.py (no GPU): the weak-scaling workload, the production
schedule (bandit.cpp:609-640) and the launch accounting."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_weak_scaling_config(bench):
    c4 = bench.CONFIGS["c4"]
    assert bench.scaled_cfg(c4, 1) is c4
    for n in (2, 4, 8):
        c = bench.scaled_cfg(c4, n)
        # per-GPU work fixed: one C4 shard and one C4 batch per GPU
        assert c["capacity"] == n * c4["capacity"] and c["batch"] == n * c4["batch"]
        assert c["capacity"] // n == 16384 and c["batch"] // n == 4096
        assert (c["lmax"], c["group"], c["loss"]) == (c4["lmax"], c4["group"], c4["loss"])
        assert c["name"].startswith(f"C4 per GPU x {n}")


def test_schedule_matches_reference_debt(bench):
    c4 = bench.CONFIGS["c4"]
    warm, per_step = bench.schedule(c4, 50)
    assert warm == 16384 // 16
    per = bench.W_WORKERS * c4["batch"] / (bench.MU * bench.T_TRAINERS)
    # whole groups, debt carried: the running total never drifts by a group
    total = 0
    for i, n in enumerate(per_step):
        total += n * 16
        assert abs(total - per * (i + 1)) < 16
    # weak scaling multiplies the production N-fold
    _, per8 = bench.schedule(bench.scaled_cfg(c4, 8), 50)
    assert abs(sum(per8) - 8 * sum(per_step)) <= 8  # each carries < 1 group of debt


def test_launch_accounting(bench):
    c4 = bench.CONFIGS["c4"]
    assert bench.launches_per_step(c4, 1) == 5
    assert bench.launches_per_step(bench.scaled_cfg(c4, 2), 2) == 6      # + finalize
    assert bench.launches_per_step(bench.scaled_cfg(c4, 4), 4) == 7      # + ring lookahead
    assert bench.launches_per_step(bench.CONFIGS["c2"], 1) == 6          # positive bias route


def test_documented_switches_exist():
    """Every environment switch INTEGRATION.md §5 documents is read by the library."""
    import re

    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    sec = doc[doc.index("## 5. Environment switches"):]
    names = set(re.findall(r"`(RB_[A-Z_]+)`", sec))
    src = "".join(open(os.path.join(ROOT, "paper_2604_08706_b200", "csrc", f)).read()
                  for f in ("buffer.cu", "loss.cu", "rng.cu"))
    assert names, "no switches documented"
    for n in names:
        assert f'"{n}"' in src, f"{n} documented but not read"
