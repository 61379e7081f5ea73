"""Host logic of bench.py (no GPU): the strong/weak-scaling workloads, the production
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


def test_scaling_configs(bench):
    c4 = bench.CONFIGS["c4"]
    assert bench.scaled_cfg(c4, 1)["capacity"] == c4["capacity"]
    for n in (2, 4, 8):
        # default: strong scaling — BASELINE configs[3], the 16384 buffer and
        # B = 4096 split into n shards (one per GPU)
        c = bench.scaled_cfg(c4, n)
        assert (c["capacity"], c["batch"], c["scaling"]) == (16384, 4096, "strong")
        assert c["capacity"] % n == 0 and c["batch"] % n == 0
        assert c["name"].startswith(f"C4 over {n} GPUs")
        # --weak: one C4 shard and one C4 batch per GPU
        w = bench.scaled_cfg(c4, n, weak=True)
        assert w["capacity"] == n * c4["capacity"] and w["batch"] == n * c4["batch"]
        assert w["scaling"] == "weak" and w["name"].startswith(f"C4 per GPU x {n}")
        assert (w["lmax"], w["group"], w["loss"]) == (c4["lmax"], c4["group"], c4["loss"])
        # both arms print the same config object
        assert bench.config_dict(c, n) == bench.config_dict(dict(c), n)
        assert bench.config_dict(c, n)["shards"] == n


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
    _, per8 = bench.schedule(bench.scaled_cfg(c4, 8, weak=True), 50)
    assert abs(sum(per8) - 8 * sum(per_step)) <= 8  # each carries < 1 group of debt


def test_launch_accounting(bench):
    c4 = bench.CONFIGS["c4"]
    assert bench.launches_per_step(c4, 1) == 5
    assert bench.launches_per_step(bench.scaled_cfg(c4, 2), 2) == 6      # + finalize
    assert bench.launches_per_step(bench.scaled_cfg(c4, 4), 4) == 6      # strong: B stays 4096
    assert bench.launches_per_step(bench.scaled_cfg(c4, 4, weak=True), 4) == 7  # + ring lookahead
    assert bench.launches_per_step(bench.CONFIGS["c2"], 1) == 5          # positive bias: one route launch


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
