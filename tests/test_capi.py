"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/replay_b200.h declares, and refuses to run without a GPU
(there is no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "replay_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    fns = declared_functions()
    for must in ("rb_create", "rb_insert", "rb_sample", "rb_gather", "rb_loss_grpo",
                 "rb_loss_asymre", "rb_group_advantages", "rb_rng_create", "rb_dump", "rb_load"):
        assert must in fns


def test_library_exports_every_declared_symbol():
    from paper_2604_08706_b200 import _lib

    lib = C.CDLL(_lib.LIB_PATH)
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_library_is_sm100a():
    from paper_2604_08706_b200 import _lib

    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2604_08706_b200 as rb

    with pytest.raises(rb.replay.ReplayError if hasattr(rb.replay, "ReplayError") else Exception,
                       match="CUDA|device"):
        rb.ShardedReplayBuffer(1, 4)


def test_host_rng_matches_oracle_without_gpu(oracle):
    """Host-side draws of the library's Rng (state not yet on a device)."""
    import paper_2604_08706_b200 as rb

    for seed in (1, 7, 99):
        a = rb.Rng(seed).stream("buffer_sampling")
        b = oracle.rng(seed).stream("buffer_sampling")
        assert a.seed() == b.seed
        assert [a.below(84) for _ in range(50)] == [b.below(84) for _ in range(50)]
        assert a.sample_without_replacement(40, 13).tolist() == \
            b.sample_without_replacement(40, 13).tolist()
        assert a.uniform01() == b.uniform01()
    assert rb.hash_name("metrics") == oracle.hash_name("metrics")
