"""Per-call wall time of the e2e (host-buffer) replay step, C4."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

args = bench.argparse.Namespace(steps=8, warmup=3, config="c4", no_e2e=True, graph=False, weak=False)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    world = int(os.environ.get("EMU_WORLD", "1"))  # rank 0 of an emulated N-GPU job
    res, buf, wl, rng = bench.run_ours(args, 0, world, None)
    cfg = bench.scaled_cfg(bench.CONFIGS["c4"], world, getattr(args, "weak", False))
    B = cfg["batch"]
    hb = {k: v.cpu().pin_memory() for k, v in wl.steps[-1][0].items()}
    pad = B * cfg["lmax"] + 8
    tok_h = torch.empty(pad, dtype=torch.int32).pin_memory()
    off_h = torch.empty(B + 1, dtype=torch.int64).pin_memory()
    dl_h = torch.empty(pad, dtype=torch.float32).pin_memory()
    lpn_h = torch.randn(pad, dtype=torch.float32).mul_(0.01).sub_(1.0).pin_memory()
    shift = 10**12
    asy = os.environ.get("ASYNC") == "1"  # rb_set_async_outputs, no syncs between calls
    buf.set_async_outputs(asy)
    sync = (lambda: None) if asy else torch.cuda.synchronize
    for it in range(6):
        hb2 = dict(hb)
        hb2["rollout_id"] = (hb["rollout_id"] + shift * (it + 1)).pin_memory()
        t = [time.perf_counter()]
        buf.insert(**hb2, assume_unique=True)
        sync()
        t.append(time.perf_counter())
        buf.sample_device(B, rng)
        sync()
        t.append(time.perf_counter())
        buf.gather(tok_h, None, off_h)
        t.append(time.perf_counter())
        st = buf.loss_grpo(lpn_h, dl_h, 0.2, 0.2)
        _ = st.objective
        t.append(time.perf_counter())
        d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
        print("insert %.3f  sample %.3f  gather %.3f  loss %.3f  total %.3f ms" % (*d, sum(d)))
