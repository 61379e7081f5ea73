"""Loss-kernel anatomy on a config (debug build): first/last CTA start/end,
CTA 0's loop and commit, the last CTA's fold, and per-launch time in a graph
of back-to-back launches (no events around each)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["REPLAY_B200_LIB"] = os.path.join(ROOT, "paper_2604_08706_b200", "libreplay_b200_clocks.so")
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2604_08706_b200 import _lib  # noqa: E402

cfg_name = os.environ.get("CFG", "c1")
args = bench.argparse.Namespace(steps=5, warmup=3, config=cfg_name, no_e2e=True, graph=False,
                                no_cpu_baseline=True)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    res, buf, wl, rng = bench.run_ours(args, 0, 1, None)
    cfg = bench.CONFIGS[cfg_name]
    pad = cfg["batch"] * cfg["lmax"] + 8
    lpn = torch.randn(pad, device="cuda").mul_(0.01).sub_(1.0)
    dl = torch.empty(pad, device="cuda")
    st = torch.zeros(5, dtype=torch.float64, device="cuda")
    f = lambda: buf.loss_grpo(lpn, dl, 0.2, 0.2, stats=st)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{cfg_name}: loss per launch in a graph of 20: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
    _lib.lib.rb_debug_timeline_loss.argtypes = [C.c_void_p, C.c_int]
    _lib.lib.rb_debug_phase_clocks_loss.argtypes = [C.c_void_p]
    tl = (C.c_ulonglong * 64)()
    _lib.check(_lib.lib.rb_debug_timeline_loss(tl, 1))
    f()
    torch.cuda.synchronize()
    _lib.check(_lib.lib.rb_debug_timeline_loss(tl, 0))
    ck = (C.c_longlong * 64)()
    _lib.check(_lib.lib.rb_debug_phase_clocks_loss(ck))
    t0 = tl[10]
    print(f"first CTA start 0, last CTA start {(tl[32 + 5] - t0) / 1e3:.2f} us, "
          f"last CTA loop end {(tl[11] - t0) / 1e3:.2f} us")
    for i, nm in [(0, "CTA0 start"), (1, "CTA0 loop done"), (2, "CTA0 commit done"),
                  (3, "last CTA fold start"), (4, "last CTA fold done")]:
        print(f"  {nm:22s} {(ck[i] - t0) / 1e3:8.2f} us")
