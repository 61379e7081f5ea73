"""PCIe bandwidth of this box: pinned H2D and D2H alone, then both directions
at once on two copy streams (the e2e loss pipeline's assumption).

    python tools/pcie_probe.py [MB]
"""
import json
import sys

import torch


def _time(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / 1e3 / reps


def main():
    mb = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    n = mb << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        d_in.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_out, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            h2d()
        with torch.cuda.stream(s2):
            d2h()
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_h2d, t_d2h, t_both = _time(h2d), _time(d2h), _time(both)
    print(json.dumps({"bytes": n, "h2d_gbs": n / t_h2d / 1e9, "d2h_gbs": n / t_d2h / 1e9,
                      "duplex_gbs_each_way": n / t_both / 1e9}))


if __name__ == "__main__":
    main()
