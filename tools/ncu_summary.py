"""Key metrics from an ncu --set full report (raw page)."""
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "sm__maximum_warps_per_active_cycle_pct",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]


def metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2] if len(r) > 2 else r[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6}
    res = {}
    for w in WANT:
        if w in h:
            i = h.index(w)
            unit = u[i] if i < len(u) else ""
            try:
                res[w] = float(v[i].replace(",", "")) * scale.get(unit, 1)
            except ValueError:
                res[w] = v[i]
    stalls = {n.split("smsp__average_warps_issue_stalled_")[1].split("_per")[0]: v[i]
              for i, n in enumerate(h)
              if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")}
    top = sorted(((float(x or 0), k) for k, x in stalls.items()), reverse=True)[:6]
    return res, top


if __name__ == "__main__":
    # values are normalised to bytes / nanoseconds
    for rep in sys.argv[1:]:
        res, top = metrics(rep)
        print(rep)
        for k, x in res.items():
            print(f"   {k:60s} {x}")
        print("   top stalls (warps per issue):", ", ".join(f"{k}={x:.2f}" for x, k in top))
