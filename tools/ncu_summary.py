"""Key metrics of one-kernel `ncu --set full` captures: python tools/ncu_summary.py rep... [> out].
Time, DRAM bytes and bandwidth, SM / issue utilisation, occupancy, the top warp-stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]


def summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))
    out = [f"== {rep}", f"kernel: {d.get('Kernel Name')}"]
    for k in KEYS:
        if k in d:
            out.append(f"{k:62s} {d[k]:>16s} {u.get(k, '')}")
    st = {}
    for k in h:
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st[k[33:]] = float(d[k].replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    out.append("warp stalls: " + ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in
                                           sorted(st.items(), key=lambda x: -x[1])[:8]))
    return "\n".join(out)


if __name__ == "__main__":
    print("\n\n".join(summary(r) for r in sys.argv[1:]))
