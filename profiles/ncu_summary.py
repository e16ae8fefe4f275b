#!/usr/bin/env python3
"""Per-launch summary of an `ncu --page raw --csv` export: duration, tensor pipe, issue
activity, DRAM / L2 bytes, shared-memory bank conflicts and the top warp stall reasons.

  python profiles/ncu_summary.py raw.csv [--stalls 4]
"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "gpu__time_duration.sum" in r][0]
    return rows[hi], rows[hi + 1], rows[hi + 2:]


def main():
    path = sys.argv[1]
    nst = int(sys.argv[sys.argv.index("--stalls") + 1]) if "--stalls" in sys.argv else 4
    h, units, data = load(path)
    ix = {k: i for i, k in enumerate(h)}
    scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}

    def g(r, k):  # durations in us, byte counts in MB
        try:
            return float(r[ix[k]].replace(",", "")) * scale.get(units[ix[k]], 1.0)
        except (KeyError, ValueError):
            return float("nan")

    stall_keys = [k for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    cols = [("us", "gpu__time_duration.sum", 1), ("tc%", "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
            ("issue%", "sm__issue_active.avg.pct_of_peak_sustained_elapsed", 1),
            ("warps", "sm__warps_active.avg.per_cycle_active", 1),
            ("dramMB", None, 1), ("l2%", "lts__t_sectors.avg.pct_of_peak_sustained_elapsed", 1),
            ("bankc", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
            ("grid", "launch__grid_size", 1)]
    alt = {"sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed":
           "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"}
    print(" #  " + " ".join(f"{c:>8}" for c, _, _ in cols) + "  top stalls (warps per issue)")
    for n, r in enumerate(data):
        vals = []
        for c, k, s in cols:
            if c == "dramMB":
                v = g(r, "dram__bytes_read.sum") + g(r, "dram__bytes_write.sum")
            else:
                v = g(r, k)
                if v != v and k in alt:
                    v = g(r, alt[k])
                v *= s
            vals.append(v)
        st = sorted(((g(r, k), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for k in stall_keys), reverse=True)[:nst]
        print(f"{n:>2}  " + " ".join(f"{v:>8.1f}" for v in vals) + "  " + ", ".join(f"{k}={v:.2f}" for v, k in st))


if __name__ == "__main__":
    main()
