#!/usr/bin/env python3
"""Summarise ncu evidence into profiles/ (run here, on the CPU box).

  python profiles/summarize.py launches <launches.csv> <out.md>     # per-kernel launch list shares
  python profiles/summarize.py full <prof.ncu-rep> <out.md> [traffic.json]  # --set full metrics
  python profiles/summarize.py steady <launches.csv> <out.md> <traffic.json>  # time + DRAM per launch
"""
import collections
import csv
import io
import json
import subprocess
import sys


def short(name):
    """Bare kernel name with template args: 'k_gather<8, float, __half>' / 'cub::DeviceRadixSort...'."""
    n = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].replace("void ", "").strip()
    head = n.split("<")[0]
    base = head.split("::")[-1]
    if head.startswith("cub::"):
        base = "cub::" + base
    return (base + n[len(head):])[:70]


def launches(csv_path, out):
    rows = list(csv.reader(open(csv_path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    seq = [(short(r[ki]), float(r[vi].replace(",", ""))) for r in data if len(r) > vi]
    agg = collections.defaultdict(list)
    for n, v in seq:
        agg[n].append(v)
    total = sum(v for _, v in seq)
    lines = [f"# ncu launch list ({csv_path})", "",
             "gpu__time_duration.sum per launch, --clock-control none: cold-cache and serialised, so compare",
             "SHARES, not absolute times.", "",
             "| kernel | launches | mean us | total us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e3:.1f} | {sum(v) / total:.1%} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Achieved Occupancy",
        "Registers Per Thread", "Compute (SM) Throughput", "Grid Size", "Block Size", "Waves Per SM",
        "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tcgen05.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]


def full(rep, out, traffic_json=None):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(det)))
    h = rows[0]
    ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ii], short(r[ki]))
        if r[mi] in WANT:
            per.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    traffic = {}
    rawvals = {}
    for r in rr[2:]:
        if len(r) < len(rh):
            continue
        rid, kn = r[rh.index("ID")], short(r[rh.index("Kernel Name")])
        vals = {}
        for m in RAW:
            if m in rh:
                vals[m] = r[rh.index(m)]
        rawvals[(rid, kn)] = vals
        try:
            b = float(vals["dram__bytes_read.sum"].replace(",", "")) + float(vals["dram__bytes_write.sum"].replace(",", ""))
            unit = rr[1][rh.index("dram__bytes_read.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            base = kn.split("<")[0]  # matches the library's launch labels
            traffic.setdefault(base, []).append(b * scale)
        except Exception:
            pass
    lines = [f"# ncu --set full summary ({rep})", ""]
    for (rid, kn), d in per.items():
        lines.append(f"## [{rid}] {kn}")
        for k in WANT:
            if k in d:
                lines.append(f"- {k}: {d[k]}")
        for k, v in rawvals.get((rid, kn), {}).items():
            lines.append(f"- {k}: {v}")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json:
        json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif sys.argv[1] == "full":
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)


def steady(csv_path, out, traffic_json):
    """Launch list of one steady-state forward with gpu__time_duration + dram bytes per launch
    (--cache-control none): per-kernel share of device time and mean DRAM traffic per launch
    (the bench's roofline.traffic)."""
    rows = list(csv.reader(open(csv_path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3, "usecond": 1,
             "us": 1, "msecond": 1e3, "ms": 1e3}
    per = collections.OrderedDict()
    for r in data:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[ii], {"name": short(r[ki])})
        d[r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["name"].split("<")[0]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    total = sum(a[1] for a in agg.values())
    lines = [f"# steady-state launch list ({csv_path})", "",
             "One network forward after warm-up (AUTO dataflow decided), ncu --clock-control none",
             "--cache-control none (L2 warm across launches, as in the bench); times are serialised.", "",
             "| kernel | launches | total us | share | mean us | mean DRAM MB/launch |", "|---|---:|---:|---:|---:|---:|"]
    for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {t:.1f} | {t / total:.1%} | {t / n:.2f} | {b / n / 1e6:.2f} |")
    lines.append(f"| total | {sum(a[0] for a in agg.values())} | {total:.1f} | 100% | | |")
    open(out, "w").write("\n".join(lines) + "\n")
    tr = {}
    try:
        tr = json.load(open(traffic_json))
    except Exception:
        pass
    for k, (n, t, b) in agg.items():
        tr[k] = b / n
    json.dump(tr, open(traffic_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__" and sys.argv[1] == "steady":
    steady(sys.argv[2], sys.argv[3], sys.argv[4])
