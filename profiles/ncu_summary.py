#!/usr/bin/env python
"""Summarise an ncu report (--set full) or a launch-list CSV into a small text
table committed under profiles/.

  python profiles/ncu_summary.py report gpurun_out/rN_prof.ncu-rep > profiles/rN_full.txt
  python profiles/ncu_summary.py launches gpurun_out/rN_launches.csv > profiles/rN_launches.txt
  python profiles/ncu_summary.py traffic gpurun_out/rN_prof.ncu-rep profiles/traffic_garden.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict

STAGE_OF = [("k_count", "count"), ("k_project", "project"), ("k_dup", "dup"), ("k_render_fwd", "render_fwd"),
            ("k_render_bwd", "render_bwd"), ("k_gauss_bwd", "gauss_bwd")]

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def _raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def _num(s):
    try:
        return float(s.replace(",", ""))
    except Exception:
        return None


def report(path):
    h, units, rows = _raw(path)
    print(f"# ncu --set full summary of {path}")
    for r in rows:
        name = r[h.index("Kernel Name")]
        print(f"\n## {name[:90]}")
        for m in METRICS:
            if m in h:
                print(f"  {m:70s} {r[h.index(m)]:>16s} {units[h.index(m)]}")
        st = []
        for i, c in enumerate(h):
            if c.startswith("smsp__pcsamp_warps_issue_stalled") and not c.endswith("not_issued"):
                v = _num(r[i])
                if v:
                    st.append((v, c.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        tot = sum(v for v, _ in st) or 1.0
        st.sort(reverse=True)
        print("  stalls: " + ", ".join(f"{c} {100 * v / tot:.0f}%" for v, c in st[:8]))


def _stage_of_sequence(names):
    """Stage of each launch of one step, from the launch order: count, scan, project; the pair
    sort (hist / scan / scatter passes) up to k_dup; dup (its scan and k_dup); the entry sort and
    ranges up to the forward; then the forward, backward and per-Gaussian kernels."""
    out, phase = [], "count"
    for nm in names:
        if nm.startswith("k_count"):
            phase = "count"
        elif nm.startswith("k_project"):
            phase = "project"
        elif phase == "project" and nm.startswith("k_rs_hist"):
            phase = "sort_pairs"
        elif nm.startswith("k_dup"):
            phase = "dup"
        elif phase == "dup" and not nm.startswith("k_dup"):
            phase = "sort_entries"
        elif nm.startswith("k_render_fwd"):
            phase = "render_fwd"
        elif nm.startswith("k_render_bwd"):
            phase = "render_bwd"
        elif nm.startswith("k_gauss_bwd"):
            phase = "gauss_bwd"
        if phase == "sort_pairs" and nm.startswith("k_scan_1p") and out and out[-1] == "sort_pairs" and \
                names[len(out) - 1].startswith("k_rs_scatter"):
            phase = "dup"  # the scan of the tile counts that follows the last pair pass
        out.append(phase)
    return out


def traffic(path, out):
    """DRAM bytes (read + write) per stage of one step, from an ncu --set full capture of that step
    (bench.py --profile under ncu --profile-from-start off)."""
    h, units, rows = _raw(path)
    sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    names = [r[h.index("Kernel Name")].replace("mvgs::", "").replace("void ", "") for r in rows]
    stages = _stage_of_sequence(names)
    res = {}
    for r, st in zip(rows, stages):
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):  # units differ per metric
            tot += _num(r[h.index(m)]) * sc.get(units[h.index(m)], 1)
        res[st] = res.get(st, 0.0) + tot
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    k = OrderedDict()
    for r in data:
        k.setdefault(r[ii], {"name": r[ki]})[r[mi]] = r[vi]
    items = list(k.values())
    # the last step: from the last k_count onwards
    last = max(i for i, it in enumerate(items) if "k_count" in it["name"])
    step = items[last:]
    tot = sum(_num(it.get("gpu__time_duration.sum", "0")) for it in step)
    print(f"# ncu launch list (--clock-control none, serialised, cold cache) of one step: {path}")
    print(f"# {len(step)} launches, sum {tot / 1e3:.1f} us")
    print(f"{'kernel':60s} {'us':>9s} {'share':>6s} {'DRAM rd':>12s} {'DRAM wr':>12s}")
    for it in step:
        t = _num(it.get("gpu__time_duration.sum", "0"))
        nm = it["name"].replace("mvgs::", "").replace("void ", "")
        print(f"{nm[:60]:60s} {t / 1e3:9.1f} {100 * t / tot:5.1f}% {it.get('dram__bytes_read.sum', ''):>12s} "
              f"{it.get('dram__bytes_write.sum', ''):>12s}")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "report":
        report(sys.argv[2])
    elif cmd == "launches":
        launches(sys.argv[2])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
