#!/usr/bin/env python
"""Per-instruction hot spots of one kernel from an ncu --set full report (source page, SASS).

  python profiles/sass_hot.py REPORT KERNEL_SUBSTRING [--top N] [--all]
Prints total warp-level instructions executed, the stall-sample share, and the top SASS
lines by samples (with executed counts), so instruction mix and hot loops can be read here.
"""
import csv
import io
import subprocess
import sys


def main():
    rep, name = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{name}",
                          "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
    rows, seen = [], set()
    for r in csv.DictReader(io.StringIO("\n".join(lines[i:]))):
        if r["Address"] in seen:  # the source page can list a function's SASS twice
            continue
        seen.add(r["Address"])
        rows.append(r)
    def num(x):
        try:
            return float(x)
        except Exception:
            return 0.0
    tot_i = sum(num(r["Instructions Executed"]) for r in rows)
    tot_s = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rows)
    print(f"# {lines[0]}\n# warp instructions executed: {tot_i:.4g}; stall samples: {tot_s:.0f}")
    mix = {}
    for r in rows:
        op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
        if op.startswith("@"):
            op = r["Source"].strip().split()[1]
        op = op.split(".")[0]
        mix[op] = mix.get(op, 0) + num(r["Instructions Executed"])
    print("# mix: " + ", ".join(f"{k} {v / tot_i:.1%}" for k, v in sorted(mix.items(), key=lambda kv: -kv[1])[:18]))
    if "--all" in sys.argv:
        sel = rows
    else:
        sel = sorted(rows, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[:top]
        sel = sorted(sel, key=lambda r: int(r["Address"], 16) if r["Address"].startswith("0x") else 0)
    for r in sel:
        print(f'{r["Address"]:>8} {num(r["Warp Stall Sampling (All Samples)"]) / max(tot_s, 1):6.1%} '
              f'{num(r["Instructions Executed"]):>12.0f}  {r["Source"][:90]}')


if __name__ == "__main__":
    main()
