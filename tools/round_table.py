"""Markdown table of a round's bench lines (profiles/rNN_bench_c3.json + rNN_bench_rules.jsonl).

usage: python tools/round_table.py r02
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = sys.argv[1] if len(sys.argv) > 1 else "r02"
P = os.path.join(ROOT, "profiles")


def row(d):
    c, r = d.get("config", {}), d.get("roofline") or {}
    work = c.get("workload", "")
    if c.get("kernel_options"):
        work += " [" + ", ".join(c["kernel_options"]) + "]"
    kern = r.get("kernel", "")
    ms = r.get("decode_ms_per_launch") or d.get("ms_per_step")
    roof = ""
    if r:
        roof = "%.3f of %.1f %s" % (r["frac"], r["peak"], r["unit"])
        if r.get("onchip"):
            res = "issue-slot" if "issue" in r["onchip"].get("resource", "") else "LSU wavefront"
            roof += "; on-chip %.2f of the %s peak" % (r["onchip"]["frac"], res)
        if r.get("int8_equivalent"):
            ie = r["int8_equivalent"]
            roof += "; int8-equivalent %.0f TOPS (%.2f of the int8 peak)" % (ie["tops"], ie["tops"] / ie["int8_peak_tops"])
    e2e = (d.get("e2e") or {}).get("value")
    cpu = (d.get("cpu_baseline") or {}).get("value")
    return "| %s | `%s` | %.3g %s | %.4f | %s | %s | %s |" % (
        work, kern, d["value"], d["unit"], ms or 0, roof, "%.3g" % e2e if e2e else "—", "%.3g" % cpu if cpu else "—")


print("| Workload | Kernel | value | decode ms / launch | roofline | e2e | CPU oracle |")
print("|---|---|---|---|---|---|---|")
print(row(json.load(open(os.path.join(P, R + "_bench_c3.json")))))
for line in open(os.path.join(P, R + "_bench_rules.jsonl")):
    line = line.strip()
    if line:
        print(row(json.loads(line)))
