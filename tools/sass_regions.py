"""Per-region instruction / stall / smem-wavefront breakdown of an ncu report's SASS page."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
gran = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0x400
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; ix = {k: i for i, k in enumerate(h)}; data = rows[2:]
tot = sum(int(r[ix["Instructions Executed"]] or 0) for r in data)
print("total warp inst %.4g" % tot)
seg = collections.OrderedDict()
base = min(int(r[ix["Address"]], 16) for r in data)
for r in data:
    a = int(r[ix["Address"]], 16) - base
    n = int(r[ix["Instructions Executed"]] or 0)
    e = seg.setdefault(a // gran, [0, 0, 0, set()])
    e[0] += n; e[1] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    e[2] += int(r[ix["L1 Wavefronts Shared"]] or 0)
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else ""
    if op.startswith("@"): op = r[ix["Source"]].split()[1]
    if op.split(".")[0] in ("LDS", "STS", "LDG", "STG", "BRA"): e[3].add(op.split(".")[0])
for k, v in seg.items():
    if v[0] > tot * 0.005:
        print("%6s %8.1fM  stalls %7d  smem_wf %7.1fM %s" % (hex(k * gran), v[0] / 1e6, v[1], v[2] / 1e6, ",".join(sorted(v[3]))))
