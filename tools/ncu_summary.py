import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h, units, vals = r[0], r[1], r[2]
want = sys.argv[2].split(",") if len(sys.argv) > 2 else []
for i, k in enumerate(h):
    if not want or any(w in k for w in want):
        print(f"{k:90s} {units[i]:12s} {vals[i]}")
