"""Copy one gpu_full.sh run (gpurun_out/*_TAG.*) into profiles/ as the round's artefacts.

usage: python tools/collect_profiles.py TAG [ROUND]
Writes profiles/rNN_bench_c3.json, rNN_bench_reference_c3.json, rNN_bench_rules.jsonl,
rNN_launches_c3.csv, rNN_tests.txt, rNN_smoke.txt, rNN_ncu_<kernel>.txt (key metrics of each
ncu --set full capture) and traffic.json (DRAM bytes per launch, read by bench.py).
"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1]
RND = sys.argv[2] if len(sys.argv) > 2 else "r01"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex.sum", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
        "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio")
# capture -> (summary name, traffic key)
CAPS = {"prof_hyb": ("hyb", "c3"), "prof_sos": ("sos", "c2"), "prof_sosbits": ("sos_bits", "c2"), "prof_sosc4": ("sos_c4", "c4"),
        "prof_l2": ("l2", "c4"), "prof_store": ("store", "c5"), "prof_smem": ("smem", "c2som")}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def to_bytes(u, v):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return float(v.replace(",", "")) * scale.get(u, 1)


# probes per launch of the captures whose shared-memory wavefronts are reported per probe
PROBES = {"prof_hyb": 10_000_000, "prof_smem": 1_000_000,     # kernels whose W rows live in shared memory
          "prof_sosbits": 1_000_000}
traffic = {}
for cap, (name, cfg) in CAPS.items():
    rep = os.path.join(G, f"{cap}_{TAG}.ncu-rep")
    if not os.path.exists(rep):
        continue
    d = raw(rep)
    kname = d.get("Kernel Name", ("", "?"))[1].split("(")[0].split("::")[-1].split("<")[0]
    tkey = f"{kname}|{cfg}"
    with open(os.path.join(P, f"{RND}_ncu_{name}.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none, one launch ({cap}_{TAG}); kernel: {d.get('Kernel Name', ('', '?'))[1][:120]}\n")
        for k in KEYS:
            if k in d:
                f.write(f"{k:90s} {d[k][0]:12s} {d[k][1]}\n")
    if "dram__bytes_read.sum" in d:
        b = to_bytes(*d["dram__bytes_read.sum"]) + to_bytes(*d["dram__bytes_write.sum"])
        traffic[tkey] = {"dram_bytes_per_launch": b, "source": f"profiles/{RND}_ncu_{name}.txt",
                         "note": "ncu --set full, one launch, --clock-control none"}
        if cap in PROBES and "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum" in d:
            wf = float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"][1].replace(",", ""))
            traffic[tkey]["smem_wavefronts_per_probe"] = wf / PROBES[cap]
            traffic[tkey]["probes_in_capture"] = PROBES[cap]
        if cap in PROBES and "smsp__inst_executed.sum" in d:
            traffic[tkey]["warp_instructions_per_probe"] = float(d["smsp__inst_executed.sum"][1].replace(",", "")) / PROBES[cap]
if traffic:
    json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
for src, dst in ((f"bench_full_{TAG}.json", f"{RND}_bench_c3.json"),
                 (f"bench_ref_{TAG}.json", f"{RND}_bench_reference_c3.json"),
                 (f"bench_rules_{TAG}.jsonl", f"{RND}_bench_rules.jsonl"),
                 (f"launches_{TAG}.csv", f"{RND}_launches_c3.csv"),
                 (f"tests_{TAG}.txt", f"{RND}_tests.txt"), (f"smoke_{TAG}.txt", f"{RND}_smoke.txt"),
                 (f"motivation_{TAG}.json", f"{RND}_motivation.json")):
    s = os.path.join(G, src)
    if os.path.exists(s):
        if dst.endswith(".json") and "motivation" not in dst:   # the JSON line only
            lines = [l for l in open(s) if l.startswith("{")]
            open(os.path.join(P, dst), "w").write(lines[-1] if lines else "")
        else:
            shutil.copy(s, os.path.join(P, dst))
print("traffic:", json.dumps(traffic))
