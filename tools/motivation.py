"""E5 -- the paper's per-iteration profile (fig:motivation) on the GPU path.

fig:first: running time spent in each sum-of-max iteration; fig:converge: the cumulative
number of probes converged after each iteration.  Scenario 2 (C=16, L=512, M=50000 stored,
30000 probes), here with e=7 erased clusters, under sum-of-max (all
neurons of erased clusters on at start) and under the joint scheme (hybrid) for contrast;
plus the Scenario-1 shape at M=5000 and the metric's M=20000.

Per-iteration time: the decode is one persistent kernel, so iteration r's time is measured as
T(max_iters = r) - T(max_iters = r - 1) (every probe stops at min(r, its own convergence), so
the difference is the work of round r).  CUDA-event timing, median of 5 after 2 warm-ups.
Usage: python tools/motivation.py OUT.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gbgen  # noqa: E402
import paper_1303_7032_b200 as gb  # noqa: E402

CASES = [("scenario2", 16, 512, 50000, 7, 30000), ("c2_m5k", 8, 128, 5000, 4, 100000),
         ("c3_m20k", 8, 128, 20000, 4, 100000), ("scenario2_e13", 16, 512, 50000, 13, 30000)]


def timed(net, pr, rule, T, reps=5):
    out = net.alloc_outputs(pr.shape[0])
    for _ in range(2):
        net.decode(pr, rule, gamma=1, max_iters=T, out=out)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        net.decode(pr, rule, gamma=1, max_iters=T, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), out


def main():
    res = []
    for name, c, l, m, e, k in CASES:
        msgs = gbgen.messages(0x5EED, m, c, l)
        pr, _ = gbgen.probes(0x5EED + 1, msgs, k, e, l)
        net = gb.Net(c, l)
        net.store(torch.from_numpy(msgs.view(np.int16)).cuda())
        net.seal()
        prd = torch.from_numpy(pr.view(np.int16)).cuda()
        for rule in (gb.SUM_OF_MAX, gb.HYBRID):
            full_ms, out = timed(net, prd, rule, 20)
            it = out[1].cpu().numpy().view(np.uint16).astype(np.int64)
            ok = out[2].cpu().numpy() == 0
            R = int(it.max()) if len(it) else 0
            cum = np.cumsum(np.bincount(it[ok], minlength=R + 1)).tolist()
            per_round, prev = [], 0.0
            for r in range(1, R + 1):
                t, _ = timed(net, prd, rule, r)
                per_round.append(t - prev)
                prev = t
            res.append({"case": name, "c": c, "l": l, "M": m, "erased": e, "probes": k,
                        "rule": {1: "sum-of-max", 2: "hybrid"}[rule], "kernel": net.decode_kernel(rule),
                        "total_ms": full_ms, "ms_per_round": per_round, "converged_after_round": cum,
                        "not_converged": int((~ok).sum())})
            print(json.dumps(res[-1]), flush=True)
        net.close()
    json.dump(res, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
