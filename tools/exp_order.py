"""Experiment: upper bound of the metric kernel's gain from a bank-conflict-free probe order.

Times decode_hyb8_kernel at C3 on (a) the bench's probe order and (b) the same probes reordered
on the host so that every 8-probe group (one quarter-warp phase) holds 4 probes with erasure mask
E and 4 with the complement ~E: with the kernel's (lane & 7) % 4 slot rotation the 8 lanes of a
phase then target 8 distinct clusters at every step (no bank conflicts on the prune / push loads).
Same work either way (probes are independent).  Usage: python tools/exp_order.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gbgen  # noqa: E402
import paper_1303_7032_b200 as gb  # noqa: E402

c, l, m, e, k = 8, 128, 20000, 4, 10_000_000
msgs = gbgen.messages(0x5EED, m, c, l)
probes, _ = gbgen.probes(0x5EED + 1, msgs, k, e, l)
mask = ((probes == 0xFFFF).astype(np.int64) << np.arange(8)).sum(1)
order = []
buckets = {}
for i, mk in enumerate(mask):
    buckets.setdefault(int(mk), []).append(i)
left = []
for mk in list(buckets):
    cm = (~mk) & 0xFF
    if mk > cm or cm not in buckets:
        continue
    a, b = buckets[mk], buckets[cm]
    g = min(len(a), len(b)) // 4
    for j in range(g):
        order += a[4 * j:4 * j + 4] + b[4 * j:4 * j + 4]
    left += a[4 * g:] + b[4 * g:]
for mk in buckets:
    if ((~mk) & 0xFF) not in buckets:
        left += buckets[mk]
order = np.array(order + left)
assert len(order) == k and len(set(order.tolist())) == k
print("ideal groups cover %.3f of the probes" % (1 - len(left) / k))
net = gb.Net(c, l, device=0)
net.store(torch.from_numpy(msgs.view(np.int16)).cuda())
net.seal()
out = net.alloc_outputs(k, device=True)
res = {}
for name, pr in (("bench order", probes), ("complement phases", probes[order])):
    pd = torch.from_numpy(np.ascontiguousarray(pr).view(np.int16)).cuda()
    for _ in range(3):
        net.decode(pd, 2, gamma=2, max_iters=20, out=out)
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        net.decode(pd, 2, gamma=2, max_iters=20, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[name] = float(np.median(ts))
    print(name, "%.4f ms" % res[name], net.decode_kernel(2))
