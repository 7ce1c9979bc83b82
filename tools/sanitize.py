"""Small decode/store workload for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import gbgen
import paper_1303_7032_b200 as gb

for (c, l, m, k, e) in ((4, 16, 50, 300, 2), (8, 128, 5000, 700, 4), (12, 40, 500, 100, 5), (3, 3, 4, 20, 2)):
    msgs = gbgen.messages(1, m, c, l)
    pr, _ = gbgen.probes(2, msgs, k, e, l, random_count=k // 10)
    net = gb.Net(c, l)
    net.store(torch.from_numpy(msgs.view(np.int16)).cuda())
    net.seal()
    for rule in (0, 1, 2):
        net.decode(torch.from_numpy(pr.view(np.int16)).cuda(), rule, gamma=2, max_iters=6)
    torch.cuda.synchronize()
    net.close()
print("sanitize workload done")
