"""Small decode/store workload for compute-sanitizer (memcheck / racecheck / synccheck).

Covers every kernel family: store (scattered + privatised) + apply + seal, OR of packed
partials, decode_hyb8 (sparse loop) / decode_hyb8r (rotated layout, every first-step row count) /
decode_smem (both slot instances), decode_l2t + decode_l2 (list mode), SOS on the CUDA cores
(sos_bits, with its overflow to the pair kernel in list mode and to the generic kernel) / pair /
streamed-A (incl. Lp = 512 with the state in the global scratch) / 4-warp / generic, the
cycle-exit flag, the tensor-core SOM kernel, and the host-buffer pipeline (3 streams).
"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import gbgen
import paper_1303_7032_b200 as gb

for (c, l, m, k, e) in ((4, 16, 50, 300, 2), (8, 128, 5000, 700, 4), (12, 40, 500, 100, 5), (3, 3, 4, 20, 2),
                        (16, 256, 20000, 150, 8), (12, 100, 3000, 100, 5), (8, 512, 3000, 64, 4),
                        (16, 512, 3000, 40, 7), (4, 600, 300, 50, 2)):
    msgs = gbgen.messages(1, m, c, l)
    pr, _ = gbgen.probes(2, msgs, k, e, l, random_count=k // 10)
    rng = np.random.default_rng(k)
    for i in range(0, k, 5):   # mixed erasure counts (wide-slot / list-mode paths)
        pr[i, rng.choice(c, int(rng.integers(0, c + 1)), replace=False)] = 0xFFFF
    net = gb.Net(c, l)
    if os.environ.get("SANITIZE_NO_PAIR") == "1":   # racecheck without the CTA-pair kernels
        net.set_option("sos_pair", 0)
    net.store(torch.from_numpy(msgs.view(np.int16)).cuda())
    net.seal()
    probes = torch.from_numpy(pr.view(np.int16)).cuda()
    for rule in (0, 1, 2):
        net.decode(probes, rule, gamma=2, max_iters=6)
    net.decode_symbols(probes, 2, gamma=2, max_iters=6)
    net.decode(probes, 0, gamma=0, max_iters=6, flags=gb.FLAG_CYCLE_EXIT)
    if c == 8 and l == 128:
        net.set_option("som_tensor", 1)
        net.decode(probes, 1, gamma=1, max_iters=6)
        net.set_option("som_tensor", 0)
        for split in (0, 1):
            net.set_option("hyb8_split", split)
            net.decode(probes, 2, gamma=1, max_iters=6)
        for nr in (6, 7, 8):
            net.set_option("hyb8_rows", nr)
            net.decode(probes, 2, gamma=1, max_iters=6)
        net.set_option("hyb8_rows", 0)
        net.set_option("hyb8_split", -1)
        # sum-of-sum on the CUDA cores, forced, with random probes (overflow -> pair list mode,
        # then -> generic with the pair off) and the tensor path forced
        rp = torch.from_numpy(gbgen.probes(9, msgs, 400, 6, l, random_count=200)[0].view(np.int16)).cuda()
        for ob, sp in ((1, 1), (1, 0), (0, 1)):
            net.set_option("sos_bits", ob)
            net.set_option("sos_pair", sp)
            net.decode(rp, 0, gamma=1, max_iters=6)
        net.set_option("sos_bits", -1)
        net.set_option("sos_pair", 1)
        # host buffers: the three-stream pipeline
        ph = torch.from_numpy(pr.view(np.int16)).pin_memory()
        out = net.alloc_outputs(k, device=False, pin=True)
        net.decode(ph, 2, gamma=1, max_iters=6, out=out)
        part = gb.Net(c, l)
        part.store(torch.from_numpy(msgs[: m // 2].view(np.int16)).cuda())
        part.seal()
        fresh = gb.Net(c, l)
        fresh.or_bits(torch.stack([part.bits(), net.bits()]).contiguous())
        fresh.seal()
        fresh.clear()
        fresh.or_upper(torch.stack([part.pack_upper(), net.pack_upper()]).contiguous())
        fresh.seal()
        part.close()
        fresh.close()
    torch.cuda.synchronize()
    net.close()
print("sanitize workload done")
