"""The NVLS store merge: gb_or_bits_multimem reads the OR of every GPU's
partial packed rows through a multicast address (multimem.ld_reduce.or, reduced in the
NVSwitch).  This build has one GPU, so the group has one member: the multicast mapping,
the PTX and dist.sharded_store_nvls run for real, and the OR over one partial must give
exactly the single-rank W (Eq.(1) is an OR of cliques).  Skipped when
the GPU has no multicast support (torch symmetric memory reports no multicast pointer)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["GB_ROOT"])
import gbgen
import paper_1303_7032_b200 as gb
from paper_1303_7032_b200 import dist as gdist
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
out = {}
try:
    try:
        gdist._LocalMulticast(1024, torch.device("cuda", 0))
    except Exception as e:          # diagnosis for the skip reason
        out["local_error"] = repr(e)
    to_dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()
    for c, l, m in ((8, 128, 6000), (5, 33, 700), (16, 256, 40000)):
        msgs = gbgen.messages(91 + c, m, c, l)
        ref = gb.Net(c, l)
        ref.store(to_dev(msgs))
        ref.seal()
        net = gb.Net(c, l)
        ok = gdist.sharded_store_nvls(net, to_dev(msgs))
        if not ok:
            out["skip"] = "no multicast support: " + out.get("local_error", "")
            break
        gdist.seal_status_all(net)
        torch.cuda.synchronize()
        same_w8 = bool(torch.equal(net.weights(), ref.weights()))
        net.seal()
        ref.seal()
        same_wb = bool(torch.equal(net.bits(), ref.bits()))
        # or_bits_multimem ORs into the existing W8 (a second pass leaves W unchanged)
        mc = gdist.multicast_buffer(net.n_padded * net.nw, torch.device("cuda", 0))
        buf, hdl = mc
        buf.view(net.n_padded, net.nw).copy_(ref.bits())
        hdl.barrier(channel=0)
        net.or_bits_multimem(hdl.multicast_ptr)
        net.seal()
        torch.cuda.synchronize()
        same_again = bool(torch.equal(net.bits(), ref.bits()))
        out[f"{c},{l},{m}"] = [same_w8, same_wb, same_again]
        net.close()
        ref.close()
finally:
    dist.destroy_process_group()
print("RESULT " + json.dumps(out))
"""


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_nvls_or_merge_equals_single_store():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), GB_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", WORKER], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    lines = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-4000:]
    res = json.loads(lines[-1][len("RESULT "):])
    if "skip" in res:
        pytest.skip(res["skip"])
    res.pop("local_error", None)
    assert res and all(all(v) for v in res.values()), res
