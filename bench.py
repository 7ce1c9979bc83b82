#!/usr/bin/env python
"""bench.py -- probes decoded/s for the GBNN hybrid rule (arXiv:1303.7032) on B200.

Driver contract (one JSON line from rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, NCCL)

A step is one pass of the whole hot path over one batch:
  rank 0: gb_clear -> gb_store(the M messages) -> gb_seal; [N>1: NCCL broadcast
  of rank 0's packed rows Wb; other ranks: gb_clear -> gb_or_bits -> gb_seal]
  -> gb_decode(hybrid, this rank's K probes, device-resident).  Weak scaling:
  K probes per GPU.
Default workload = BASELINE config C3: c=8 l=128, M=20000, e=4 erased of 8,
hybrid rule, gamma=2, max_iters=20, K=10^7 probes per GPU.

`value` is device-timed (CUDA events, max over ranks); `e2e` repeats the step
through the same C-ABI with pinned HOST buffers (H2D of messages+probes and
D2H of state/iters/status inside the timed region); `roofline` is measured
live on the decode kernel; `cpu_baseline` times the CPU oracle on a bounded
sample on this host (rank 0, N=1 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "probes decoded/sec, hybrid rule, c=8 l=128, 1-8 B200; % of TC/HBM roofline"
RULE_NAMES = {0: "sum-of-sum", 1: "sum-of-max", 2: "hybrid"}
CONFIGS = {
    # name: (c, l, M, e, rule, K per GPU, description)
    "c3": (8, 128, 20000, 4, 2, 10_000_000, "BASELINE C3: c=8 l=128 M=20k e=4 hybrid, 10^7 probes/GPU"),
    "c2": (8, 128, 5000, 4, 2, 100_000, "BASELINE C2 point: c=8 l=128 M=5k e=4, 10^5 probes"),
    "c1": (4, 16, 50, 2, 2, 1000, "BASELINE C1: c=4 l=16 M=50 e=2, 1000 probes"),
    "c4": (16, 256, 100000, 8, 1, 1_000_000, "BASELINE C4: c=16 l=256 M=100k e=8, 10^6 probes"),
    "c5": (16, 256, 10_000_000, 0, -1, 0, "BASELINE C5: store of 10^7 messages at c=16 l=256 (sharded over ranks, partial W merged over NCCL)"),
    # the paper's Scenario 2: its only published runtime (14.86 s for
    # 30000 probes on a Tesla C1060 => 2019 probes/s) is quoted as vs_baseline context.
    "s2": (16, 512, 50000, 7, 2, 30000, "Scenario 2 (PAPER.md L731): c=16 l=512 M=50k e=7 hybrid, 30000 probes"),
}
PAPER_BASELINE = {"s2": 30000 / 14.86}
SEED = 0x5EED
L2_FLUSH_BYTES = 512 << 20


def dist_env():
    """(world size, rank, local device).  GB_DIST_BACKEND=gloo (test only) lets several ranks
    share one GPU to exercise the N>1 code path where only one GPU exists; the default is NCCL
    with one rank per GPU."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("GB_DIST_BACKEND", "nccl") != "nccl":
        import torch
        local = local % max(1, torch.cuda.device_count())
    return ws, rank, local


def init_dist(local):
    import torch
    import torch.distributed as tdist
    backend = os.environ.get("GB_DIST_BACKEND", "nccl")
    if backend == "nccl":
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        tdist.init_process_group(backend)
    return tdist


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), "measured"
    return 6650.0, 1590.0, "fallback"


def ncu_entry(kernel, workload):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return {}
    return json.load(open(p)).get(f"{kernel}|{workload}", {})


def ncu_traffic(kernel, workload):
    return ncu_entry(kernel, workload).get("dram_bytes_per_launch")


class ClockSampler:
    """nvidia-smi clocks/throttle sampling while the timed region runs."""
    FIELDS = ["timestamp", "clocks.sm", "clocks.max.sm", "power.draw",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()
        t0 = time.time()
        while not self.rows and time.time() - t0 < 5:
            time.sleep(0.02)

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append((time.time(), parts))

    def mark(self):
        return len(self.rows)

    def stop(self, first):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = self.rows[first:] or self.rows[-1:]
        sm = sorted(float(r[1][1]) for r in rows if r[1][1].replace(".", "").isdigit())
        mx = max((float(r[1][2]) for r in rows if r[1][2].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[1][4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max((float(r[1][3]) for r in rows
                                                          if r[1][3].replace(".", "").isdigit()), default=None)}


def cpu_oracle_sample(msgs, probes, c, l, rule, gamma, max_iters, budget_s, gpu_out=None, threads=None):
    """Time the CPU oracle (as it stands) on a bounded prefix of the workload.  Returns
    (n, seconds, parity of the prefix vs the GPU, mean bail-out blocks per probe) -- the
    blocks are the oracle's work counter (PAPER.md L445-451 walk; SOS: rounds)."""
    os.environ["OMP_NUM_THREADS"] = str(threads or host_cores())   # all host cores (torchrun sets 1)
    import numpy as np
    import oracle
    w, _ = oracle.store(msgs, c, l)
    cal = min(len(probes), 256)
    t0 = time.perf_counter()
    oracle.decode(w, c, l, probes[:cal], rule, gamma=gamma, max_iters=max_iters)
    rate = cal / max(time.perf_counter() - t0, 1e-6)
    n = int(min(len(probes), max(cal, rate * budget_s)))
    t0 = time.perf_counter()
    st, it, ss, blk = oracle.decode(w, c, l, probes[:n], rule, gamma=gamma, max_iters=max_iters, with_blocks=True)
    dt = time.perf_counter() - t0
    parity = None
    if gpu_out is not None:
        gs, gi, gt = gpu_out
        parity = bool(np.array_equal(gs[:n], st) and np.array_equal(gi[:n], it) and np.array_equal(gt[:n], ss))
    return n, dt, parity, float(blk.mean())


def run_reference(args, cfg):
    """--impl reference: the CPU oracle, as it stands, on host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import numpy as np
    import gbgen
    c, l, m, e, rule, k, desc = cfg
    msgs = gbgen.messages(SEED, m, c, l)
    per_step = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    pool = min(k, 200_000)
    probes, _ = gbgen.probes(SEED + 1, msgs, pool, e, l)
    os.environ["OMP_NUM_THREADS"] = str(host_cores())   # all host cores (torchrun sets 1)
    import oracle
    w, _ = oracle.store(msgs, c, l)
    cal = 256
    t0 = time.perf_counter()
    oracle.decode(w, c, l, probes[:cal], rule, gamma=args.gamma, max_iters=args.max_iters)
    rate = cal / (time.perf_counter() - t0)
    n = int(min(pool, max(cal, rate * per_step)))
    times = []
    for s in range(args.warmup + args.steps):
        off = (s * n) % max(1, pool - n + 1)
        t0 = time.perf_counter()
        oracle.store(msgs, c, l)
        oracle.decode(w, c, l, probes[off:off + n], rule, gamma=args.gamma, max_iters=args.max_iters)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * len(times) / tot
    sample = f"{n} probes/step of {desc} (+ store of all {m} messages each step)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "probes/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (gbgen splitmix64, seed 0x5EED)",
        "config": config_dict(args, cfg, ws),
        "cpu_baseline": {"value": value, "unit": "probes/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
                         "kind": "oracle", "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": value, "unit": "probes/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def io_bytes_per_step(c, l, k):
    nw = c * ((l + 31) // 32)
    return k * (2 * c + 4 * nw + 3)


def l2_policy(c, l, k):
    """(flush before every timed step?, the config text) -- a function of the workload only,
    so both arms print the same config."""
    io = io_bytes_per_step(c, l, k)
    if io >= L2_FLUSH_BYTES // 2:
        return False, "inputs larger than L2 (%.0f MB of probes+results per step per GPU; L2 126 MB)" % (io / 1e6)
    return True, "L2 flushed (512 MiB write) before each timed step; per-step event windows summed"


def symbols_agree(sym, state_dev, c, l, n=4096):
    """Harness check of gb_decode_symbols against the device state of the same batch on the
    first n probes: a cluster's symbol is its only set bit, 0xFFFF if none, 0xFFFE if several."""
    import numpy as np
    wc = (l + 31) // 32
    st = state_dev[:n].cpu().numpy().view(np.uint32).reshape(-1, c, wc)
    bits = ((st[..., None] >> np.arange(32, dtype=np.uint32)) & 1).reshape(st.shape[0], c, 32 * wc)
    cnt = bits.sum(axis=2)
    want = np.where(cnt == 0, 0xFFFF, np.where(cnt > 1, 0xFFFE, bits.argmax(axis=2))).astype(np.uint16)
    return bool(np.array_equal(sym[:n].view(np.uint16), want))


def config_dict(args, cfg, ws):
    c, l, m, e, rule, k, desc = cfg
    d = {"workload": desc, "c": c, "l": l, "M": m, "erased": e, "rule": RULE_NAMES[rule],
         "gamma": args.gamma, "max_iters": args.max_iters, "probes_per_gpu": k,
         "global_batch": k * ws,
         "parallelism": f"dp{ws} (probe shards; W stored on rank 0, packed rows broadcast over NCCL)",
         "l2": l2_policy(c, l, k)[1], "seed": SEED}
    if getattr(args, "opt", None):
        d["kernel_options"] = list(args.opt)   # gb_set_option overrides (bit-exact kernel choices)
    return d


SM_COUNT, SM_CLOCK_GHZ = 148, 1.965   # B200 (B200_PROFILING.md); clocks sampled in the C3 line


def run_store(args, cfg):
    """C5: storage scaling.  Step = gb_clear + gb_store(this rank's M/N messages) + NCCL MAX merge of
    W8 (uint8) + gb_seal.  Strong scaling: M fixed, sharded over the ranks."""
    import numpy as np
    import torch
    import gbgen
    import paper_1303_7032_b200 as gb
    from paper_1303_7032_b200 import dist as gdist
    c, l, m, e, rule, k, desc = cfg
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        tdist = init_dist(local)
    dev = torch.device("cuda", local)
    lo, hi = gdist.strong_bounds(m, rank, ws)
    if args.impl == "reference":
        if rank == 0:
            import oracle
            os.environ["OMP_NUM_THREADS"] = str(host_cores())   # all host cores (torchrun sets 1)
            n = 200_000
            msgs = gbgen.messages(SEED, n, c, l)
            t0 = time.perf_counter()
            for _ in range(args.steps):
                oracle.store(msgs, c, l)
            v = n * args.steps / (time.perf_counter() - t0)
            print(json.dumps({"impl": "reference", "metric": "messages stored/sec (C5)", "value": v,
                              "unit": "messages/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                              "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
                              "data": "synthetic", "config": {"workload": desc},
                              "cpu_baseline": {"value": v, "unit": "messages/s", "cores": 1, "kind": "oracle",
                                               "sample": f"{n} messages per step"},
                              "e2e": {"value": v, "unit": "messages/s", "h2d_bytes_per_step": 0,
                                      "d2h_bytes_per_step": 0}}), flush=True)
        return 0
    msgs = gbgen.messages(SEED, m, c, l) if m <= 20_000_000 else None
    shard = torch.from_numpy(np.ascontiguousarray(msgs[lo:hi]).view(np.int16)).to(dev)
    net = gb.Net(c, l, device=local)
    stream = torch.cuda.current_stream()
    store_step = {"bits": gdist.sharded_store_bits, "max": gdist.sharded_store,
                  "upper": gdist.sharded_store_upper}[args.merge]
    for _ in range(args.warmup):
        store_step(net, shard)
    gdist.seal_status_all(net)
    torch.cuda.synchronize()
    l0 = net.launch_count()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        store_step(net, shard)
    b.record(stream)
    torch.cuda.synchronize()
    ms = gdist.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
    value = m * args.steps / (ms / 1e3)
    hbm, _, kind = measured_peaks()
    np_ = net.n_padded
    # algorithmic bytes per step: message input 2C B each + W8 (u8 n_p^2) written + seal read/packed
    alg = (hi - lo) * 2 * c + np_ * np_ + 2 * np_ * np_ + np_ * np_ // 8
    achieved = alg / (ms / args.steps / 1e3) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "messages stored/sec (C5 storage scaling)", "value": value, "unit": "messages/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (gbgen, seed 0x5EED)",
            "config": {"workload": desc, "c": c, "l": l, "M": m, "messages_per_gpu": hi - lo,
                       "edge_writes_per_message": c * (c - 1),
                       "merge": {"bits": "all-gather of packed partial W + gb_or_bits",
                                 "max": "all-reduce MAX of u8 W8",
                                 "upper": "all-gather of the packed upper-triangle blocks + gb_or_upper"}[args.merge]
                                if ws > 1 else "none (1 rank)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": None, "kernel": "store_priv_kernel+apply_kernel+seal_kernel",
                         "note": "bytes = message input + W8 + seal; the store kernel is bound on chip by "
                                 "shared-memory atomics (see smem_atomics)"},
            "smem_atomics": {"bit_sets_per_s": (hi - lo) * c * (c - 1) / (ms / args.steps / 1e3),
                             "ideal_per_s": SM_COUNT * 32 * SM_CLOCK_GHZ * 1e9,
                             "frac": (hi - lo) * c * (c - 1) / (ms / args.steps / 1e3) / (SM_COUNT * 32 * SM_CLOCK_GHZ * 1e9),
                             "note": "M*C*(C-1) random bit sets into shared-memory tiles vs one conflict-free "
                                     "32-lane shared atomic per SM per clock (148 SMs, 1.965 GHz)"},
            "gpu_launches": net.launch_count() - l0}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--rule", type=int, default=None)
    ap.add_argument("--messages", type=int, default=None)
    ap.add_argument("--probes", type=int, default=None)
    ap.add_argument("--gamma", type=int, default=2)
    ap.add_argument("--merge", default="upper", choices=["bits", "max", "upper"],
                    help="C5 store merge over ranks: all-gather of the packed upper triangle + OR (N3), "
                         "of the whole packed W + OR, or u8 MAX all-reduce")
    ap.add_argument("--max-iters", type=int, default=20)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=18.0)   # calibration on 256 probes overestimates the time (~0.7x measured)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--opt", action="append", default=[],
                    help="kernel-selection option NAME=VALUE for gb_set_option (A/B experiments)")
    ap.add_argument("--cpu-threads", type=int, default=None,
                    help="host threads of the cpu_baseline oracle (default: all cores; 1 for the C1 figure)")
    args = ap.parse_args()
    c, l, m, e, rule, k, desc = CONFIGS[args.config]
    if args.rule is not None:
        rule = args.rule
    if args.messages is not None:
        m = args.messages
    if args.probes is not None:
        k = args.probes
    if (args.rule, args.messages, args.probes) != (None, None, None):
        desc = f"c={c} l={l} M={m} e={e} {RULE_NAMES[rule]}, {k} probes/GPU"
    cfg = (c, l, m, e, rule, k, desc)
    args.warmup = max(args.warmup, 3)
    if args.config == "c5":
        return run_store(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)

    import numpy as np
    import torch
    import gbgen
    import paper_1303_7032_b200 as gb
    from paper_1303_7032_b200 import dist as gdist

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist = init_dist(local)
    else:
        dist = None
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    msgs = gbgen.messages(SEED, m, c, l)
    probes, _ = gbgen.probes(SEED + 1, msgs, k, e, l, start=gdist.weak_bounds(k, rank)[0])
    # W is stored on rank 0 and replicated (north_star): only rank 0 holds the messages
    my_msgs = msgs if rank == 0 else msgs[:0]
    msgs_d = torch.from_numpy(np.ascontiguousarray(my_msgs).view(np.int16)).to(dev)
    probes_d = torch.from_numpy(probes.view(np.int16)).to(dev)
    net = gb.Net(c, l, device=local, **{kv.split("=")[0]: int(kv.split("=")[1]) for kv in args.opt})
    out = net.alloc_outputs(k, device=True)
    stream = torch.cuda.current_stream()
    nw = net.nw
    t_dec = []

    def step(timed):
        # rank 0: clear + store + seal; [N>1: broadcast of the packed rows; others: clear +
        # or_bits + seal].  The seal does not synchronise the host.
        gdist.replicated_store(net, msgs_d)
        if timed:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
        net.decode(probes_d, rule, gamma=args.gamma, max_iters=args.max_iters, out=out)
        if timed:
            b.record(stream)
            t_dec.append((a, b))

    for _ in range(args.warmup):
        step(False)
    gdist.seal_status_all(net)   # the seals of the warm-up found W well formed (outside the timed region)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    first = sampler.mark()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = net.launch_count()
    flush_l2, l2_note = l2_policy(c, l, k)
    if not flush_l2:
        # inputs + outputs of one step are larger than L2: one event window over all steps
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step(True)
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    else:
        # small batch: flush L2 (write a 512 MiB buffer) before every timed step; per-step event
        # windows (excluding the flush) are summed
        flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
        wins = []
        for _ in range(args.steps):
            flush.zero_()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            step(True)
            a1.record(stream)
            wins.append((a0, a1))
        torch.cuda.synchronize()
        ms = sum(a0.elapsed_time(a1) for a0, a1 in wins)
    if dist is not None:
        dist.barrier()
    clocks = sampler.stop(first)
    launches = net.launch_count() - l0
    dec_ms = sum(a.elapsed_time(b) for a, b in t_dec) / len(t_dec)
    ms, dec_ms = gdist.max_over_ranks([ms, dec_ms], device=dev)
    value = ws * k * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (the decode kernel, one launch per call)
    hbm, bf16, peak_kind = measured_peaks()
    bytes_per_probe = 2 * c + 4 * nw + 2 + 1
    kernel = net.decode_kernel(rule)
    if kernel.startswith("sos_") and kernel != "sos_bits_kernel":
        # tensor-bound.  Algorithmic int8 ops = sum over probes of its rounds x 2 n_p^2 (Eq.(11) per
        # probe-round).  Both SOS kernels refill converged slots of their 128-probe tiles, so the
        # executed work is the algorithmic work plus the last partial rounds (a fixed-tile kernel
        # would execute tile-rounds x 128 x 2 n_p^2, reported for comparison).
        it_h = out[1].cpu().numpy().view(np.uint16).astype(np.int64)
        pad = (-k) % 128
        tiles = np.concatenate([it_h, np.zeros(pad, np.int64)]).reshape(-1, 128).max(axis=1)
        npad = net.n_padded
        ops_alg = float(it_h.sum()) * 2 * npad * npad
        ops_tile = float(tiles.sum()) * 2 * 128 * npad * npad
        fp4 = kernel.startswith("sos_fp4")
        # int8 dense = 2 x bf16, e2m1 (block-scaled FP4) dense = 4 x bf16 (guide's nominal 4.5 / 9 vs
        # 2.25 PFLOP/s) x the measured bf16 peak
        peak = (4.0 if fp4 else 2.0) * bf16
        achieved = ops_alg / (dec_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOPS(fp4)" if fp4 else "TOPS(int8)",
                "frac": achieved / peak, "traffic": ncu_traffic(kernel, args.config), "kernel": kernel,
                "ops_per_probe_round": 2 * npad * npad, "probe_rounds": int(it_h.sum()),
                "tile_rounds_if_no_refill": int(tiles.sum()),
                "ops_basis": "algorithmic (per-probe rounds); the kernels refill converged TMEM lanes, so "
                             "executed work = algorithmic + the partial last rounds",
                "peak_source": peak_kind + (" (4 x MEASURED_PEAKS.json bf16_tflops, fp4/bf16 nominal ratio)" if fp4
                                            else " (2 x MEASURED_PEAKS.json bf16_tflops, int8/bf16 nominal ratio)"),
                "decode_ms_per_launch": dec_ms, "decode_share_of_step": dec_ms / (ms / args.steps)}
    else:
        achieved = k * bytes_per_probe / (dec_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": ncu_traffic(kernel, args.config), "kernel": kernel,
                "algorithmic_bytes_per_probe": bytes_per_probe,
                "peak_source": peak_kind + " (MEASURED_PEAKS.json hbm_gbs)",
                "decode_ms_per_launch": dec_ms, "decode_share_of_step": dec_ms / (ms / args.steps)}
        if kernel == "sos_bits_kernel":
            # sum-of-sum on the CUDA cores (sparse states): an I/O roofline like the bit kernels; for
            # comparison, the dense int8 contraction the tensor-core kernels would run for the same
            # probe-rounds (2 n_p^2 per probe-round) per second of this kernel
            it_h = out[1].cpu().numpy().view(np.uint16).astype(np.int64)
            npad = net.n_padded
            roof["int8_equivalent"] = {"tops": float(it_h.sum()) * 2 * npad * npad / (dec_ms / 1e3) / 1e12,
                                       "int8_peak_tops": 2.0 * bf16, "probe_rounds": int(it_h.sum()),
                                       "note": "dense-contraction ops the tensor-core path executes for the "
                                               "same rounds; this kernel adds only the active rows"}
        wpp = ncu_entry(kernel, args.config).get("smem_wavefronts_per_probe")
        ipp = ncu_entry(kernel, args.config).get("warp_instructions_per_probe")
        if kernel == "sos_bits_kernel" and ipp:
            # its binding on-chip resource: issue slots (4 warp-instructions per SM per clock);
            # instructions per probe from the committed ncu capture, time from this run
            sm_clk = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0)) \
                if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
            per_s = ipp * k / (dec_ms / 1e3)
            peak_is = 4 * torch.cuda.get_device_properties(dev).multi_processor_count * sm_clk * 1e6
            roof["onchip"] = {"resource": "issue slots (4 warp-instructions per SM per clock)",
                              "warp_instructions_per_probe": ipp, "achieved_per_s": per_s, "peak_per_s": peak_is,
                              "frac": per_s / peak_is, "source": ncu_entry(kernel, args.config).get("source"),
                              "note": "instructions per probe from the committed ncu capture named in source "
                                      "(ncu cannot run inside the timed bench); time from this run"}
            wpp = None
        if wpp:
            # the binding on-chip resource of the bit kernels: shared-memory wavefronts through the
            # LSU data pipe (one wavefront per SM per clock); per-probe count from the ncu capture
            sm_clk = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", 1965.0)) \
                if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1965.0
            per_s = wpp * k / (dec_ms / 1e3)
            peak_wf = torch.cuda.get_device_properties(dev).multi_processor_count * sm_clk * 1e6
            roof["onchip"] = {"resource": "shared-memory wavefronts (LSU data pipe, 1 per SM per clock)",
                              "wavefronts_per_probe": wpp, "achieved_per_s": per_s, "peak_per_s": peak_wf,
                              "frac": per_s / peak_wf, "source": ncu_entry(kernel, args.config).get("source"),
                              "note": "wavefronts per probe from the committed ncu capture named in source "
                                      "(ncu cannot run inside the timed bench); time from this run"}

    # e2e through the C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        msgs_h = torch.from_numpy(np.ascontiguousarray(my_msgs).view(np.int16)).pin_memory()
        probes_h = torch.from_numpy(probes.view(np.int16)).pin_memory()
        out_h = net.alloc_outputs(k, device=False, pin=True)

        def e2e_step():
            gdist.replicated_store(net, msgs_h)
            net.decode(probes_h, rule, gamma=args.gamma, max_iters=args.max_iters, out=out_h)

        e2e_step()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        te = gdist.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
        state_bits = {"value": ws * k * args.e2e_steps / (te / 1e3), "unit": "probes/s",
                      "h2d_bytes_per_step": int(my_msgs.nbytes + probes.nbytes),
                      "d2h_bytes_per_step": int(k * (4 * nw + 3)),
                      "how": "gb_store + gb_seal + gb_decode with pinned host buffers (library-staged, "
                             "H2D / kernel / D2H pipelined on three streams); the full final state bits come back"}
        ok = (np.array_equal(out_h[0].numpy(), out[0].cpu().numpy()) and
              np.array_equal(out_h[1].numpy(), out[1].cpu().numpy()))
        state_bits["matches_device_path"] = bool(ok)
        # the same step through gb_decode_symbols: the retrieved message (2 B per cluster) comes
        # back instead of the state bits -- the result a host caller of the decoder reads (the
        # headline e2e; the state-bits variant is reported beside it)
        sym_h = (torch.empty((k, c), dtype=torch.int16).pin_memory(), torch.empty(k, dtype=torch.int16).pin_memory(),
                 torch.empty(k, dtype=torch.uint8).pin_memory())

        def sym_step():
            gdist.replicated_store(net, msgs_h)
            net.decode_symbols(probes_h, rule, gamma=args.gamma, max_iters=args.max_iters, out=sym_h)

        sym_step()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        a.record(stream)
        for _ in range(args.e2e_steps):
            sym_step()
        b.record(stream)
        torch.cuda.synchronize()
        ts = gdist.max_over_ranks([a.elapsed_time(b)], device=dev)[0]
        e2e = {"value": ws * k * args.e2e_steps / (ts / 1e3), "unit": "probes/s",
               "h2d_bytes_per_step": int(my_msgs.nbytes + probes.nbytes),
               "d2h_bytes_per_step": int(k * (2 * c + 3)),
               "how": "gb_store + gb_seal + gb_decode_symbols with pinned host buffers (library-staged, "
                      "H2D / kernel / D2H pipelined on three streams): the retrieved message per probe (one uint16 per "
                      "cluster) + rounds + status",
               "matches_device_path": bool(np.array_equal(sym_h[1].numpy(), out[1].cpu().numpy()) and
                                           np.array_equal(sym_h[2].numpy(), out[2].cpu().numpy()) and
                                           symbols_agree(sym_h[0].numpy(), out[0], c, l)),
               "state_bits": state_bits}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        gs = out[0].cpu().numpy().view(np.uint32)
        gi = out[1].cpu().numpy().view(np.uint16)
        gt = out[2].cpu().numpy()
        n, dt, parity, blk = cpu_oracle_sample(msgs, probes, c, l, rule, args.gamma, args.max_iters,
                                               args.cpu_budget, (gs, gi, gt), threads=args.cpu_threads)
        if rule != 0:
            # algorithmic W-row bytes of the paper's bail-out-early walk (PAPER.md
            # L445-451; hybrid: + the (C-e)e prune blocks), counted by the oracle on the sample
            wrow = blk * l / 8.0
            roof["wrow"] = {"blocks_per_probe": blk, "bytes_per_probe": wrow,
                            "achieved_GBps": wrow * k / (dec_ms / 1e3) / 1e9,
                            "source": f"oracle work counter on the cpu_baseline sample ({n} probes)",
                            "note": "L-bit blocks of W the paper's per-neuron walk reads; the kernel's push "
                                    "reads other rows (it ORs source rows until the target is covered)"}
        cpu = {"value": n / dt, "unit": "probes/s", "cores": int(os.environ.get("OMP_NUM_THREADS", host_cores())),
               "kind": "oracle", "sample": f"first {n} probes of the same batch ({desc}), W from the same "
                                           f"{m} messages; {dt:.1f} s", "cpu": cpu_model(),
               "parity_vs_gpu_on_sample": parity}

    conv = None
    if rank == 0:
        # E5 (fig:converge): probes converged after each round (cumulative)
        it_all = out[1].cpu().numpy().view(np.uint16).astype(np.int64)
        st_all = out[2].cpu().numpy()
        ok = st_all == 0
        hist = np.bincount(it_all[ok], minlength=int(it_all.max(initial=0)) + 1)
        conv = {"converged_by_round": np.cumsum(hist).tolist(), "not_converged": int((~ok).sum()),
                "mean_rounds": float(it_all.mean()) if len(it_all) else 0.0,
                "note": "cumulative count of probes whose status is CONVERGED with iters <= r "
                        "(r = 0, 1, ...; hybrid counts its bail-out rounds, R6)"}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "probes/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "weak",
                "vs_baseline": (value / PAPER_BASELINE[args.config]) if (args.config in PAPER_BASELINE and
                                                                        rule == CONFIGS[args.config][4]) else None,
                "dtype": "u32",
                "data": "synthetic (gbgen splitmix64, seed 0x5EED; iid uniform symbols, uniform erasures)",
                "config": config_dict(args, cfg, ws), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, "convergence": conv}
        print(json.dumps(line), flush=True)
    net.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
