"""Multi-GPU plumbing for the GBNN path.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL on the GPU
box, gloo in the CPU tests).  Nothing here computes any part of the method:

* decode shards naturally -- the columns of Eq.(11) S^t = W V^t are
  independent, so each rank decodes its own contiguous
  probe range with no data-path collective;
* store has one real exchange step -- each rank ORs the cliques of its
  message shard into a partial W8, and the partials are merged by an
  all-reduce MAX on uint8 (MAX over {0,1} is OR; Eq.(1) is an OR of
  cliques).  MAX must never be applied to packed bit
  words (max(0b01, 0b10) = 0b10 != 0b11), so the merge takes the u8 matrix;
* or the partials are exchanged packed: each rank seals its
  partial W (bit rows Wb, n_p^2/8 bytes), the Wb's are all-gathered, and every
  rank ORs all of them into its W8 (gb_or_bits) -- per rank (G-1) n_p^2/8 bytes
  received instead of the ring all-reduce's 2 (G-1)/G n_p^2 bytes of u8;
* for decode (north_star, BASELINE config C3) W is built on one rank and
  replicated: the root stores the messages and seals, its packed rows Wb
  (n_p^2/8 bytes: 128 KiB at c=8 l=128) are broadcast, and every other rank
  ORs them into its cleared W8 (gb_or_bits) and seals -- all ranks end with
  byte-identical W8 / Wb.

Collectives on a gloo group (the CPU tests and the one-GPU multi-rank test)
take a host round trip, so the same code runs with NCCL on the GPU box.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def world():
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def weak_bounds(k_per_rank: int, rank: int):
    """Global probe range of ``rank`` when every rank decodes k_per_rank probes."""
    return rank * k_per_rank, (rank + 1) * k_per_rank


def strong_bounds(k_total: int, rank: int, world_size: int):
    """Near-equal contiguous split of k_total probes (results are split-invariant)."""
    base, extra = divmod(k_total, world_size)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def message_shard(msgs, rank: int, world_size: int):
    """Round-robin message shard of this rank (any split gives the same W)."""
    return msgs[rank::world_size]


def merge_weights_(w8: torch.Tensor, group=None) -> torch.Tensor:
    """In-place all-reduce MAX of the u8 weight matrix (= OR of the partial W's)."""
    if w8.dtype != torch.uint8:
        raise TypeError("merge_weights_ needs the uint8 W8 matrix (MAX on packed bits is not OR)")
    if dist.is_available() and dist.is_initialized():
        if w8.is_cuda and not _is_nccl(group):
            h = w8.detach().cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
            w8.copy_(h)
        else:
            dist.all_reduce(w8, op=dist.ReduceOp.MAX, group=group)
    return w8


def _is_nccl(group=None):
    return dist.get_backend(group) == "nccl"


def broadcast_(t: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """In-place broadcast of ``t`` from rank ``src`` (NCCL on the tensor's device; gloo via host)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    if t.is_cuda and not _is_nccl(group):
        h = t.detach().cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)
    return t


def broadcast_weights_(w8: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Replicate the u8 W8 of rank ``src`` (after this, call seal on every rank)."""
    return broadcast_(w8, src, group)


def replicated_store(net, msgs, src: int = 0, group=None, stream=None):
    """W built once on rank ``src`` and replicated by a broadcast (north_star):
    src: gb_clear + gb_store(msgs) + gb_seal; broadcast of its packed rows Wb; every other
    rank: gb_clear + gb_or_bits(Wb) + gb_seal.  Only ``src`` reads ``msgs``."""
    rank, ws = world()
    if group is not None:
        rank, ws = dist.get_rank(group), dist.get_world_size(group)
    net.clear(stream)
    if rank == src and msgs is not None and msgs.shape[0]:
        net.store(msgs, stream)
    if ws == 1:
        net.seal(stream, check=False)
        return
    if rank == src:
        net.seal(stream, check=False)
        wb = net.bits()
    else:
        wb = torch.empty((net.n_padded, net.nw), dtype=torch.int32, device=f"cuda:{net.device}")
    broadcast_(wb, src, group)
    if rank != src:
        net.or_bits(wb.unsqueeze(0), stream)
        net.seal(stream, check=False)


def max_over_ranks(values, device=None):
    """Element-wise max over ranks of a list of floats (timing windows)."""
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def sum_over_ranks(values, device=None):
    """Element-wise sum over ranks of a list of integers (counters)."""
    t = torch.tensor(list(values), dtype=torch.int64, device=device)
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(x) for x in t.tolist()]


def sharded_store(net, msgs_shard, group=None, stream=None):
    """gb_clear + gb_store(shard) + MAX merge + gb_seal on one rank (no host sync: the
    outcome is checked by seal_status_all)."""
    net.clear(stream)
    if msgs_shard.shape[0]:
        net.store(msgs_shard, stream)
    merge_weights_(net.weights(), group)
    net.seal(stream, check=False)


def seal_status_all(net, group=None):
    """gb_seal_status on every rank, agreed over the group: if any rank's seal failed
    (broken invariants, or its shard held messages with invalid symbols) every rank
    raises, so no rank is left waiting in a later collective."""
    from . import GBError
    err = None
    try:
        net.seal_status()
    except GBError as e:
        err = e
    if not (dist.is_available() and dist.is_initialized()):
        if err:
            raise err
        return
    bad = sum_over_ranks([1 if err else 0], device=f"cuda:{net.device}" if _is_nccl(group) else None)[0]
    if bad:
        raise err if err else GBError(-1, f"gb_seal failed on {bad} other rank(s)")


def gather_bits(wb: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather this rank's packed rows Wb [n_p, nw] (int32) into [G, n_p, nw]."""
    if not (dist.is_available() and dist.is_initialized()):
        return wb.unsqueeze(0).contiguous()
    ws = dist.get_world_size(group)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((ws,) + tuple(wb.shape), dtype=wb.dtype, device=wb.device)
        dist.all_gather_into_tensor(out, wb.contiguous(), group=group)
        return out
    # gloo (CPU tests, and the one-GPU test hook GB_DIST_BACKEND=gloo): host round trip
    src = wb.detach().cpu().contiguous()
    out = torch.empty((ws,) + tuple(src.shape), dtype=src.dtype)
    dist.all_gather(list(out.unbind(0)), src, group=group)
    return out.to(wb.device)


def gather_(t: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather a 1-D tensor into [G, n] (NCCL on the device; gloo via host)."""
    if not (dist.is_available() and dist.is_initialized()):
        return t.unsqueeze(0).contiguous()
    ws = dist.get_world_size(group)
    if _is_nccl(group):
        out = torch.empty((ws,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out
    src = t.detach().cpu().contiguous()
    out = torch.empty((ws,) + tuple(src.shape), dtype=src.dtype)
    dist.all_gather(list(out.unbind(0)), src, group=group)
    return out.to(t.device)


def sharded_store_upper(net, msgs_shard, group=None, stream=None):
    """N3 merge with the upper triangle only (W symmetric): gb_clear +
    gb_store(shard) + gb_seal, gb_pack_upper (C(C-1)/2 of the C^2 cluster-pair blocks),
    all-gather, gb_or_upper (ORs each block and its mirror into W8) + gb_seal."""
    net.clear(stream)
    if msgs_shard.shape[0]:
        net.store(msgs_shard, stream)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        net.seal(stream, check=False)
        allu = gather_(net.pack_upper(stream=stream), group)
        net.clear(stream)
        net.or_upper(allu, stream)
    net.seal(stream, check=False)


def sharded_store_bits(net, msgs_shard, group=None, stream=None):
    """gb_clear + gb_store(shard) + gb_seal (pack the partial) + all-gather of
    the packed partials + gb_or_bits + gb_seal on one rank (N3 merge).  The seals
    do not synchronise the host; the invalid-message count of the shard stays on the
    device until seal_status_all (no rank raises before the collective)."""
    net.clear(stream)
    if msgs_shard.shape[0]:
        net.store(msgs_shard, stream)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        net.seal(stream, check=False)
        allb = gather_bits(net.bits(), group)
        net.or_bits(allb, stream)
    net.seal(stream, check=False)


_MC = {}   # (group name, words, device) -> (buffer, handle): one allocation per shape


class _LocalMulticast:
    """A one-GPU multicast object (CUDA driver multicast API through cuda-python): the
    group-of-one case, where no handle has to be exported to other processes.  Gives the
    same (buffer, handle) pair as torch symmetric memory: ``multicast_ptr`` and ``barrier``."""

    def __init__(self, words: int, device):
        from cuda.bindings import driver as cu
        dev = torch.device(device).index or 0
        torch.cuda.init()

        def ok(r):
            err = r[0] if isinstance(r, tuple) else r
            if err != cu.CUresult.CUDA_SUCCESS:
                raise RuntimeError(f"CUDA driver: {err}")
            return r[1] if isinstance(r, tuple) and len(r) == 2 else r
        size = words * 4
        prop = cu.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.handleTypes = 0
        prop.size = size
        gran = ok(cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = (size + gran - 1) // gran * gran
        prop.size = size
        self.mc = ok(cu.cuMulticastCreate(prop))
        ok(cu.cuMulticastAddDevice(self.mc, ok(cu.cuDeviceGet(dev))))
        ap = cu.CUmemAllocationProp()
        ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = dev
        self.mem = ok(cu.cuMemCreate(size, ap, 0))
        ok(cu.cuMulticastBindMem(self.mc, 0, self.mem, 0, size, 0))
        acc = cu.CUmemAccessDesc()
        acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uva = ok(cu.cuMemAddressReserve(size, gran, 0, 0))
        ok(cu.cuMemMap(self.uva, size, 0, self.mem, 0))
        ok(cu.cuMemSetAccess(self.uva, size, [acc], 1))
        self.mva = ok(cu.cuMemAddressReserve(size, gran, 0, 0))
        ok(cu.cuMemMap(self.mva, size, 0, self.mc, 0))
        ok(cu.cuMemSetAccess(self.mva, size, [acc], 1))
        self.multicast_ptr = int(self.mva)

        class _Arr:
            pass
        a = _Arr()
        a.__cuda_array_interface__ = {"shape": (words,), "typestr": "<i4", "data": (int(self.uva), False),
                                      "version": 3, "strides": None}
        self.buffer = torch.as_tensor(a, device=torch.device("cuda", dev))

    def barrier(self, channel=0):
        torch.cuda.synchronize()


def multicast_buffer(words: int, device, group=None):
    """A buffer of ``words`` int32 per GPU of the group with its multicast (NVLS) mapping:
    torch symmetric memory (its rendezvous exports the multicast handle to the other ranks),
    else for a group of one a local multicast object; None when neither is available."""
    import torch.distributed._symmetric_memory as symm_mem
    g = group if group is not None else dist.group.WORLD
    key = (g.group_name, words, str(device))
    if key not in _MC:
        buf = symm_mem.empty(words, dtype=torch.int32, device=device)
        hdl = symm_mem.rendezvous(buf, g.group_name)
        if getattr(hdl, "multicast_ptr", 0):
            _MC[key] = (buf, hdl)
        elif dist.get_world_size(g) == 1:
            try:
                loc = _LocalMulticast(words, device)
                _MC[key] = (loc.buffer, loc)
            except Exception:   # no multicast on this GPU / driver
                _MC[key] = None
        else:
            _MC[key] = None
    return _MC[key]


def sharded_store_nvls(net, msgs_shard, group=None, stream=None):
    """The NVLS form of sharded_store_bits: each rank stores its shard, seals
    (packing the partial Wb) and copies Wb into its symmetric buffer; after a barrier, one
    kernel per rank (gb_or_bits_multimem) reads the OR of all ranks' partials through the
    multicast address -- reduced inside the NVSwitch -- into its cleared W8; seal.  No data
    moves through NCCL.  Returns False (nothing done) when the group has no multicast support."""
    mc = multicast_buffer(net.n_padded * net.nw, torch.device("cuda", net.device), group)
    if mc is None:
        return False
    buf, hdl = mc
    net.clear(stream)
    if msgs_shard.shape[0]:
        net.store(msgs_shard, stream)
    net.seal(stream, check=False)
    buf.view(net.n_padded, net.nw).copy_(net.bits())
    hdl.barrier(channel=0)                 # every rank's partial is in place
    net.clear(stream)
    net.or_bits_multimem(hdl.multicast_ptr, stream)
    hdl.barrier(channel=0)                 # every rank has read the partials (buffer reusable)
    net.seal(stream, check=False)
    return True
