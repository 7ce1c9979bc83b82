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
* alternatively W is built once and replicated with a broadcast.
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
    if dist.is_initialized():
        dist.all_reduce(w8, op=dist.ReduceOp.MAX, group=group)
    return w8


def broadcast_weights_(w8: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    if dist.is_initialized():
        dist.broadcast(w8, src=src, group=group)
    return w8


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
    """gb_clear + gb_store(shard) + MAX merge + gb_seal on one rank."""
    net.clear(stream)
    if msgs_shard.shape[0]:
        net.store(msgs_shard, stream)
    merge_weights_(net.weights(), group)
    net.seal(stream)


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


def sharded_store_bits(net, msgs_shard, group=None, stream=None):
    """gb_clear + gb_store(shard) + gb_seal (pack the partial) + all-gather of
    the packed partials + gb_or_bits + gb_seal on one rank (N3 merge)."""
    net.clear(stream)
    if msgs_shard.shape[0]:
        net.store(msgs_shard, stream)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        net.seal(stream)
        allb = gather_bits(net.bits(), group)
        net.or_bits(allb, stream)
    net.seal(stream)
