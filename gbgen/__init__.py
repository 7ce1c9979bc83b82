"""Seeded synthetic inputs for the GBNN hot path (test + bench harness).

This module is the ONE piece shared by the oracle side (``oracle/``, tests) and
the CUDA side (``paper_1303_7032_b200``, bench).  It holds none of the
method's arithmetic: no clique storage, no scores, no retrieval rule.  It only
draws counter-based random numbers shaped like the paper's workloads:

* messages: C symbols iid uniform in [0, L)  (Scenario 1:
  "8 symbols uniformly sampled from the integers 1 to 128"; 0-based here,
  DESIGN.md reading R1);
* probes: a stored message drawn with replacement (reading R15),
  with e clusters erased, the erased set a uniform e-subset per probe
  ("erase some parts of them"; reading R12);
* optionally a slice of random, non-stored probes (reading R15).

Generator: x_{s,t,i} = splitmix64(seed ^ (t << 56) ^ i), with
streams t = 0 message symbols, 1 probe-source index, 2 erasure choice,
3 random non-stored probe symbols.  Pure numpy uint64 arithmetic (wraps mod
2^64), vectorised and chunked so 10^7 probes fit in a few hundred MB.
"""
from __future__ import annotations

import numpy as np

ERASED = 0xFFFF

_C1 = np.uint64(0x9E3779B97F4A7C15)
_C2 = np.uint64(0xBF58476D1CE4E5B9)
_C3 = np.uint64(0x94D049BB133111EB)
_CHUNK = 1 << 20


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vigna's splitmix64 finaliser applied elementwise to uint64 counters."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64, copy=True) + _C1
        z = (z ^ (z >> np.uint64(30))) * _C2
        z = (z ^ (z >> np.uint64(27))) * _C3
        return z ^ (z >> np.uint64(31))


def stream(seed: int, t: int, start: int, count: int) -> np.ndarray:
    """x_{seed,t,i} for i in [start, start+count)."""
    base = np.uint64((seed ^ (t << 56)) & 0xFFFFFFFFFFFFFFFF)
    idx = np.arange(start, start + count, dtype=np.uint64)
    return splitmix64(base ^ idx)


def messages(seed: int, m: int, c: int, l: int) -> np.ndarray:
    """M messages of C symbols, iid uniform in [0, L).  uint16 [M, C]."""
    if not (c >= 1 and 1 <= l < ERASED):
        raise ValueError("need c >= 1 and 1 <= l < 65535")
    out = np.empty((m, c), dtype=np.uint16)
    flat = out.reshape(-1)
    for s in range(0, m * c, _CHUNK):
        n = min(_CHUNK, m * c - s)
        flat[s:s + n] = (stream(seed, 0, s, n) % np.uint64(l)).astype(np.uint16)
    return out


def erasure_masks(seed: int, k: int, c: int, e, start: int = 0) -> np.ndarray:
    """bool [k, C]: True where the cluster is erased.

    Partial Fisher-Yates over the C clusters per probe: for j < e_k swap
    perm[j] with perm[j + (x_{2, k*C+j} mod (C-j))]; the first e_k entries of
    perm are erased.  ``e`` is an int or an int array of per-probe counts.
    """
    e_arr = np.broadcast_to(np.asarray(e, dtype=np.int64), (k,))
    if k and (e_arr.min() < 0 or e_arr.max() > c):
        raise ValueError("erasure count must lie in [0, C]")
    perm = np.broadcast_to(np.arange(c, dtype=np.int64), (k, c)).copy()
    flat = perm.reshape(-1)
    base = np.arange(k, dtype=np.int64) * c
    emax = int(e_arr.max()) if k else 0
    uniform = bool(k) and int(e_arr.min()) == emax
    ctr = (np.arange(start, start + k, dtype=np.uint64) * np.uint64(c)) if emax else None
    sbase = np.uint64((seed ^ (2 << 56)) & 0xFFFFFFFFFFFFFFFF)
    for j in range(emax):
        xj = splitmix64(sbase ^ (ctr + np.uint64(j)))          # x_{seed,2,k*C+j}
        r = (xj % np.uint64(c - j)).astype(np.int64)
        src = base + j + r
        a = flat[base + j].copy()
        b = flat[src]
        if uniform:
            flat[base + j] = b
            flat[src] = a
        else:
            act = j < e_arr
            flat[(base + j)[act]] = b[act]
            flat[src[act]] = a[act]
    mask = np.zeros((k, c), dtype=bool)
    mflat = mask.reshape(-1)
    for j in range(emax):
        if uniform:
            mflat[base + perm[:, j]] = True
        else:
            act = j < e_arr
            mflat[(base + perm[:, j])[act]] = True
    return mask


def probes(seed: int, msgs: np.ndarray, k: int, e, l: int,
           random_count: int = 0, start: int = 0):
    """K probes: stored messages (with replacement) with e clusters erased.

    The last ``random_count`` probes are random non-stored words (stream 3)
    erased the same way.  ``start`` offsets the global probe counter, so a
    shard [start, start+K) of a larger batch is generated identically on any
    rank.  Returns (probes uint16 [K, C], source int64 [K]; source = -1 for
    random probes).
    """
    m, c = msgs.shape
    if k and m == 0 and random_count < k:
        raise ValueError("no stored messages to draw probes from")
    out = np.empty((k, c), dtype=np.uint16)
    src = np.empty(k, dtype=np.int64)
    e_arr = np.broadcast_to(np.asarray(e, dtype=np.int64), (k,))
    n_stored = k - random_count
    for s in range(0, k, _CHUNK):
        n = min(_CHUNK, k - s)
        idx = np.arange(s, s + n)
        stored = idx < n_stored
        blk = np.empty((n, c), dtype=np.uint16)
        sblk = np.full(n, -1, dtype=np.int64)
        if stored.any():
            ns = int(stored.sum())
            pick = (stream(seed, 1, start + s, ns) % np.uint64(m)).astype(np.int64)
            blk[:ns] = msgs[pick]
            sblk[:ns] = pick
        if (~stored).any():
            nr = int((~stored).sum())
            r0 = start + s + n - nr
            sym = stream(seed, 3, r0 * c, nr * c) % np.uint64(l)
            blk[n - nr:] = sym.astype(np.uint16).reshape(nr, c)
        mask = erasure_masks(seed, n, c, e_arr[s:s + n], start=start + s)
        blk[mask] = ERASED
        out[s:s + n] = blk
        src[s:s + n] = sblk
    return out, src
