"""Brute-force references that pin the oracle (independent of oracle/ code).

Each function restates a property the paper (or SURVEY.md §8c's derived
facts F1-F3) fixes, implemented a different way from the oracle's literal
synchronous iteration:

* ``edges_from_set``    -- W as a Python set of (i, j) pairs (Eq.(1)).
* ``bail_out_early``    -- the per-neuron cluster walk of PAPER.md L445-451
                           with the Q8 reading (the neuron itself must be on).
* ``self_supporting``   -- every active neuron has an active neighbour in
                           every other cluster (fixed-point condition of
                           Eq.(6)-(7) with gamma > 0).
* ``greatest_ss_enum``  -- union of all self-supporting subsets of X
                           (exhaustive; |X| <= ~14).  F1.
* ``peel``              -- worklist removal in arbitrary order until stable
                           (greatest fixed point; Knaster-Tarski).  F1.
* ``consistent_cliques``-- stored messages agreeing with the probe (Lemma 3).
"""
from __future__ import annotations

import itertools

import numpy as np


def edges_from_set(msgs, c, l):
    edges = set()
    for m in np.asarray(msgs).reshape(-1, c).tolist():
        for a in range(c):
            for b in range(c):
                if a != b:
                    edges.add((a * l + m[a], b * l + m[b]))
    return edges


def bail_out_early(w, c, l, v, i):
    """thread i walks clusters 1..C; own cluster adds 1
    directly (for an active neuron, reading Q8); another cluster adds 1 at
    the first active neighbour; the first silent cluster stops the walk."""
    if not v[i]:
        return 0
    ci = i // l
    score = 0
    for cc in range(c):
        if cc == ci:
            score += 1
            continue
        hit = False
        for j in range(cc * l, cc * l + l):
            if w[j, i] > 0 and v[j] > 0:
                hit = True
                break
        if not hit:
            return 0
        score += 1
    return int(score == c)


def has_support(w, c, l, s, i, cc):
    return any(s[j] and w[j, i] for j in range(cc * l, cc * l + l))


def self_supporting(w, c, l, s, frozen=()):
    """True iff every active non-frozen neuron of s has an active neighbour
    in every other cluster."""
    for i in np.flatnonzero(s):
        if (i // l) in frozen:
            continue
        for cc in range(c):
            if cc != i // l and not has_support(w, c, l, s, i, cc):
                return False
    return True


def greatest_ss_enum(w, c, l, x, frozen=()):
    """Union of all self-supporting S with frozen part of x <= S <= x."""
    x = np.asarray(x, dtype=np.uint8)
    free = [i for i in np.flatnonzero(x) if (i // l) not in frozen]
    fixed = [i for i in np.flatnonzero(x) if (i // l) in frozen]
    union = np.zeros_like(x)
    for r in range(len(free) + 1):
        for sub in itertools.combinations(free, r):
            s = np.zeros_like(x)
            s[list(sub) + fixed] = 1
            if self_supporting(w, c, l, s, frozen):
                union |= s
    return union


def peel(w, c, l, x, frozen=(), seed=0):
    """Remove unsupported (non-frozen) neurons one at a time, in a random
    order, until none is unsupported."""
    rng = np.random.default_rng(seed)
    s = np.asarray(x, dtype=np.uint8).copy()
    changed = True
    while changed:
        changed = False
        idx = np.flatnonzero(s)
        rng.shuffle(idx)
        for i in idx:
            if (i // l) in frozen:
                continue
            for cc in range(c):
                if cc != i // l and not has_support(w, c, l, s, i, cc):
                    s[i] = 0
                    changed = True
                    break
    return s


def consistent_cliques(msgs, probe, erased=0xFFFF):
    out = []
    for m in np.asarray(msgs).tolist():
        if all(p == erased or p == mm for p, mm in zip(probe, m)):
            out.append(m)
    return out


# ---------------------------------------------------------------- work counter
def walk_blocks(w, c, l, v, i, scope):
    """L-bit blocks thread i examines in one bail-out-early walk (PAPER.md
    L445-451): clusters in ``scope`` other than c(i), ascending; the cluster
    that contributes no signal is examined and stops the walk.  Returns
    (blocks, survived)."""
    ci = i // l
    blocks = 0
    for cc in range(c):
        if cc == ci or cc not in scope:
            continue
        blocks += 1
        if not has_support(w, c, l, v, i, cc):
            return blocks, False
    return blocks, True


def decode_work(w, c, l, probe, rule, max_iters=200, erased=0xFFFF):
    """Blocks read by a whole SOM (rule 1) or hybrid (rule 2) decode, walk by
    walk: every round, every active in-scope neuron walks (SOM: all clusters;
    hybrid: the erased clusters, Alg. 2, with the (C-e)*e blocks of
    the known rows its prune reads, Alg. 2).  The next state is read
    off the walks themselves (a neuron stays iff its walk completes), so this
    shares nothing with the oracle's Eq.(6)-(7) sum.  Returns (blocks, rounds)."""
    probe = list(probe)
    known = [cc for cc in range(c) if probe[cc] != erased]
    er = [cc for cc in range(c) if probe[cc] == erased]
    v = np.zeros(c * l, np.uint8)
    for cc in known:
        if probe[cc] >= l:
            return 0, 0
        v[cc * l + probe[cc]] = 1
    blocks = 0
    if rule == 1:
        for cc in er:
            v[cc * l:(cc + 1) * l] = 1
        scope, movable = set(range(c)), set(range(c))
    else:
        if not er:
            return 0, 0
        for cc in er:
            col = np.ones(l, np.uint8)
            for k in known:
                col &= w[k * l + probe[k], cc * l:(cc + 1) * l]
            v[cc * l:(cc + 1) * l] = col
        blocks += len(known) * len(er)
        scope, movable = set(er), set(er)
    for r in range(1, max_iters + 1):
        vn = v.copy()
        for i in np.flatnonzero(v):
            if i // l not in movable:
                continue
            b, ok = walk_blocks(w, c, l, v, i, scope)
            blocks += b
            if not ok:
                vn[i] = 0
        if (vn == v).all():
            return blocks, r
        v = vn
    return blocks, max_iters
