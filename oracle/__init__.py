"""CPU oracle for GBNN store/decode (arXiv:1303.7032) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA path (``paper_1303_7032_b200``) and never imports it.

The arithmetic lives in ``gb_oracle.c`` (plain literal loops over 0/1 byte
arrays, one function per paper passage; see its header).  This file only
compiles/loads it and marshals numpy arrays.

Parity status per function (DESIGN.md §"Oracle pins"):
  store        pinned: PAPER.md L497-508 printed W; numpy X^T X identity;
               Python-set edge count; density closed form 1-(1-1/L^2)^M.
  decode SOS   pinned: PAPER.md L515-522 trajectory (gamma=1), gamma=2
               convergence (L525), numpy score identity, fixed points,
               single-clique and M=0 closed cases; on random instances at the
               Scenario-1 shape every round equals the library contraction
               (W + gamma I) V + per-cluster max/== and the stopping rule of
               Alg. 1 (test_sos_decode_is_composed_library_rounds).
  decode SOM   pinned: Thm 1 (Python bail-out-early), gamma invariance,
               brute-force greatest self-supporting subset, Lemmas 1-3,
               PAPER.md L668-669 pool example.
  decode HYB   pinned: F2 (== SOM on clique-consistent probes), F3 prune
               identity, brute-force frozen-known fixed point, e=0 / e=C.
  work counter pinned (``with_blocks=True``): equals an independent
               walk-by-walk replay of PAPER.md L445-451 (tests/brute.py
               decode_work) on random tiny instances, and the closed forms
               for M=0 and a single stored clique (SOM, hybrid); SOS counts
               rounds.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

SOS, SOM, HYBRID = 0, 1, 2
CONVERGED, MAX_ITERS, INVALID, CYCLE = 0, 1, 2, 3
CYCLE_EXIT = 1   # flag: stop an oscillating SOS probe at V^r == V^{r-2} (N4)
ERASED = 0xFFFF
AMBIGUOUS = 0xFFFE

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gb_oracle.c")
_LIB = os.path.join(_HERE, "libgb_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile gb_oracle.c with gcc -O2 -fopenmp (the checker, not the product)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fopenmp", "-fPIC", "-shared",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        lib.oracle_store.argtypes = [P, i32, i32, P, i64]
        lib.oracle_store.restype = i64
        lib.oracle_decode.argtypes = [P, i32, i32, P, i64, i32, i32, i32, P, P, P, P]
        lib.oracle_decode.restype = i32
        lib.oracle_decode_flags.argtypes = [P, i32, i32, P, i64, i32, i32, i32, i32, P, P, P, P]
        lib.oracle_decode_flags.restype = i32
        lib.oracle_sos_trace.argtypes = [P, i32, i32, P, i32, i32, P, P]
        lib.oracle_sos_trace.restype = i32
        lib.oracle_som_step.argtypes = [P, i32, i32, P, i32, P]
        lib.oracle_som_step.restype = i32
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def words_per_cluster(l: int) -> int:
    return (l + 31) // 32


def store(msgs: np.ndarray, c: int, l: int, w: np.ndarray | None = None):
    """OR the cliques of ``msgs`` (uint16 [M, C]) into W (u8 [n, n]).

    Returns (W, n_invalid).  PAPER.md L149-153, Eq.(1).
    """
    n = c * l
    if w is None:
        w = np.zeros((n, n), dtype=np.uint8)
    msgs = np.ascontiguousarray(msgs, dtype=np.uint16).reshape(-1, c)
    bad = _load().oracle_store(_ptr(w), c, l, _ptr(msgs), msgs.shape[0])
    return w, int(bad)


def decode(w: np.ndarray, c: int, l: int, probes: np.ndarray, rule: int,
           gamma: int = 2, max_iters: int = 20, with_blocks: bool = False, flags: int = 0):
    """Decode probes (uint16 [K, C], 0xFFFF = erased) under ``rule``.

    Returns (state uint32 [K, C*Wc], iters uint16 [K], status uint8 [K]
    [, blocks int64 [K]]).
    """
    probes = np.ascontiguousarray(probes, dtype=np.uint16).reshape(-1, c)
    k = probes.shape[0]
    nw = c * words_per_cluster(l)
    w = np.ascontiguousarray(w, dtype=np.uint8)
    assert w.shape == (c * l, c * l)
    state = np.zeros((k, nw), dtype=np.uint32)
    iters = np.zeros(k, dtype=np.uint16)
    status = np.zeros(k, dtype=np.uint8)
    blocks = np.zeros(k, dtype=np.int64) if with_blocks else None
    rc = _load().oracle_decode_flags(_ptr(w), c, l, _ptr(probes), k, rule, gamma, max_iters, flags,
                                     _ptr(state), _ptr(iters), _ptr(status),
                                     _ptr(blocks) if with_blocks else None)
    if rc != 0:
        raise ValueError("oracle_decode: invalid arguments")
    if with_blocks:
        return state, iters, status, blocks
    return state, iters, status


def sos_trace(w: np.ndarray, c: int, l: int, v0: np.ndarray, gamma: int, rounds: int):
    """Literal SOS trajectory: (S int64 [rounds, n], V u8 [rounds+1, n])."""
    n = c * l
    v0 = np.ascontiguousarray(v0, dtype=np.uint8)
    s = np.zeros((rounds, n), dtype=np.int64)
    v = np.zeros((rounds + 1, n), dtype=np.uint8)
    _load().oracle_sos_trace(_ptr(np.ascontiguousarray(w, dtype=np.uint8)), c, l, _ptr(v0),
                             gamma, rounds, _ptr(s), _ptr(v))
    return s, v


def som_step(w: np.ndarray, c: int, l: int, v: np.ndarray, gamma: int) -> np.ndarray:
    """One literal Eq.(6)-(7) step on a 0/1 state (u8 [n])."""
    v = np.ascontiguousarray(v, dtype=np.uint8)
    out = np.zeros_like(v)
    _load().oracle_som_step(_ptr(np.ascontiguousarray(w, dtype=np.uint8)), c, l, _ptr(v),
                            gamma, _ptr(out))
    return out


def unpack_state(state: np.ndarray, c: int, l: int) -> np.ndarray:
    """Cluster-padded bit words -> u8 [K, n] 0/1 (harness formatting)."""
    wc = words_per_cluster(l)
    state = np.asarray(state, dtype=np.uint32).reshape(-1, c, wc)
    bits = ((state[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(np.uint8)
    return bits.reshape(state.shape[0], c, wc * 32)[:, :, :l].reshape(state.shape[0], c * l)


def symbols(state: np.ndarray, c: int, l: int) -> np.ndarray:
    """Retrieved message of each final state (R16): per
    cluster the index of its only active neuron, ERASED when none is active, AMBIGUOUS
    when several are.  uint16 [K, C].  Plain count over the unpacked 0/1 state."""
    v = unpack_state(state, c, l).reshape(-1, c, l)
    out = np.empty(v.shape[:2], dtype=np.uint16)
    for k in range(v.shape[0]):
        for cc in range(c):
            on = np.flatnonzero(v[k, cc])
            out[k, cc] = ERASED if on.size == 0 else (on[0] if on.size == 1 else AMBIGUOUS)
    return out


def onehot(msgs: np.ndarray, c: int, l: int) -> np.ndarray:
    """u8 [K, n] one-hot encoding of full messages."""
    msgs = np.asarray(msgs).reshape(-1, c)
    out = np.zeros((msgs.shape[0], c * l), dtype=np.uint8)
    for cc in range(c):
        out[np.arange(msgs.shape[0]), cc * l + msgs[:, cc].astype(np.int64)] = 1
    return out
