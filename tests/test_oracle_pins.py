"""Pin the CPU oracle to what the paper and the mathematics fix (CPU only).

Every test names the passage (PAPER.md line / equation / theorem) or the
SURVEY.md §8c derived fact it checks.  None of them re-types the oracle's
loops: they use printed values, closed forms, numpy library routines, or the
independent brute-force code in tests/brute.py.
"""
import numpy as np
import pytest

import gbgen
import oracle
from oracle import SOS, SOM, HYBRID, CONVERGED, MAX_ITERS, INVALID, ERASED
from tests import brute
from tests.helpers import load_golden


# ---------------------------------------------------------------- fixtures
def va_network():
    g = load_golden("va_oscillation.txt")
    msgs = np.array([[int(t) - 1 for t in row] for row in g["messages"]], dtype=np.uint16)
    w_printed = np.array([[int(t) for t in row] for row in g["W"]], dtype=np.int64)
    traj = {k: np.array([int(t) for t in g[k][0]], dtype=np.int64)
            for k in ("v0", "s0", "v1", "s1", "v2", "s2", "v3")}
    return msgs, w_printed, traj


def rand_instance(seed, c, l, m):
    msgs = gbgen.messages(seed, m, c, l)
    w, bad = oracle.store(msgs, c, l)
    assert bad == 0
    return msgs, w


# ---------------------------------------------------------------- encoding
def test_message_code_paper_l154():
    """(9,4,3,10) at C=4, L=16 -> printed bit string.
    The oracle's e=0 hybrid decode returns the probe's one-hot code in the
    canonical packed layout; unpack and compare with the printed string."""
    g = load_golden("message_code.txt")
    msg = np.array([[int(t) - 1 for t in g["message"][0]]], dtype=np.uint16)
    code = "".join(g["code"][0])
    w = np.zeros((64, 64), dtype=np.uint8)
    st, it, ss = oracle.decode(w, 4, 16, msg, HYBRID, gamma=1)
    bits = oracle.unpack_state(st, 4, 16)[0]
    assert "".join(str(b) for b in bits) == code
    assert it[0] == 0 and ss[0] == CONVERGED


# ---------------------------------------------------------------- store
def test_store_matches_printed_va_matrix():
    """storing the 4 messages gives the printed W
    (gamma=1 on the printed diagonal; the stored part is W - I)."""
    msgs, w_printed, _ = va_network()
    w, bad = oracle.store(msgs, 3, 3)
    assert bad == 0
    np.testing.assert_array_equal(w.astype(np.int64) + np.eye(9, dtype=np.int64), w_printed)


@pytest.mark.parametrize("c,l,m", [(4, 16, 50), (3, 5, 12), (8, 32, 300), (5, 7, 0)])
def test_store_library_identity_and_set(c, l, m):
    """F4: W = [X^T X > 0] with intra-cluster blocks zeroed (numpy matmul);
    edge count = number of distinct (i, j) tuples (Python set); symmetric
    (PAPER.md L306 w_ij = w_ji); zero intra-cluster blocks (L145)."""
    msgs, w = rand_instance(100 + m, c, l, m)
    x = oracle.onehot(msgs, c, l).astype(np.int64) if m else np.zeros((0, c * l), np.int64)
    ref = (x.T @ x > 0).astype(np.uint8)
    for cc in range(c):
        ref[cc * l:(cc + 1) * l, cc * l:(cc + 1) * l] = 0
    np.testing.assert_array_equal(w, ref)
    edges = brute.edges_from_set(msgs, c, l)
    assert int(w.sum()) == len(edges)
    assert all(w[i, j] == 1 for i, j in edges)
    np.testing.assert_array_equal(w, w.T)
    for cc in range(c):
        assert not w[cc * l:(cc + 1) * l, cc * l:(cc + 1) * l].any()


def test_store_idempotent_commutative_and_invalid():
    """S:L182 / Eq.(1) OR semantics: storing twice or in another order
    gives the same W; a message with a symbol >= L stores nothing and is
    counted."""
    msgs, w = rand_instance(7, 4, 16, 40)
    w2, _ = oracle.store(msgs, 4, 16, w.copy())
    np.testing.assert_array_equal(w, w2)
    w3, _ = oracle.store(msgs[::-1].copy(), 4, 16)
    np.testing.assert_array_equal(w, w3)
    bad = np.array([[1, 2, 16, 3]], dtype=np.uint16)
    w4, nbad = oracle.store(bad, 4, 16, w.copy())
    assert nbad == 1
    np.testing.assert_array_equal(w4, w)


@pytest.mark.parametrize("c,l,m", [(4, 16, 50), (8, 128, 5000), (8, 128, 20000)])
def test_store_density_closed_form(c, l, m):
    """F6: per cluster-pair block the number of set pairs is the occupancy of
    L^2 cells by M uniform throws: mean L^2(1-(1-1/L^2)^M), variance
    L^2(L^2-1)(1-2/L^2)^M + L^2(1-1/L^2)^M - L^4(1-1/L^2)^{2M}
    (iid uniform symbols).  Every block within 5 sigma."""
    msgs, w = rand_instance(4242, c, l, m)
    q = l * l
    mean = q * (1 - (1 - 1 / q) ** m)
    var = q * (q - 1) * (1 - 2 / q) ** m + q * (1 - 1 / q) ** m - q * q * (1 - 1 / q) ** (2 * m)
    sd = max(np.sqrt(var), 1e-9)
    tot = 0
    for a in range(c):
        for b in range(a + 1, c):
            cnt = int(w[a * l:(a + 1) * l, b * l:(b + 1) * l].sum())
            tot += cnt
            assert abs(cnt - mean) <= 5 * sd + 1e-9, (a, b, cnt, mean, sd)
    pairs = c * (c - 1) // 2
    dens = tot / (pairs * q)
    assert abs(dens - (1 - (1 - 1 / q) ** m)) <= 5 * sd * np.sqrt(pairs) / (pairs * q) + 1e-12


# ---------------------------------------------------------------- SOS
def test_sos_oscillation_trajectory_paper_l515():
    """gamma=1, probe (?,?,1): s^0, v^1, s^1, v^2, s^2,
    v^3 exactly as printed and v^3 == v^1 (oscillation)."""
    msgs, _, t = va_network()
    w, _ = oracle.store(msgs, 3, 3)
    s, v = oracle.sos_trace(w, 3, 3, t["v0"].astype(np.uint8), 1, 3)
    np.testing.assert_array_equal(s[0], t["s0"])
    np.testing.assert_array_equal(v[1], t["v1"])
    np.testing.assert_array_equal(s[1], t["s1"])
    np.testing.assert_array_equal(v[2], t["v2"])
    np.testing.assert_array_equal(s[2], t["s2"])
    np.testing.assert_array_equal(v[3], t["v3"])
    np.testing.assert_array_equal(v[3], v[1])


@pytest.mark.parametrize("T", [1, 2, 3, 19, 20])
def test_sos_oscillation_decode_never_converges(T):
    """PAPER.md L522 "oscillating between v^2 and v^3 forever": the batch
    decode runs to the cap; V^T is v^1 for odd T and v^2 for even T
    (readings R5-R7)."""
    msgs, _, t = va_network()
    w, _ = oracle.store(msgs, 3, 3)
    probe = np.array([[ERASED, ERASED, 0]], dtype=np.uint16)
    st, it, ss = oracle.decode(w, 3, 3, probe, SOS, gamma=1, max_iters=T)
    assert ss[0] == MAX_ITERS and it[0] == T
    want = t["v1"] if T % 2 else t["v2"]
    np.testing.assert_array_equal(oracle.unpack_state(st, 3, 3)[0], want)


@pytest.mark.parametrize("T", [3, 4, 20])
def test_sos_cycle_exit_paper_l515(T):
    """N4 cycle exit (flag-gated): on the printed oscillation of
    PAPER.md L515-517 (gamma=1, v^3 == v^1 != v^2) the probe stops at round 3
    with status CYCLE and state v^3 = v^1 (printed); with T < 3 the cap wins;
    gamma=2 (L525) still converges in 3 rounds; SOM/hybrid are unaffected."""
    msgs, _, t = va_network()
    w, _ = oracle.store(msgs, 3, 3)
    probe = np.array([[ERASED, ERASED, 0]], dtype=np.uint16)
    st, it, ss = oracle.decode(w, 3, 3, probe, SOS, gamma=1, max_iters=T, flags=oracle.CYCLE_EXIT)
    assert ss[0] == oracle.CYCLE and it[0] == 3
    np.testing.assert_array_equal(oracle.unpack_state(st, 3, 3)[0], t["v3"])
    np.testing.assert_array_equal(oracle.unpack_state(st, 3, 3)[0], t["v1"])
    st, it, ss = oracle.decode(w, 3, 3, probe, SOS, gamma=1, max_iters=2, flags=oracle.CYCLE_EXIT)
    assert ss[0] == MAX_ITERS and it[0] == 2
    np.testing.assert_array_equal(oracle.unpack_state(st, 3, 3)[0], t["v2"])
    st, it, ss = oracle.decode(w, 3, 3, probe, SOS, gamma=2, max_iters=T, flags=oracle.CYCLE_EXIT)
    assert ss[0] == CONVERGED and it[0] == 3
    for rule in (SOM, HYBRID):
        a = oracle.decode(w, 3, 3, probe, rule, gamma=1, max_iters=T, flags=oracle.CYCLE_EXIT)
        b = oracle.decode(w, 3, 3, probe, rule, gamma=1, max_iters=T)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


def test_sos_cycle_exit_is_the_literal_run_stopped_early():
    """The cycle-exit result of every probe equals the literal (flag-free) run
    cut at the exit round: same state at T = exit round, and a literal run of
    exit+2j rounds returns the same state (period 2)."""
    rng_seed = 11
    c, l = 5, 6
    msgs, w = rand_instance(rng_seed, c, l, 25)
    pr, _ = gbgen.probes(rng_seed + 1, msgs, 300, 3, l, random_count=100)
    st, it, ss = oracle.decode(w, c, l, pr, SOS, gamma=0, max_iters=20, flags=oracle.CYCLE_EXIT)
    cyc = np.flatnonzero(ss == oracle.CYCLE)
    assert cyc.size > 0   # gamma=0 oscillates often on this instance
    for i in cyc[:40]:
        r = int(it[i])
        for T in (r, r + 2, r + 4):
            s2, i2, q2 = oracle.decode(w, c, l, pr[i:i + 1], SOS, gamma=0, max_iters=T)
            assert q2[0] == MAX_ITERS and i2[0] == T
            np.testing.assert_array_equal(s2[0], st[i])
        s3, _, _ = oracle.decode(w, c, l, pr[i:i + 1], SOS, gamma=0, max_iters=r - 1)
        assert not np.array_equal(s3[0], st[i])
    rest = np.flatnonzero(ss != oracle.CYCLE)
    s4, i4, q4 = oracle.decode(w, c, l, pr[rest], SOS, gamma=0, max_iters=20)
    np.testing.assert_array_equal(s4, st[rest])
    np.testing.assert_array_equal(i4, it[rest])
    np.testing.assert_array_equal(q4, ss[rest])


def test_sos_gamma2_converges_paper_l525():
    """PAPER.md L525 "If we increase gamma = 2, then the network converges".
    Hand-derived: v^1 = (1,1,1,1,1,1,1,0,0), s^1 = (5,4,4,4,5,4,8,0,0),
    v^2 = (1,0,0,0,1,0,1,0,0), s^2 = (3,2,2,2,3,2,4,0,0), v^3 = v^2:
    CONVERGED after 3 rounds to (1,2,1) (1-based)."""
    msgs, _, t = va_network()
    w, _ = oracle.store(msgs, 3, 3)
    s, v = oracle.sos_trace(w, 3, 3, t["v0"].astype(np.uint8), 2, 3)
    np.testing.assert_array_equal(s[1], [5, 4, 4, 4, 5, 4, 8, 0, 0])
    np.testing.assert_array_equal(s[2], [3, 2, 2, 2, 3, 2, 4, 0, 0])
    probe = np.array([[ERASED, ERASED, 0]], dtype=np.uint16)
    st, it, ss = oracle.decode(w, 3, 3, probe, SOS, gamma=2, max_iters=20)
    assert ss[0] == CONVERGED and it[0] == 3
    np.testing.assert_array_equal(oracle.unpack_state(st, 3, 3)[0], [1, 0, 0, 0, 1, 0, 1, 0, 0])


@pytest.mark.parametrize("gamma", [0, 1, 2, 5])
def test_sos_score_is_library_matmul(gamma):
    """F5 / Eq.(10)-(11): the SOS score is S = (W + gamma I) V, checked
    against numpy int64 matmul on random states; Eq.(4)-(5) selection checked
    against numpy max/== per cluster."""
    c, l = 4, 16
    msgs, w = rand_instance(11, c, l, 60)
    rng = np.random.default_rng(5)
    for _ in range(10):
        v0 = (rng.random(c * l) < 0.2).astype(np.uint8)
        s, v = oracle.sos_trace(w, c, l, v0, gamma, 1)
        ref = (w.astype(np.int64) + gamma * np.eye(c * l, dtype=np.int64)) @ v0.astype(np.int64)
        np.testing.assert_array_equal(s[0], ref)
        blk = ref.reshape(c, l)
        np.testing.assert_array_equal(v[1].reshape(c, l), (blk == blk.max(axis=1, keepdims=True)))


@pytest.mark.parametrize("c,l,m,e,gamma", [(8, 128, 5000, 4, 2), (8, 128, 5000, 5, 1), (4, 16, 60, 2, 0),
                                           (6, 40, 900, 3, 3)])
def test_sos_decode_is_composed_library_rounds(c, l, m, e, gamma):
    """Alg. 1 end to end on random instances at the Scenario-1
    shape: the oracle's SOS decode equals rounds of the library contraction
    S = (W + gamma I) V (numpy int64 matmul, Eq.(10)-(11)) followed by the
    per-cluster max / == selection (Eq.(4)-(5)), started from V^0 = known
    one-hot, erased 0 and stopped at the first round with
    V^{t+1} == V^t (iters = that round, CONVERGED) or after T rounds
    (MAX_ITERS).  Pins the multi-round trajectories and the stopping rule, not
    only one round."""
    msgs, w = rand_instance(31 + c + e, c, l, m)
    pr, _ = gbgen.probes(32 + e, msgs, 40, e, l, random_count=8)
    T = 12
    st, it, ss = oracle.decode(w, c, l, pr, SOS, gamma=gamma, max_iters=T)
    A = w.astype(np.int64) + gamma * np.eye(c * l, dtype=np.int64)
    got = oracle.unpack_state(st, c, l)
    for i, p in enumerate(pr):
        v = np.zeros(c * l, np.int64)
        for cc in range(c):
            if p[cc] != ERASED:
                v[cc * l + int(p[cc])] = 1
        rounds, status = T, MAX_ITERS
        for r in range(1, T + 1):
            blk = (A @ v).reshape(c, l)
            vn = (blk == blk.max(axis=1, keepdims=True)).astype(np.int64).reshape(-1)
            done = np.array_equal(vn, v)
            v = vn
            if done:
                rounds, status = r, CONVERGED
                break
        assert (int(it[i]), int(ss[i])) == (rounds, status), f"probe {i}"
        np.testing.assert_array_equal(got[i], v, err_msg=f"probe {i}")


def test_fixed_points_and_closed_cases_all_rules():
    """Lemma 2 (L541-548) and closed cases of SURVEY §8c:
    * stored message, e=0, gamma>=1: SOS/SOM 1 round unchanged, hybrid 0;
    * single stored clique, 1<=e<C: SOS 2 rounds exact, SOM 2 rounds exact,
      hybrid 1 round exact; SOM with e=C also 2 rounds exact;
    * M=0, 0<e<C: SOS 2 rounds -> known one-hot + erased all on; SOM 2
      rounds -> empty; hybrid 1 round -> known one-hot, erased empty."""
    c, l = 5, 7
    msgs, w = rand_instance(3, c, l, 30)
    full = msgs[:10]
    oh = oracle.onehot(full, c, l)
    for rule, rounds in ((SOS, 1), (SOM, 1), (HYBRID, 0)):
        st, it, ss = oracle.decode(w, c, l, full, rule, gamma=1)
        np.testing.assert_array_equal(oracle.unpack_state(st, c, l), oh)
        assert (it == rounds).all() and (ss == CONVERGED).all()
    one = gbgen.messages(9, 1, c, l)
    w1, _ = oracle.store(one, c, l)
    for e in range(1, c + 1):
        pr, _ = gbgen.probes(e, one, 4, e, l)
        want = oracle.onehot(np.repeat(one, 4, axis=0), c, l)
        for rule, rounds in ((SOS, 2), (SOM, 2), (HYBRID, 1)):
            if e == c and rule != SOM:
                continue
            st, it, ss = oracle.decode(w1, c, l, pr, rule, gamma=2)
            np.testing.assert_array_equal(oracle.unpack_state(st, c, l), want)
            assert (it == rounds).all() and (ss == CONVERGED).all(), (rule, e, it)
    w0 = np.zeros((c * l, c * l), np.uint8)
    pr, _ = gbgen.probes(1, one, 6, 2, l)
    known = (pr != ERASED)
    st, it, ss = oracle.decode(w0, c, l, pr, SOS, gamma=1)
    v = oracle.unpack_state(st, c, l).reshape(-1, c, l)
    assert (it == 2).all() and (ss == CONVERGED).all()
    for k in range(pr.shape[0]):
        for cc in range(c):
            exp = np.zeros(l, np.uint8)
            if known[k, cc]:
                exp[pr[k, cc]] = 1
            else:
                exp[:] = 1
            np.testing.assert_array_equal(v[k, cc], exp)
    st, it, ss = oracle.decode(w0, c, l, pr, SOM, gamma=1)
    assert (it == 2).all() and not st.any()
    st, it, ss = oracle.decode(w0, c, l, pr, HYBRID, gamma=1)
    assert (it == 1).all()
    v = oracle.unpack_state(st, c, l).reshape(-1, c, l)
    for k in range(pr.shape[0]):
        for cc in range(c):
            exp = np.zeros(l, np.uint8)
            if known[k, cc]:
                exp[pr[k, cc]] = 1
            np.testing.assert_array_equal(v[k, cc], exp)


# ---------------------------------------------------------------- SOM
def test_som_step_equals_bail_out_early_thm1():
    """Theorem 1 (L459-479): bail-out-early (L445-451, Python) produces the
    same v^{t+1} as Eq.(6)-(7) for any gamma > 0; gamma in {1,2,7}."""
    rng = np.random.default_rng(0)
    for trial in range(300):
        c = int(rng.integers(2, 5))
        l = int(rng.integers(1, 6))
        n = c * l
        w = (rng.random((n, n)) < rng.random()).astype(np.uint8)
        w = np.triu(w, 1)
        w = w | w.T
        for cc in range(c):
            w[cc * l:(cc + 1) * l, cc * l:(cc + 1) * l] = 0
        v = (rng.random(n) < rng.random()).astype(np.uint8)
        ref = np.array([brute.bail_out_early(w, c, l, v, i) for i in range(n)], dtype=np.uint8)
        for gamma in (1, 2, 7):
            np.testing.assert_array_equal(oracle.som_step(w, c, l, v, gamma), ref)


def _tiny_cases(n_cases, seed):
    rng = np.random.default_rng(seed)
    for _ in range(n_cases):
        c = int(rng.integers(2, 5))
        l = int(rng.integers(1, 5))
        m = int(rng.integers(0, 10))
        msgs = gbgen.messages(int(rng.integers(1 << 30)), m, c, l)
        w, _ = oracle.store(msgs, c, l)
        e = int(rng.integers(0, c + 1))
        if m and rng.random() < 0.7:
            pr, _ = gbgen.probes(int(rng.integers(1 << 30)), msgs, 1, e, l)
        else:
            pr = gbgen.messages(int(rng.integers(1 << 30)), 1, c, l)
            pr[0, rng.permutation(c)[:e]] = ERASED
        yield c, l, msgs, w, pr, e


def _x0(pr, c, l, erased_on):
    x = np.zeros(c * l, np.uint8)
    for cc in range(c):
        if pr[0, cc] == ERASED:
            x[cc * l:(cc + 1) * l] = erased_on
        else:
            x[cc * l + pr[0, cc]] = 1
    return x


def test_som_greatest_fixed_point_bruteforce_f1():
    """F1: SOM's result is the greatest self-supporting subset of X^0
    (Knaster-Tarski on the monotone deflationary round map).  Checked against
    exhaustive subset enumeration (|X^0| <= 14) and random-order peeling.
    Lemma 1: the number of rounds is <= |X^0| + 1."""
    n_enum = 0
    for c, l, msgs, w, pr, e in _tiny_cases(600, 1):
        x0 = _x0(pr, c, l, 1)
        st, it, ss = oracle.decode(w, c, l, pr, SOM, gamma=1, max_iters=200)
        got = oracle.unpack_state(st, c, l)[0]
        assert ss[0] == CONVERGED and it[0] <= x0.sum() + 1
        np.testing.assert_array_equal(got, brute.peel(w, c, l, x0, seed=int(it[0])))
        if x0.sum() <= 14:
            n_enum += 1
            np.testing.assert_array_equal(got, brute.greatest_ss_enum(w, c, l, x0))
    assert n_enum > 300


def test_som_lemmas_monotone_containment():
    """Lemma 1 (L531-539): active(t+1) <= active(t) along the literal
    trajectory; Lemma 3 (L550-560): every stored message consistent with the
    probe is contained in the final state; Lemma 2: a stored clique is
    stable."""
    for c, l, msgs, w, pr, e in _tiny_cases(300, 2):
        v = _x0(pr, c, l, 1)
        for _ in range(c * l + 2):
            vn = oracle.som_step(w, c, l, v, 1)
            assert not (vn & (1 - v)).any()
            if (vn == v).all():
                break
            v = vn
        for m in brute.consistent_cliques(msgs, pr[0].tolist()):
            oh = oracle.onehot(np.array([m]), c, l)[0]
            assert (v >= oh).all()
            np.testing.assert_array_equal(oracle.som_step(w, c, l, oh, 3), oh)


def test_pool_exception_paper_l668():
    """stored (1,3,1),(1,3,2); probe (1,3,?) keeps both
    neurons 1 and 2 of the erased cluster (SOM and hybrid)."""
    g = load_golden("pool_exception.txt")
    c, l = 3, 4
    msgs = np.array([[int(t) - 1 for t in r] for r in g["messages"]], dtype=np.uint16)
    pr = np.array([[ERASED if t == "?" else int(t) - 1 for t in g["probe"][0]]], dtype=np.uint16)
    want = {int(t) - 1 for t in g["candidates_cluster3"][0]}
    w, _ = oracle.store(msgs, c, l)
    for rule in (SOM, HYBRID):
        st, it, ss = oracle.decode(w, c, l, pr, rule, gamma=1)
        v = oracle.unpack_state(st, c, l)[0].reshape(c, l)
        assert set(np.flatnonzero(v[2]).tolist()) == want
        assert v[0, 0] == 1 and v[1, 2] == 1 and ss[0] == CONVERGED


def test_va_probe_som_and_hybrid():
    """§V-A probe (?,?,1) under SOM and hybrid: one round, final state =
    neurons 1..7 (1-based) = the union of the 4 consistent cliques
    (Lemma 3 + F1)."""
    msgs, _, _ = va_network()
    w, _ = oracle.store(msgs, 3, 3)
    probe = np.array([[ERASED, ERASED, 0]], dtype=np.uint16)
    for rule in (SOM, HYBRID):
        st, it, ss = oracle.decode(w, 3, 3, probe, rule, gamma=1)
        np.testing.assert_array_equal(oracle.unpack_state(st, 3, 3)[0], [1] * 7 + [0, 0])
        assert it[0] == 1 and ss[0] == CONVERGED


# ---------------------------------------------------------------- HYBRID
def test_hybrid_bruteforce_frozen_fixed_point_f2_f3():
    """F3: the prune S^0 == C-e equals the AND of the known neurons' W rows
    (computed here from W directly); the hybrid result is the greatest
    fixed point of the frozen-known map from that X^0 (peeling with known
    clusters frozen, and subset enumeration when small).
    F2: on clique-consistent probes hybrid final == SOM final.
    e = C: hybrid == SOM (state and rounds).  e = 0: 0 rounds."""
    n_f2 = 0
    for c, l, msgs, w, pr, e in _tiny_cases(600, 3):
        st, it, ss = oracle.decode(w, c, l, pr, HYBRID, gamma=1, max_iters=200)
        got = oracle.unpack_state(st, c, l)[0]
        known = [cc for cc in range(c) if pr[0, cc] != ERASED]
        x0 = np.zeros(c * l, np.uint8)
        for cc in range(c):
            if pr[0, cc] != ERASED:
                x0[cc * l + pr[0, cc]] = 1
            else:
                col = np.ones(l, np.uint8)
                for k in known:
                    col &= w[k * l + pr[0, k], cc * l:(cc + 1) * l]
                x0[cc * l:(cc + 1) * l] = col
        if e == 0:
            assert it[0] == 0
            np.testing.assert_array_equal(got, x0)
            continue
        np.testing.assert_array_equal(got, brute.peel(w, c, l, x0, frozen=set(known)))
        if x0.sum() <= 14:
            np.testing.assert_array_equal(got, brute.greatest_ss_enum(w, c, l, x0, frozen=set(known)))
        som_st, som_it, _ = oracle.decode(w, c, l, pr, SOM, gamma=1, max_iters=200)
        if e == c:
            np.testing.assert_array_equal(st, som_st)
            assert it[0] == som_it[0]
        kp = [m for m in brute.consistent_cliques(msgs, pr[0].tolist())]
        if kp:
            n_f2 += 1
            np.testing.assert_array_equal(st, som_st)
    assert n_f2 > 100


def test_invalid_probe_and_arguments():
    """Boundary behaviour shared with the C-ABI: a probe
    symbol >= L (and != erased) gives status INVALID with an empty state;
    gamma = 0 is rejected for SOM/hybrid (Thm 1 needs gamma > 0)."""
    msgs, w = rand_instance(1, 4, 16, 20)
    pr = np.array([[0, 16, ERASED, 3], [0, 1, ERASED, 3]], dtype=np.uint16)
    for rule in (SOS, SOM, HYBRID):
        st, it, ss = oracle.decode(w, 4, 16, pr, rule, gamma=1)
        assert ss[0] == INVALID and it[0] == 0 and not st[0].any()
        assert ss[1] != INVALID
    with pytest.raises(ValueError):
        oracle.decode(w, 4, 16, pr, SOM, gamma=0)
    with pytest.raises(ValueError):
        oracle.decode(w, 4, 16, pr, SOS, gamma=1, max_iters=0)


def test_hybrid_equals_som_on_stored_probes_c8():
    """F2 at the paper's Scenario-1 shape (C=8, L=128):
    on stored-message probes hybrid final == SOM final, and hybrid rounds
    <= SOM rounds (the prune only shrinks the pool, Thm 4)."""
    msgs, w = rand_instance(77, 8, 128, 5000)
    pr, _ = gbgen.probes(78, msgs, 60, 4, 128)
    a = oracle.decode(w, 8, 128, pr, HYBRID, gamma=2)
    b = oracle.decode(w, 8, 128, pr, SOM, gamma=2)
    np.testing.assert_array_equal(a[0], b[0])
    assert (a[1] <= b[1]).all()


# ---------------------------------------------------------------- rates
@pytest.mark.slow
def test_scenario1_rate_bands():
    """PAPER.md L710-713 (Scenario 1: C=8, L=128, M=5000, gamma=2, T=20):
    e=3 both > 0.97 (band >= 0.95); e=5 SOS slightly > 0.5 (band
    [0.45, 0.65]), SOM > 0.90 (band >= 0.87); e=6 SOM > 0.20 (band >= 0.17)
    and above SOS.  Success = unique exact recovery (reading R16).  Hybrid
    success set == SOM success set (F2 / L801)."""
    c, l, m, k = 8, 128, 5000, 500
    msgs, w = rand_instance(2024, c, l, m)
    rates = {}
    for e in (3, 5, 6):
        pr, src = gbgen.probes(3000 + e, msgs, k, e, l)
        oh = oracle.onehot(msgs[src], c, l)
        for rule in (SOS, SOM, HYBRID):
            st, it, ss = oracle.decode(w, c, l, pr, rule, gamma=2, max_iters=20)
            ok = (oracle.unpack_state(st, c, l) == oh).all(axis=1)
            rates[(e, rule)] = ok
    r = {key: v.mean() for key, v in rates.items()}
    assert r[(3, SOS)] >= 0.95 and r[(3, SOM)] >= 0.95
    assert 0.45 <= r[(5, SOS)] <= 0.65 and r[(5, SOM)] >= 0.87
    assert r[(6, SOM)] >= 0.17 and r[(6, SOM)] > r[(6, SOS)]
    for e in (3, 5, 6):
        np.testing.assert_array_equal(rates[(e, SOM)], rates[(e, HYBRID)])


# ---------------------------------------------------------------- work counter (§8c / §8d)
def test_work_counter_equals_bruteforce_walks():
    """The oracle's bail-out work counter (``with_blocks=True``; SURVEY §8c
    "Work counters") equals the blocks examined by an independent walk-by-walk
    replay of PAPER.md L445-451 (tests/brute.py ``decode_work``): SOM walks
    every cluster for every active neuron, hybrid walks the erased clusters
    and adds the (C-e)*e known-row blocks of its prune (Alg. 2).
    The replay's next state comes from the walks themselves (a neuron stays
    iff its walk completes), so it also re-checks the rounds.  SOS counts
    rounds (one dense product each, Eq.(11))."""
    n = 0
    for c, l, msgs, w, pr, e in _tiny_cases(400, 11):
        for rule in (SOM, HYBRID):
            st, it, ss, blk = oracle.decode(w, c, l, pr, rule, gamma=1, max_iters=200, with_blocks=True)
            b, r = brute.decode_work(w, c, l, pr[0], rule)
            assert blk[0] == b and it[0] == r, (c, l, e, rule, blk[0], b, it[0], r)
            n += 1
        st, it, ss, blk = oracle.decode(w, c, l, pr, SOS, gamma=1, max_iters=9, with_blocks=True)
        assert blk[0] == it[0]
    assert n == 800


@pytest.mark.parametrize("c,l", [(8, 128), (5, 7)])
def test_work_counter_closed_forms(c, l):
    """Closed forms of the bail-out-early walk count:
    * M=0, 0<e<C: SOM round 1 walks each of the (C-e) + e*L active neurons one
      block (the first other cluster is silent, W=0), round 2 finds nothing
      active -> C-e+e*L blocks, 2 rounds; hybrid reads only its prune (C-e)*e;
    * one stored clique, 1<=e<=C: SOM round 1 = C(C-1) (clique neurons walk
      every other cluster) + e(L-1) (a non-clique erased neuron has no edge,
      one block), round 2 = C(C-1) -> 2C(C-1)+e(L-1); e=0 -> C(C-1), 1 round;
      hybrid (1<=e<C): prune (C-e)e + e clique neurons walking the e-1 other
      erased clusters = e(C-1)."""
    one = gbgen.messages(5, 1, c, l)
    w1, _ = oracle.store(one, c, l)
    w0 = np.zeros_like(w1)
    for e in range(0, c + 1):
        pr, _ = gbgen.probes(e + 1, one, 3, e, l)
        _, it, _, blk = oracle.decode(w1, c, l, pr, SOM, gamma=1, with_blocks=True)
        want = c * (c - 1) if e == 0 else 2 * c * (c - 1) + e * (l - 1)
        assert (blk == want).all(), (e, blk, want)
        if 1 <= e < c:
            _, it, _, blk = oracle.decode(w1, c, l, pr, HYBRID, gamma=1, with_blocks=True)
            assert (blk == e * (c - 1)).all() and (it == 1).all()
            _, it, _, blk = oracle.decode(w0, c, l, pr, SOM, gamma=1, with_blocks=True)
            assert (blk == c - e + e * l).all() and (it == 2).all()
            _, it, _, blk = oracle.decode(w0, c, l, pr, HYBRID, gamma=1, with_blocks=True)
            assert (blk == (c - e) * e).all() and (it == 1).all()


# ---------------------------------------------------------------- retrieved message (symbols)
def test_symbols_of_onehot_and_ensembles():
    """oracle.symbols (the retrieved message; R16): a one-hot
    state of message m maps back to m exactly (PAPER.md L146-147 encoding), an empty
    cluster to ERASED, a cluster with two active neurons to AMBIGUOUS -- including
    padding-adjacent neurons at a ragged L."""
    for c, l in ((4, 16), (8, 128), (3, 3), (5, 100)):
        msgs = gbgen.messages(3, 50, c, l)
        wc = oracle.words_per_cluster(l)
        st = np.zeros((50, c * wc), np.uint32)
        for k in range(50):
            for cc in range(c):
                s = int(msgs[k, cc])
                st[k, cc * wc + s // 32] |= np.uint32(1 << (s % 32))
        assert np.array_equal(oracle.symbols(st, c, l), msgs)
        assert np.array_equal(oracle.unpack_state(st, c, l), oracle.onehot(msgs, c, l))
        st2 = st.copy()
        st2[0, :wc] = 0                                   # cluster 0 of probe 0 empty
        s1 = (int(msgs[1, 0]) + 1) % l                    # a second neuron in cluster 0 of probe 1
        st2[1, s1 // 32] |= np.uint32(1 << (s1 % 32))
        sym = oracle.symbols(st2, c, l)
        assert sym[0, 0] == oracle.ERASED and sym[1, 0] == oracle.AMBIGUOUS
        assert np.array_equal(sym[2:], msgs[2:]) and np.array_equal(sym[0, 1:], msgs[0, 1:])
