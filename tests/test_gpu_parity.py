"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, bit-exact.

Decoded states, iteration counts and statuses are integer/bit results, so the
bar is exact equality.  Inputs come from gbgen (seeded,
shaped like the paper's workloads).
"""
import os

import numpy as np
import pytest

import gbgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RULES = (0, 1, 2)


@pytest.fixture(scope="module")
def gb():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1303_7032_b200 as pkg
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    return pkg


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda()


def padded_w(w, c, l):
    wc = (l + 31) // 32
    lp = 32 * wc
    out = np.zeros((c * lp, c * lp), np.uint8)
    for a in range(c):
        for b in range(c):
            out[a * lp:a * lp + l, b * lp:b * lp + l] = w[a * l:(a + 1) * l, b * l:(b + 1) * l]
    return out


def make_net(gb, msgs, c, l):
    net = gb.Net(c, l)
    if len(msgs):
        net.store(to_dev(msgs))
    net.seal()
    return net


def gpu_decode(net, probes, rule, gamma, T):
    st, it, ss = net.decode(to_dev(probes), rule, gamma=gamma, max_iters=T)
    torch.cuda.synchronize()
    return (st.cpu().numpy().view(np.uint32), it.cpu().numpy().view(np.uint16), ss.cpu().numpy())


def assert_same(got, want, rule, tag=""):
    st, it, ss = got
    ost, oit, oss = want
    bad = np.flatnonzero((st != ost).any(axis=1) | (it != oit) | (ss != oss))
    assert bad.size == 0, (f"{tag} rule {rule}: {bad.size} mismatching probes, first {bad[:5]}; "
                           f"gpu it={it[bad[:3]]} ss={ss[bad[:3]]} oracle it={oit[bad[:3]]} ss={oss[bad[:3]]}")


# ---------------------------------------------------------------- store
@pytest.mark.parametrize("c,l,m", [(4, 16, 50), (3, 3, 4), (5, 33, 200), (8, 128, 20000),
                                   (16, 256, 100000), (2, 1, 3), (7, 100, 3000)])
def test_store_matches_oracle(gb, c, l, m):
    msgs = gbgen.messages(10 + m, m, c, l)
    w, _ = oracle.store(msgs, c, l)
    net = make_net(gb, msgs, c, l)
    got = net.weights().cpu().numpy()
    np.testing.assert_array_equal(got, padded_w(w, c, l))
    assert net.info() == (c, l, net.n_padded, m)


@pytest.mark.parametrize("c,l,m", [(8, 128, 20000), (16, 512, 60000), (5, 33, 5000), (64, 32, 3000),
                                   (3, 100, 5000), (16, 256, 300000)])
@pytest.mark.parametrize("path", ["privatised", "scatter"])
def test_store_paths_match_oracle(gb, c, l, m, path):
    """Both store kernels (shared-memory bit tiles + apply pass for large
    batches; scattered byte stores, forced with GB_OPT_STORE_SCATTER) give the
    oracle's W (Eq.(1)) byte for byte, accumulate over calls (OR),
    and skip + count messages holding a symbol >= L (reading R21)."""
    msgs = gbgen.messages(77 + m + c, m, c, l)
    bad = msgs[:5].copy()
    bad[0, c - 1] = l
    bad[1, 0] = 0xFFFF
    bad[2, c // 2] = 0xFFFE
    allm = np.concatenate([msgs[: m // 3], bad[:3], msgs[m // 3:]])
    net = gb.Net(c, l, store_scatter=int(path == "scatter"))
    net.store(to_dev(allm[: len(allm) // 2]))
    net.store(to_dev(allm[len(allm) // 2:]))
    with pytest.raises(gb.GBError) as ei:
        net.seal()
    assert ei.value.code == gb.GB_EINVAL and "3 stored message" in str(ei.value)
    w, _ = oracle.store(msgs, c, l)
    np.testing.assert_array_equal(net.weights().cpu().numpy(), padded_w(w, c, l))
    net.close()


@pytest.mark.parametrize("c,l", [(5, 33), (16, 256), (3, 3)])
def test_seal_invariants_every_tile(gb, c, l):
    """gb_seal checks Eq.(1)'s structure (binary entries, w_ij = w_ji P:L306,
    no intra-cluster edge P:L145, no padding edge) on every 32x32 tile: an
    edit anywhere in W8 is caught; the packed rows equal W8 (decode parity)."""
    msgs = gbgen.messages(3, 400, c, l)
    w, _ = oracle.store(msgs, c, l)
    net = make_net(gb, msgs, c, l)
    w8 = net.weights()
    np_ = net.n_padded
    lp = np_ // c
    rng = np.random.default_rng(c * 1000 + l)
    real = [cc * lp + x for cc in range(c) for x in range(l)]
    for _ in range(6):
        i, j = (int(v) for v in rng.choice(real, 2))
        if i // lp == j // lp:
            continue
        old = int(w8[i, j])
        w8[i, j] = 1 - old                       # asymmetric
        with pytest.raises(gb.GBError, match="asymmetric"):
            net.seal()
        w8[j, i] = 1 - old                       # symmetric again: fine
        net.seal()
        w8[i, j] = old
        w8[j, i] = old
        w8[i, j] = 2
        w8[j, i] = 2                             # symmetric but not binary
        with pytest.raises(gb.GBError, match="non-binary"):
            net.seal()
        w8[i, j] = old
        w8[j, i] = old
    net.seal()
    if l < lp:                                   # padding neuron of the last cluster
        p_, q = (c - 1) * lp + l, int(real[0])
        w8[p_, q] = 1
        w8[q, p_] = 1
        with pytest.raises(gb.GBError, match="padding"):
            net.seal()
        w8[p_, q] = 0
        w8[q, p_] = 0
    d = int(real[-1])
    w8[d, d] = 1                                 # diagonal = intra-cluster
    with pytest.raises(gb.GBError, match="intra-cluster"):
        net.seal()
    w8[d, d] = 0
    net.seal()
    np.testing.assert_array_equal(w8.cpu().numpy(), padded_w(w, c, l))


@pytest.mark.parametrize("l,m,k", [(128, 20000, 3001), (100, 5000, 777), (97, 12000, 31), (128, 0, 64),
                                   (128, 30000, 1)])
def test_hyb8_matches_oracle_and_generic(gb, l, m, k):
    """The C=8 hybrid kernel (staged push, TMA-stored output) against the
    oracle and against the generic shared-memory kernel (GB_OPT_HYB8 = 0): ragged
    batch (k not a multiple of 32, k < 32), every erasure count 0..8 (e > 4
    goes to the wide-slot kernel), invalid probes, random non-stored probes."""
    c = 8
    msgs = gbgen.messages(900 + l + m, max(m, 1), c, l)[:m]
    pr, _ = gbgen.probes(901 + k, msgs if m else gbgen.messages(5, 10, c, l), k, 4, l, random_count=k // 5)
    rng = np.random.default_rng(k + l)
    for i in range(0, k, 3):                      # mixed erasure counts per probe
        e = int(rng.integers(0, c + 1))
        row = gbgen.messages(1000 + i, 1, c, l)[0] if rng.random() < 0.5 else pr[i].copy()
        row[row == 0xFFFF] = rng.integers(0, l)
        row[rng.choice(c, e, replace=False)] = 0xFFFF
        pr[i] = row
    if k > 10:
        pr[5, 2] = l                                 # invalid symbol
        pr[7, 0] = 0xFFFE
    w, _ = oracle.store(msgs, c, l) if m else (np.zeros((c * l, c * l), np.uint8), None)
    net = make_net(gb, msgs, c, l)
    dens = w.sum() / max(1, c * (c - 1) * l * l)    # edge density between clusters
    assert net.decode_kernel(2) == ("decode_hyb8r_kernel" if dens > 0.65 else "decode_hyb8_kernel")
    want = oracle.decode(w, c, l, pr, 2, gamma=1, max_iters=20)
    got = gpu_decode(net, pr, 2, 1, 20)
    assert_same(got, want, 2, f"hyb8 l={l} m={m} k={k}")
    net.set_option("hyb8", 0)
    assert net.decode_kernel(2) == "decode_smem_kernel"
    assert_same(gpu_decode(net, pr, 2, 1, 20), want, 2, "generic")
    assert_same(gpu_decode(net, pr, 2, 1, 3), oracle.decode(w, c, l, pr, 2, gamma=1, max_iters=3), 2, "T=3")
    net.set_option("hyb8", 1)
    assert_same(gpu_decode(net, pr, 2, 1, 3), oracle.decode(w, c, l, pr, 2, gamma=1, max_iters=3), 2, "hyb8 T=3")
    for split in (0, 1):                            # sparse loop / rotated layout (density heuristic forced)
        net.set_option("hyb8_split", split)
        assert net.decode_kernel(2) == ("decode_hyb8r_kernel" if split else "decode_hyb8_kernel")
        assert_same(gpu_decode(net, pr, 2, 1, 20), want, 2, f"hyb8 split2={split}")
    net.set_option("hyb8_split", 1)
    for nr in (6, 7, 8):                          # rows of the rotated kernel's first push step
        net.set_option("hyb8_rows", nr)
        assert_same(gpu_decode(net, pr, 2, 1, 20), want, 2, f"hyb8 rotated rows={nr}")
        assert_same(gpu_decode(net, pr, 2, 1, 2), oracle.decode(w, c, l, pr, 2, gamma=1, max_iters=2), 2,
                    f"hyb8 rotated rows={nr} T=2")
    net.close()


def test_or_bits_merge_equals_single(gb):
    """OR-ing the packed partial W's (gb_bits of each shard's
    sealed net, stacked) into an empty net with gb_or_bits gives the W of the
    whole message set (Eq.(1) is an OR of cliques); plus argument errors."""
    for c, l, m in ((8, 128, 20000), (5, 33, 3000), (16, 256, 100000)):
        msgs = gbgen.messages(15 + c, m, c, l)
        whole = make_net(gb, msgs, c, l)
        parts = [make_net(gb, msgs[i::3], c, l) for i in range(3)]
        stacked = torch.stack([p_.bits() for p_ in parts]).contiguous()
        fresh = gb.Net(c, l)
        fresh.or_bits(stacked)
        fresh.seal()
        assert torch.equal(fresh.weights_view(), whole.weights_view())
        assert torch.equal(fresh.bits(), whole.bits())
        # OR into a net that already holds a shard (accumulates)
        parts[0].or_bits(stacked[1:].contiguous())
        parts[0].seal()
        assert torch.equal(parts[0].weights_view(), whole.weights_view())
        for n in parts + [whole, fresh]:
            n.close()
    net = gb.Net(4, 16)
    with pytest.raises(gb.GBError) as ei:
        net.bits()
    assert ei.value.code == gb.GB_ESTATE
    assert gb.lib().gb_or_bits(net._h, None, 1, None) == gb.GB_EINVAL
    assert gb.lib().gb_or_bits(net._h, None, -1, None) == gb.GB_EINVAL
    assert gb.lib().gb_or_bits(net._h, None, 0, None) == gb.GB_OK
    host = np.zeros((net.n_padded, net.nw), np.uint32)
    assert gb.lib().gb_or_bits(net._h, host.ctypes.data, 1, None) == gb.GB_EINVAL
    net.close()


def test_sharded_store_max_merge_equals_single(gb):
    """W of a sharded store merged by MAX on uint8 (= OR on
    {0,1}) equals the single-device W byte for byte."""
    c, l, m = 8, 128, 20000
    msgs = gbgen.messages(5, m, c, l)
    whole = make_net(gb, msgs, c, l)
    parts = [make_net(gb, msgs[i::3], c, l) for i in range(3)]
    merged = torch.maximum(torch.maximum(parts[0].weights_view(), parts[1].weights_view()),
                           parts[2].weights_view())
    assert torch.equal(merged, whole.weights_view())
    w8 = parts[0].weights()
    w8.copy_(merged)
    parts[0].seal()
    pr, _ = gbgen.probes(6, msgs, 3000, 4, l)
    a = gpu_decode(parts[0], pr, 2, 1, 20)
    b = gpu_decode(whole, pr, 2, 1, 20)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_seal_and_state_errors(gb):
    c, l = 4, 16
    net = gb.Net(c, l)
    pr = to_dev(np.zeros((4, c), np.uint16))
    with pytest.raises(gb.GBError) as ei:
        net.decode(pr, 2)
    assert ei.value.code == gb.GB_ESTATE
    bad = np.array([[1, 2, 3, 4], [1, 2, 16, 4], [0xFFFF, 1, 1, 1]], np.uint16)
    net.store(to_dev(bad))
    with pytest.raises(gb.GBError) as ei:
        net.seal()
    assert ei.value.code == gb.GB_EINVAL and "2 stored message" in str(ei.value)
    w, _ = oracle.store(bad[:1], c, l)
    np.testing.assert_array_equal(net.weights().cpu().numpy(), padded_w(w, c, l))
    net.seal()  # count was reported once; sealed and usable
    net.decode(pr, 2)
    w8 = net.weights()
    w8[0, 40] = 1  # asymmetric edge
    with pytest.raises(gb.GBError) as ei:
        net.seal()
    assert "asymmetric" in str(ei.value)
    w8[40, 0] = 1
    net.seal()
    w8[0, 1] = 1
    w8[1, 0] = 1  # intra-cluster edge
    with pytest.raises(gb.GBError) as ei:
        net.seal()
    assert "intra-cluster" in str(ei.value)
    for g, r in ((0, 1), (0, 2), (-1, 0)):
        with pytest.raises(gb.GBError):
            net.decode(pr, r, gamma=g)
    with pytest.raises(gb.GBError):
        net.decode(pr, 0, max_iters=0)


# ---------------------------------------------------------------- decode
def run_case(gb, c, l, m, k, e, rules=RULES, gamma=2, T=20, seed=0, random_count=None):
    msgs = gbgen.messages(seed * 7 + 1, m, c, l)
    if random_count is None:
        random_count = k // 10
    if m == 0:
        random_count = k
    pr, _ = gbgen.probes(seed * 7 + 2, msgs, k, e, l, random_count=random_count)
    w, _ = oracle.store(msgs, c, l)
    net = make_net(gb, msgs, c, l)
    for rule in rules:
        g = gamma if (rule == 0 or gamma > 0) else 1
        got = gpu_decode(net, pr, rule, g, T)
        want = oracle.decode(w, c, l, pr, rule, gamma=g, max_iters=T)
        assert_same(got, want, rule, f"c={c} l={l} m={m} e={e}")
    return net, pr


def test_config1_full_parity(gb):
    """BASELINE config 1: c=4 l=16, M=50, 2 of 4 erased, 1000 probes, all rules."""
    run_case(gb, 4, 16, 50, 1000, 2)


@pytest.mark.parametrize("e", [0, 1, 3, 4])
def test_config1_all_erasure_counts(gb, e):
    run_case(gb, 4, 16, 50, 400, e, seed=e + 1)


@pytest.mark.parametrize("m", [5000, 20000, 30000])
def test_config2_shape_parity(gb, m):
    """BASELINE config 2 shape (c=8 l=128, e=4, M swept), sampled batch."""
    run_case(gb, 8, 128, m, 1500, 4, seed=m)


@pytest.mark.parametrize("c,l,m,e", [(3, 3, 4, 2), (5, 33, 200, 2), (7, 100, 3000, 3), (2, 1, 1, 1),
                                     (6, 64, 500, 6), (8, 128, 0, 4), (12, 40, 800, 5),
                                     (4, 256, 2000, 2), (8, 256, 3000, 4), (9, 70, 400, 4), (10, 64, 900, 5),
                                     (20, 16, 300, 10)])
def test_odd_shapes_and_degenerate(gb, c, l, m, e):
    """Ragged clusters (L not a multiple of 32, padding), L=1, M=0, e=C."""
    run_case(gb, c, l, m, 300, e, seed=c * 100 + l)


def test_scenario2_shape_parity(gb):
    """The paper's Scenario 2 shape (C=16, L=512, M=50k, e=7):
    n_padded = 8192, SOS state buffers in global scratch, W bits 8 MiB."""
    run_case(gb, 16, 512, 50000, 24, 7, seed=2, random_count=3)


def test_config4_shape_parity(gb):
    """BASELINE config 4 shape: c=16 l=256, M=100k, 8 erased (saturated)."""
    run_case(gb, 16, 256, 100000, 40, 8, seed=4, random_count=4)


def test_va_example_on_gpu(gb):
    """PAPER.md §V-A: SOS gamma=1 never converges (state alternates with T);
    gamma=2 converges in 3 rounds; SOM/hybrid give neurons 1..7."""
    msgs = np.array([[0, 0, 0], [1, 1, 0], [2, 1, 0], [0, 2, 0]], np.uint16)
    w, _ = oracle.store(msgs, 3, 3)
    net = make_net(gb, msgs, 3, 3)
    pr = np.array([[0xFFFF, 0xFFFF, 0]], np.uint16)
    for rule, g, T in ((0, 1, 19), (0, 1, 20), (0, 2, 20), (1, 1, 20), (2, 1, 20), (0, 1, 1)):
        assert_same(gpu_decode(net, pr, rule, g, T), oracle.decode(w, 3, 3, pr, rule, g, T), rule)


def test_invalid_probes_and_gamma_range(gb):
    c, l = 4, 16
    msgs = gbgen.messages(3, 50, c, l)
    w, _ = oracle.store(msgs, c, l)
    net = make_net(gb, msgs, c, l)
    pr, _ = gbgen.probes(4, msgs, 64, 2, l)
    pr[::5, 1] = 16
    pr[1::7, 0] = 0xFFFE
    for rule in RULES:
        for g in (1, 3, 200, 255, 256, 300):
            assert_same(gpu_decode(net, pr, rule, g, 20), oracle.decode(w, c, l, pr, rule, g, 20), rule)
    assert_same(gpu_decode(net, pr, 0, 0, 20), oracle.decode(w, c, l, pr, 0, 0, 20), 0)
    for T in (1, 2, 3):
        for rule in RULES:
            assert_same(gpu_decode(net, pr, rule, 2, T), oracle.decode(w, c, l, pr, rule, 2, T), rule)


def test_empty_batch_and_split_invariance(gb):
    """k = 0 is a no-op; results do not depend on the batch split (Eq.(11)
    columns are independent)."""
    c, l = 8, 128
    msgs = gbgen.messages(8, 10000, c, l)
    net = make_net(gb, msgs, c, l)
    pr, _ = gbgen.probes(9, msgs, 5000, 4, l, random_count=500)
    empty = to_dev(np.zeros((0, c), np.uint16))
    net.decode(empty, 2)
    for rule in RULES:
        whole = gpu_decode(net, pr, rule, 2, 20)
        parts = [gpu_decode(net, pr[a:b], rule, 2, 20) for a, b in ((0, 1), (1, 777), (777, 5000))]
        for i in range(3):
            np.testing.assert_array_equal(whole[i], np.concatenate([p[i] for p in parts]))


def test_host_buffers_match_device(gb):
    """gb_decode with host (pinned and pageable) buffers == device buffers."""
    c, l = 8, 128
    msgs = gbgen.messages(11, 20000, c, l)
    net = make_net(gb, msgs, c, l)
    pr, _ = gbgen.probes(12, msgs, 1 << 20 | 123, 4, l, random_count=1000)
    dev = gpu_decode(net, pr, 2, 1, 20)
    st, it, ss = net.decode(pr, 2, gamma=1, max_iters=20)   # numpy = pageable host
    for a, b in zip(dev, (st, it, ss)):
        np.testing.assert_array_equal(a, b)
    pt = torch.from_numpy(pr.view(np.int16)).pin_memory()
    out = net.alloc_outputs(pr.shape[0], device=False, pin=True)
    net.decode(pt, 2, gamma=1, max_iters=20, out=out)
    np.testing.assert_array_equal(dev[0], out[0].numpy().view(np.uint32))
    np.testing.assert_array_equal(dev[1], out[1].numpy().view(np.uint16))
    np.testing.assert_array_equal(dev[2], out[2].numpy())


def test_metric_config_full_size_sampled(gb):
    """BASELINE config 3 at full size (c=8 l=128, M=20k, e=4, K=10^7, hybrid)
    in the launch configuration bench.py times: 3000 sampled probes checked
    against the oracle one by one, plus properties over all K: status
    CONVERGED everywhere (Cor. 2, L674-681), known clusters one-hot, and
    every stored source message contained in its final state (Lemma 3)."""
    c, l, m, k = 8, 128, 20000, 10_000_000
    msgs = gbgen.messages(0x5EED, m, c, l)
    pr, src = gbgen.probes(0x5EED + 1, msgs, k, 4, l)
    net = make_net(gb, msgs, c, l)
    assert net.decode_kernel(2) == "decode_hyb8r_kernel"   # W dense: the rotated-layout kernel
    prd = to_dev(pr)
    st, it, ss = net.decode(prd, 2, gamma=2, max_iters=20)
    torch.cuda.synchronize()
    assert int((ss != 0).sum()) == 0
    # Lemma 3 over the whole batch: the source's one-hot bits are all set.
    msg_d = torch.from_numpy(msgs[src].astype(np.int64)).cuda()
    cols = torch.arange(c, device="cuda") * 4 + (msg_d >> 5)
    words = torch.gather(st, 1, cols)
    bit = torch.bitwise_left_shift(torch.ones_like(msg_d, dtype=torch.int64), msg_d & 31)
    assert bool(((words.to(torch.int64) & 0xFFFFFFFF) & bit).ne(0).all())
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(k, 3000, replace=False))
    w, _ = oracle.store(msgs, c, l)
    want = oracle.decode(w, c, l, pr[idx], 2, gamma=2, max_iters=20)
    got = (st[idx].cpu().numpy().view(np.uint32), it[idx].cpu().numpy().view(np.uint16),
           ss[idx].cpu().numpy())
    assert_same(got, want, 2, "config3 sampled")


def test_determinism(gb):
    c, l = 8, 128
    msgs = gbgen.messages(21, 15000, c, l)
    net = make_net(gb, msgs, c, l)
    pr, _ = gbgen.probes(22, msgs, 20000, 4, l)
    for rule in RULES:
        a = gpu_decode(net, pr, rule, 2, 20)
        b = gpu_decode(net, pr, rule, 2, 20)
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("c,l,rule,want", [(8, 128, 0, "sos_tc2_kernel"), (16, 256, 0, "sos_tc3_kernel"),
                                           (4, 16, 0, "sos_tc2_kernel"), (3, 3, 0, "sos_tc2_kernel"),
                                           (8, 256, 0, "sos_tc3_kernel"), (4, 256, 0, "sos_tc2_kernel"),
                                           (8, 128, 2, "decode_hyb8_kernel"), (8, 128, 1, "decode_smem_kernel"),
                                           (4, 16, 2, "decode_smem_kernel"),
                                           (16, 256, 1, "decode_l2t_kernel"), (16, 256, 2, "decode_l2t_kernel"),
                                           (12, 40, 2, "decode_l2_kernel"), (9, 100, 1, "decode_l2t_kernel"),
                                           (9, 70, 1, "decode_generic_kernel"), (16, 512, 0, "sos_tc3x2_kernel"),
                                           (16, 512, 2, "decode_l2t_kernel"), (16, 512, 1, "decode_l2t_kernel"),
                                           (4, 600, 0, "decode_generic_kernel")])
def test_kernel_selection(gb, c, l, rule, want):
    """The product path runs the intended sm_100a kernel for each shape/rule
    (tensor-core SOS, shared-memory bit kernel, generic warp kernel).  SOS at
    n_padded <= 4096 runs on a CTA pair (sos_tc2x2 / sos_tc3x2) unless
    GB_OPT_SOS_PAIR = 0."""
    net = gb.Net(c, l)
    if rule == 0 and c <= 8 and c * 32 * ((l + 31) // 32) <= 1024 and (l + 31) // 32 in (1, 2, 4):
        # an empty (sealed) W has density 0: sum-of-sum on the CUDA cores unless sos_bits = 0
        net.seal()
        assert net.decode_kernel(rule) == "sos_bits_kernel"
        net.set_option("sos_bits", 0)
    if want in ("sos_tc2_kernel", "sos_tc3_kernel"):
        assert net.decode_kernel(rule) == want.replace("_kernel", "x2_kernel")
        net.set_option("sos_pair", 0)
    assert net.decode_kernel(rule) == want
    if want == "sos_tc3x2_kernel":   # Lp = 512 / n_p > 4096: streamed A on the CTA pair only
        net.set_option("sos_pair", 0)
        assert net.decode_kernel(0) == "sos_tc_kernel"


@pytest.mark.parametrize("rule", RULES)
def test_config2_full_size_sampled(gb, rule):
    """BASELINE config 2 at full size (c=8 l=128, e=4, K=10^5) for every rule and the
    M sweep end points, in the launch configuration bench.py times: 400 sampled
    probes checked one by one against the oracle; whole-batch properties
    (no GB_INVALID; SOM/hybrid always converge, Thm 3 / Cor. 2)."""
    c, l, k = 8, 128, 100_000
    rng = np.random.default_rng(rule)
    for m in (5000, 30000):
        msgs = gbgen.messages(0x5EED + m, m, c, l)
        pr, _ = gbgen.probes(0x5EED + m + 1, msgs, k, 4, l)
        net = make_net(gb, msgs, c, l)
        st, it, ss = gpu_decode(net, pr, rule, 2, 20)
        assert (ss != 2).all()
        if rule != 0:
            assert (ss == 0).all()
        idx = np.sort(rng.choice(k, 400, replace=False))
        w, _ = oracle.store(msgs, c, l)
        assert_same((st[idx], it[idx], ss[idx]), oracle.decode(w, c, l, pr[idx], rule, 2, 20), rule,
                    f"config2 M={m} sampled")


def test_config2_sos_full_batch_both_paths(gb):
    """The bench's C2 sum-of-sum line at its size (c=8 l=128 M=5k e=4, K=10^6, gamma 2): the
    CUDA-core kernel for sparse states (the default at this density) and the tensor-core
    pair kernel give identical states, rounds and status for every probe of the batch, and
    300 sampled probes equal the oracle."""
    c, l, m, k = 8, 128, 5000, 1_000_000
    msgs = gbgen.messages(0x5EED + m, m, c, l)
    pr, _ = gbgen.probes(0x5EED + m + 1, msgs, k, 4, l)
    net = make_net(gb, msgs, c, l)
    assert net.decode_kernel(0) == "sos_bits_kernel"
    prd = to_dev(pr)
    a = net.decode(prd, 0, gamma=2, max_iters=20)
    net.set_option("sos_bits", 0)
    assert net.decode_kernel(0) == "sos_tc2x2_kernel"
    b = net.decode(prd, 0, gamma=2, max_iters=20)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert torch.equal(x, y)
    idx = np.sort(np.random.default_rng(5).choice(k, 300, replace=False))
    w, _ = oracle.store(msgs, c, l)
    got = (a[0][idx].cpu().numpy().view(np.uint32), a[1][idx].cpu().numpy().view(np.uint16), a[2][idx].cpu().numpy())
    assert_same(got, oracle.decode(w, c, l, pr[idx], 0, 2, 20), 0, "config2 SOS sampled")
    net.close()


def test_config4_full_size_sampled(gb):
    """BASELINE config 4 (c=16 l=256, M=10^5, e=8) at the bench's size (K=10^6, the launch
    configuration bench.py times: sos_tc3x2_kernel / decode_l2t_kernel) for SOS and SOM:
    48 sampled probes per rule vs the oracle (the batch's first and last probes among them),
    and over all K the properties that hold at any size -- no invalid status, rounds in
    [1, 20]; SOS: every cluster keeps at least one neuron (the max is always attained,
    Eq.(5)); SOM: every stored source message is contained in its final state (Lemma 3)."""
    c, l, m, k = 16, 256, 100_000, 1_000_000
    msgs = gbgen.messages(0x5EED, m, c, l)
    pr, src = gbgen.probes(0x5EED + 1, msgs, k, 8, l)
    net = make_net(gb, msgs, c, l)
    w, _ = oracle.store(msgs, c, l)
    rng = np.random.default_rng(44)
    idx = np.unique(np.concatenate([[0, 1, k - 2, k - 1], rng.choice(k, 44, replace=False)]))
    wc = 8
    msg_d = torch.from_numpy(msgs[src].astype(np.int64)).cuda()
    cols = torch.arange(c, device="cuda") * wc + (msg_d >> 5)
    bit = torch.bitwise_left_shift(torch.ones_like(msg_d), msg_d & 31)
    for rule in (0, 1):
        assert net.decode_kernel(rule) == ("sos_tc3x2_kernel" if rule == 0 else "decode_l2t_kernel")
        st, it, ss = net.decode(to_dev(pr), rule, gamma=2, max_iters=20)
        torch.cuda.synchronize()
        assert int((ss == 2).sum()) == 0
        its = it.to(torch.int32) & 0xFFFF
        assert int(its.min()) >= 1 and int(its.max()) <= 20
        if rule == 0:
            blocks = (st.view(k, c, wc).to(torch.int64) & 0xFFFFFFFF).ne(0).any(dim=2)
            assert bool(blocks.all())
        else:
            words = torch.gather(st, 1, cols).to(torch.int64) & 0xFFFFFFFF
            assert bool((words & bit).ne(0).all())
        got = (st[idx].cpu().numpy().view(np.uint32), it[idx].cpu().numpy().view(np.uint16), ss[idx].cpu().numpy())
        assert_same(got, oracle.decode(w, c, l, pr[idx], rule, 2, 20), rule, "config4 sampled")


def test_config4_hybrid_full_size_sampled(gb):
    """BASELINE config 4 hybrid at the bench's size (c=16 l=256, M=10^5, e=8,
    K=10^6, decode_l2t_kernel): 24 sampled probes vs the oracle, plus over all K:
    no invalid status, known clusters one-hot, every stored source message
    contained in its final state (Lemma 3)."""
    c, l, m, k = 16, 256, 100_000, 1_000_000
    msgs = gbgen.messages(0x5EED, m, c, l)
    pr, src = gbgen.probes(0x5EED + 1, msgs, k, 8, l)
    net = make_net(gb, msgs, c, l)
    assert net.decode_kernel(2) == "decode_l2t_kernel"
    st, it, ss = net.decode(to_dev(pr), 2, gamma=2, max_iters=20)
    torch.cuda.synchronize()
    assert int((ss == 2).sum()) == 0
    wc = 8
    msg_d = torch.from_numpy(msgs[src].astype(np.int64)).cuda()
    cols = torch.arange(c, device="cuda") * wc + (msg_d >> 5)
    words = torch.gather(st, 1, cols).to(torch.int64) & 0xFFFFFFFF
    bit = torch.bitwise_left_shift(torch.ones_like(msg_d), msg_d & 31)
    assert bool((words & bit).ne(0).all())
    known = torch.from_numpy(pr.astype(np.int64)).cuda() != 0xFFFF
    only = words.eq(bit) | ~known          # a known cluster's word holds exactly the probe's bit
    assert bool(only.all())
    rng = np.random.default_rng(4)
    idx = np.sort(rng.choice(k, 24, replace=False))
    w, _ = oracle.store(msgs, c, l)
    want = oracle.decode(w, c, l, pr[idx], 2, gamma=2, max_iters=20)
    got = (st[idx].cpu().numpy().view(np.uint32), it[idx].cpu().numpy().view(np.uint16), ss[idx].cpu().numpy())
    assert_same(got, want, 2, "config4 hybrid sampled")


def test_config5_full_size_store(gb):
    """BASELINE config 5 at full size: 10^7 messages at c=16 l=256 stored by the
    privatised kernel in one call, and as 4 shards merged by the packed OR
    (gb_bits + gb_or_bits, the N3 merge) -- both equal the oracle's W (Eq.(1))
    byte for byte."""
    c, l, m = 16, 256, 10_000_000
    msgs = gbgen.messages(0x5EED, m, c, l)
    w, bad = oracle.store(msgs, c, l)
    assert bad == 0
    want = padded_w(w, c, l)
    net = make_net(gb, msgs, c, l)
    np.testing.assert_array_equal(net.weights().cpu().numpy(), want)
    parts = [make_net(gb, msgs[i::4], c, l) for i in range(4)]
    merged = gb.Net(c, l)
    merged.or_bits(torch.stack([p_.bits() for p_ in parts]).contiguous())
    merged.seal()
    np.testing.assert_array_equal(merged.weights().cpu().numpy(), want)
    for n in parts + [merged, net]:
        n.close()


def test_mixed_erasures_narrow_and_wide_slots(gb):
    """Hybrid probes with e <= 4 run on the 4-slot instance, the rest are queued to the
    8-slot instance (list mode) inside the same gb_decode; per-probe e from 0 to C in
    one batch must match the oracle for every probe (and SOM, which is all-wide)."""
    c, l, m, k = 8, 128, 10000, 3000
    msgs = gbgen.messages(31, m, c, l)
    e = np.random.default_rng(5).integers(0, c + 1, size=k)
    pr, _ = gbgen.probes(32, msgs, k, e, l, random_count=300)
    w, _ = oracle.store(msgs, c, l)
    net = make_net(gb, msgs, c, l)
    for rule in (1, 2):
        assert_same(gpu_decode(net, pr, rule, 2, 20), oracle.decode(w, c, l, pr, rule, 2, 20), rule, "mixed e")


@pytest.mark.parametrize("c,l,m,e,gamma", [(8, 128, 8000, 4, 2), (4, 16, 60, 2, 1), (3, 3, 5, 1, 0),
                                           (5, 33, 300, 2, 300), (4, 256, 3000, 2, 2), (6, 64, 2000, 3, 255),
                                           (7, 100, 1500, 3, 1), (8, 96, 3000, 5, 4), (2, 1, 1, 1, 1),
                                           (8, 128, 8000, 4, 31743), (8, 128, 8000, 4, 31744),
                                           (4, 64, 500, 2, 40000)])
def test_sos_pair_vs_single_cta(gb, c, l, m, e, gamma):
    """The CTA-pair SOS kernel (tcgen05 cta_group::2, M = 256, each CTA stages half
    of W's rows) and the single-CTA kernel give identical results, and both equal
    the oracle: the pair only re-tiles the exact int32 contraction of Eq.(10)-(11).
    gamma 31743 / 31744 at n_p = 1024 straddle the packed 16-bit epilogue's bound
    (gamma + n_p < 0x7FFF); 40000 takes the 32-bit epilogue."""
    msgs = gbgen.messages(500 + c + l, m, c, l)
    net = make_net(gb, msgs, c, l)
    pr, _ = gbgen.probes(501 + c, msgs, 1537, e, l, random_count=5)
    net.set_option("sos_bits", 0)   # the tensor-core kernels
    res = {}
    for flag in ("1", "0"):
        net.set_option("sos_pair", int(flag))
        res[flag] = gpu_decode(net, pr, 0, gamma, 20)
        assert net.decode_kernel(0) == ("sos_tc2x2_kernel" if flag == "1" else "sos_tc2_kernel")
    for x, y in zip(res["1"], res["0"]):
        np.testing.assert_array_equal(x, y)
    w8, _ = oracle.store(msgs, c, l)
    assert_same(res["1"], oracle.decode(w8, c, l, pr, oracle.SOS, gamma=gamma, max_iters=20), 0, "pair")


@pytest.mark.parametrize("c,l,m,e,gamma,k", [(16, 256, 100000, 8, 2, 300), (32, 64, 3000, 16, 1, 700),
                                             (9, 256, 20000, 4, 0, 257), (5, 250, 4000, 2, 300, 129),
                                             (16, 256, 30000, 8, 255, 200)])
def test_sos_streamed_a_vs_oracle(gb, c, l, m, e, gamma, k):
    """The streamed-A SOS kernel (1024 < n_p <= 4096: A producer warps expand the
    state into a ring of swizzled stages, TMA ring of W8 + gamma*I) equals the
    oracle and the 4-warp sos_tc_kernel (GB_OPT_SOS_STREAMED = 0) bit for bit: ragged tiles,
    gamma = 0, gamma folded into B (<= 255) and added in the epilogue (300)."""
    msgs = gbgen.messages(600 + c + l, m, c, l)
    net = make_net(gb, msgs, c, l)
    pr, _ = gbgen.probes(601 + c, msgs, k, e, l, random_count=k // 10)
    pr[3, 0] = l                       # invalid symbol
    w8, _ = oracle.store(msgs, c, l)
    want = oracle.decode(w8, c, l, pr, oracle.SOS, gamma=gamma, max_iters=20)
    for flag, name in (("1", "sos_tc3x2_kernel"), ("0", "sos_tc3_kernel")):   # CTA pair / single CTA
        net.set_option("sos_pair", int(flag))
        assert net.decode_kernel(0) == name
        got = gpu_decode(net, pr, 0, gamma, 20)
        assert_same(got, want, 0, name)
        assert_same(gpu_decode(net, pr, 0, gamma, 3),
                    oracle.decode(w8, c, l, pr, oracle.SOS, gamma=gamma, max_iters=3), 0, name + " T=3")
    net.set_option("sos_streamed", 0)
    assert net.decode_kernel(0) == "sos_tc_kernel"
    other = gpu_decode(net, pr, 0, gamma, 20)
    for x, y in zip(got, other):
        np.testing.assert_array_equal(x, y)
    net.close()


@pytest.mark.parametrize("c,l,m,e,gamma,k", [(16, 512, 50000, 7, 2, 600), (10, 500, 20000, 5, 0, 300),
                                             (3, 512, 200, 1, 300, 129), (16, 512, 5000, 12, 255, 257)])
def test_sos_streamed_a_wide_clusters(gb, c, l, m, e, gamma, k):
    """Scenario 2's shape (Lp = 512, n_p up to 8192) on the streamed-A CTA-pair kernel: one
    512-column accumulator per pass (two N = 256 MMAs), the current state in the global
    scratch.  Bit-exact vs the oracle and the 4-warp sos_tc_kernel (GB_OPT_SOS_PAIR = 0):
    ragged L (500), gamma 0 / folded (2, 255) / in the epilogue (300), T = 3, invalid and
    random probes."""
    msgs = gbgen.messages(900 + c + l, m, c, l)
    net = make_net(gb, msgs, c, l)
    pr, _ = gbgen.probes(901 + c, msgs, k, e, l, random_count=k // 10)
    pr[2, 0] = l                       # invalid symbol
    w8, _ = oracle.store(msgs, c, l)
    if c * 512 > 1024:
        assert net.decode_kernel(0) == "sos_tc3x2_kernel"
    want = oracle.decode(w8, c, l, pr, oracle.SOS, gamma=gamma, max_iters=20)
    got = gpu_decode(net, pr, 0, gamma, 20)
    assert_same(got, want, 0, "wide pair")
    assert_same(gpu_decode(net, pr, 0, gamma, 3), oracle.decode(w8, c, l, pr, oracle.SOS, gamma=gamma, max_iters=3),
                0, "wide pair T=3")
    net.set_option("sos_pair", 0)
    other = gpu_decode(net, pr, 0, gamma, 20)
    for x, y in zip(got, other):
        np.testing.assert_array_equal(x, y)
    net.close()


@pytest.mark.parametrize("c,l,m,e,k", [(16, 256, 100000, 8, 300), (16, 256, 20000, 11, 200), (12, 100, 3000, 5, 257),
                                       (16, 512, 50000, 7, 100), (9, 128, 8000, 3, 129), (16, 200, 0, 6, 64)])
@pytest.mark.parametrize("rule", [1, 2])
def test_l2t_matches_oracle_and_warp_kernel(gb, c, l, m, e, k, rule):
    """The thread-per-probe L2 kernel (staged push from L2-resident bit rows) against
    the oracle and against the warp-per-probe decode_l2_kernel (GB_OPT_L2T = 0): mixed
    erasure counts (probes with more erased clusters than its 8 hybrid slots are
    queued to the warp kernel), ragged L, M=0, invalid probes, random probes.
    """
    msgs = gbgen.messages(700 + c + l + m, max(m, 1), c, l)[:m]
    src = msgs if m else gbgen.messages(5, 10, c, l)
    pr, _ = gbgen.probes(701 + k, src, k, e, l, random_count=k // 5)
    rng = np.random.default_rng(k + c)
    for i in range(0, k, 4):
        row = pr[i].copy()
        row[row == 0xFFFF] = rng.integers(0, l)
        row[rng.choice(c, int(rng.integers(0, c + 1)), replace=False)] = 0xFFFF
        pr[i] = row
    pr[1, 0] = l
    w, _ = oracle.store(msgs, c, l) if m else (np.zeros((c * l, c * l), np.uint8), None)
    net = make_net(gb, msgs, c, l)
    want = oracle.decode(w, c, l, pr, rule, gamma=1, max_iters=20)
    assert_same(gpu_decode(net, pr, rule, 1, 20), want, rule, f"l2t c={c} l={l}")
    assert_same(gpu_decode(net, pr, rule, 1, 2), oracle.decode(w, c, l, pr, rule, gamma=1, max_iters=2), rule, "T=2")
    net.set_option("l2t", 0)
    assert_same(gpu_decode(net, pr, rule, 1, 20), want, rule, "warp kernel")
    net.close()


@pytest.mark.parametrize("c,l,m,e,k,gamma,opts,kernel", [
    (3, 3, 4, 2, 1, 1, {}, "sos_tc2x2_kernel"),                        # §V-A: v^3 == v^1
    (5, 6, 25, 3, 300, 0, {}, "sos_tc2x2_kernel"),
    (5, 6, 25, 3, 300, 0, {"sos_pair": 0}, "sos_tc2_kernel"),
    (8, 128, 30000, 5, 1000, 1, {}, "sos_tc2x2_kernel"),
    (8, 128, 20000, 4, 1000, 2, {"sos_pair": 0}, "sos_tc2_kernel"),
    (16, 256, 100000, 10, 300, 0, {}, "sos_tc3x2_kernel"),
    (16, 256, 100000, 10, 300, 0, {"sos_pair": 0}, "sos_tc3_kernel"),
    (16, 256, 100000, 10, 300, 0, {"sos_streamed": 0}, "sos_tc_kernel"),
    (8, 512, 30000, 5, 200, 0, {}, "sos_tc3x2_kernel"),
    (8, 512, 30000, 5, 200, 0, {"sos_pair": 0}, "sos_tc_kernel"),
    (4, 600, 3000, 2, 100, 0, {}, "decode_generic_kernel"),
])
def test_sos_cycle_exit_flag(gb, c, l, m, e, k, gamma, opts, kernel):
    """GB_FLAG_CYCLE_EXIT: every sum-of-sum kernel stops a probe at
    the first round r >= 2 with V^r == V^{r-2} != V^{r-1}, status GB_CYCLE, state
    V^r -- bit-exact vs the oracle with the same flag; without the flag nothing
    changes; the flag leaves sum-of-max / hybrid untouched."""
    if m == 4:
        msgs = np.array([[0, 0, 0], [1, 1, 0], [2, 1, 0], [0, 2, 0]], np.uint16)
        pr = np.array([[0xFFFF, 0xFFFF, 0]], np.uint16)
    else:
        msgs = gbgen.messages(800 + c + l, m, c, l)
        pr, _ = gbgen.probes(801 + c, msgs, k, e, l, random_count=k // 3)
    w, _ = oracle.store(msgs, c, l)
    net = make_net(gb, msgs, c, l)
    net.set_option("sos_bits", 0)   # reported name of the no-flag path; the flag never takes it
    for kk, v in opts.items():
        net.set_option(kk, v)
    assert net.decode_kernel(0) == kernel
    for T in (20, 7):
        want = oracle.decode(w, c, l, pr, 0, gamma=gamma, max_iters=T, flags=oracle.CYCLE_EXIT)
        st, it, ss = net.decode(to_dev(pr), 0, gamma=gamma, max_iters=T, flags=gb.FLAG_CYCLE_EXIT)
        torch.cuda.synchronize()
        got = (st.cpu().numpy().view(np.uint32), it.cpu().numpy().view(np.uint16), ss.cpu().numpy())
        assert_same(got, want, 0, f"cycle-exit {kernel} T={T}")
        if m == 4:
            assert want[2][0] == gb.CYCLE and want[1][0] == 3
    assert (want[2] == gb.CYCLE).any()
    assert_same(gpu_decode(net, pr, 0, gamma, 20), oracle.decode(w, c, l, pr, 0, gamma=gamma, max_iters=20), 0)
    for rule in (1, 2):
        st, it, ss = net.decode(to_dev(pr), rule, gamma=1, max_iters=20, flags=gb.FLAG_CYCLE_EXIT)
        torch.cuda.synchronize()
        got = (st.cpu().numpy().view(np.uint32), it.cpu().numpy().view(np.uint16), ss.cpu().numpy())
        assert_same(got, oracle.decode(w, c, l, pr, rule, gamma=1, max_iters=20), rule, "flag on SOM/hybrid")
    with pytest.raises(gb.GBError):
        net.decode(to_dev(pr), 0, gamma=gamma, max_iters=20, flags=2)
    net.close()


@pytest.mark.parametrize("c,l,m,e,k", [(8, 128, 5000, 4, 1000), (8, 128, 20000, 4, 700), (4, 16, 50, 2, 1000),
                                       (3, 3, 4, 2, 1), (5, 60, 2000, 3, 300), (16, 64, 3000, 9, 257),
                                       (7, 100, 0, 3, 64)])
def test_som_tensor_core_matches_oracle(gb, c, l, m, e, k):
    """N2: sum-of-max as C exact per-source-cluster int8 contractions on the tensor
    cores (hit = count > 0, Eq.(6)-(7)) equals the oracle and the bit kernel bit for
    bit: states, rounds, statuses; ragged L, C=16, M=0, the §V-A example, T=2."""
    if m == 4:
        msgs = np.array([[0, 0, 0], [1, 1, 0], [2, 1, 0], [0, 2, 0]], np.uint16)
        pr = np.array([[0xFFFF, 0xFFFF, 0]], np.uint16)
    else:
        msgs = gbgen.messages(900 + c + l, max(m, 1), c, l)[:m]
        pr, _ = gbgen.probes(901 + c, msgs if m else gbgen.messages(4, 10, c, l), k, e, l, random_count=k // 5)
        pr[2, 0] = l
    w, _ = oracle.store(msgs, c, l) if m else (np.zeros((c * l, c * l), np.uint8), None)
    net = make_net(gb, msgs, c, l)
    net.set_option("som_tensor", 1)
    assert net.decode_kernel(1) == "som_tc_kernel"
    for T in (20, 2):
        want = oracle.decode(w, c, l, pr, 1, gamma=1, max_iters=T)
        assert_same(gpu_decode(net, pr, 1, 1, T), want, 1, f"som_tc T={T}")
    net.set_option("som_tensor", 0)
    assert net.decode_kernel(1) != "som_tc_kernel"
    assert_same(gpu_decode(net, pr, 1, 3, 20), oracle.decode(w, c, l, pr, 1, gamma=3, max_iters=20), 1, "bit")
    net.close()


@pytest.mark.parametrize("c,l,m,e,gamma,k", [(8, 128, 5000, 4, 2, 3001), (8, 128, 5000, 4, 0, 700),
                                             (8, 128, 2000, 5, 5, 513), (4, 16, 50, 2, 1, 1000),
                                             (8, 64, 1500, 3, 1, 600), (7, 100, 3000, 3, 2, 777),
                                             (3, 3, 4, 2, 1, 64), (8, 33, 300, 4, 3, 300),
                                             (8, 128, 30000, 4, 2, 300), (8, 128, 5000, 4, 40, 300)])
def test_sos_bits_matches_oracle(gb, c, l, m, e, gamma, k):
    """Sum-of-sum on the CUDA cores (sos_bits_kernel: the active neurons' rows added into
    bit-sliced counters, winner-take-all plane by plane) against the oracle and the tensor-
    core kernels, bit for bit: word counts 1 / 2 / 4, ragged L, gamma 0..5, T = 1 / 3 / 20,
    invalid and random (non-stored) probes; random probes and dense W (M = 30000) push
    probes past the 32-entry list / 6 counter planes (gamma = 40 puts every probe on the
    6-plane counters and those with 24+ active neurons past them), so the overflow list is
    exercised too
    (decoded from the start by the CTA-pair tensor kernel in list mode, or by
    decode_generic_kernel when the pair kernel is off)."""
    msgs = gbgen.messages(1300 + c + l, m, c, l)
    pr, _ = gbgen.probes(1301 + c, msgs, k, e, l, random_count=k // 4)
    pr[1, 0] = l                       # invalid symbol
    w, _ = oracle.store(msgs, c, l)
    net = make_net(gb, msgs, c, l)
    net.set_option("sos_bits", 1)
    assert net.decode_kernel(0) == "sos_bits_kernel"
    for T in (20, 3, 1):
        want = oracle.decode(w, c, l, pr, 0, gamma=gamma, max_iters=T)
        got = gpu_decode(net, pr, 0, gamma, T)
        assert_same(got, want, 0, f"sos_bits c={c} l={l} m={m} T={T}")
    net.set_option("sos_pair", 0)                  # overflow list -> generic kernel
    assert_same(gpu_decode(net, pr, 0, gamma, T), want, 0, "sos_bits, overflow to the generic kernel")
    net.set_option("sos_pair", 1)
    net.set_option("sos_bits", 0)
    other = gpu_decode(net, pr, 0, gamma, 1)
    for x, y in zip(got, other):
        np.testing.assert_array_equal(x, y)
    # the period-2 exit keeps the tensor-core kernels (same results as the oracle's flag)
    net.set_option("sos_bits", 1)
    st, it, ss = net.decode(to_dev(pr), 0, gamma=gamma, max_iters=20, flags=gb.FLAG_CYCLE_EXIT)
    torch.cuda.synchronize()
    assert_same((st.cpu().numpy().view(np.uint32), it.cpu().numpy().view(np.uint16), ss.cpu().numpy()),
                oracle.decode(w, c, l, pr, 0, gamma=gamma, max_iters=20, flags=oracle.CYCLE_EXIT), 0, "cycle exit")
    net.close()


@pytest.mark.parametrize("seed", range(24))
def test_random_shapes_fuzz(gb, seed):
    """Seeded sweep over random shapes (C 2..16, L 1..300 incl. ragged and
    non-power-of-two word counts), stored-message counts, erasure counts,
    rules, gamma and max_iters: every kernel the selection can reach (pair /
    streamed-A / 4-warp / generic SOS, hyb8 / smem / l2t / l2 / generic bit
    kernels, both store kernels) against the oracle, bit for bit."""
    rng = np.random.default_rng(1000 + seed)
    for case in range(8):
        c = int(rng.integers(2, 17))
        l = int(rng.choice([1, 3, 16, 31, 33, 64, 70, 100, 128, 129, 200, 256, 300]))
        if c * 32 * ((l + 31) // 32) > 8192 or c * l > 3000:
            l = 64
        m = int(rng.choice([0, 5, 50, 500, 3000]))
        k = int(rng.integers(1, 300))
        e = int(rng.integers(0, c + 1))
        rule = int(rng.integers(0, 3))
        gamma = int(rng.choice([0, 1, 2, 5])) if rule == 0 else int(rng.choice([1, 2, 7]))
        T = int(rng.choice([1, 2, 5, 20]))
        msgs = gbgen.messages(seed * 100 + case, max(m, 1), c, l)[:m]
        src = msgs if m else gbgen.messages(3, 5, c, l)
        pr, _ = gbgen.probes(seed * 100 + case + 1, src, k, e, l, random_count=k // 4)
        w, _ = oracle.store(msgs, c, l) if m else (np.zeros((c * l, c * l), np.uint8), None)
        net = make_net(gb, msgs, c, l)
        tag = f"fuzz c={c} l={l} m={m} k={k} e={e} rule={rule} g={gamma} T={T} kernel={net.decode_kernel(rule)}"
        want = oracle.decode(w, c, l, pr, rule, gamma, T)
        assert_same(gpu_decode(net, pr, rule, gamma, T), want, rule, tag)
        if rule == 0:   # sum-of-sum on the CUDA cores and on the tensor cores, both forced
            for ob in (1, 0):
                net.set_option("sos_bits", ob)
                assert_same(gpu_decode(net, pr, rule, gamma, T), want, rule, tag + f" sos_bits={ob}")
        net.close()


@pytest.mark.parametrize("seed", range(12))
def test_random_shapes_mixed_erasures_fuzz(gb, seed):
    """Like the shape fuzz, but every probe has its own erasure count (wide-slot
    and list-mode paths), some symbols are invalid, and SOS runs with the
    period-2 cycle exit half of the time."""
    rng = np.random.default_rng(5000 + seed)
    for case in range(6):
        c = int(rng.integers(2, 17))
        l = int(rng.choice([2, 16, 32, 50, 96, 128, 130, 256]))
        if c * 32 * ((l + 31) // 32) > 4096:
            l = 32
        m = int(rng.choice([5, 100, 2000]))
        k = int(rng.integers(1, 400))
        rule = int(rng.integers(0, 3))
        gamma = int(rng.choice([0, 1, 2])) if rule == 0 else 1
        flags = int(rule == 0 and rng.random() < 0.5)
        T = int(rng.choice([2, 7, 20]))
        msgs = gbgen.messages(seed * 50 + case, m, c, l)
        pr, _ = gbgen.probes(seed * 50 + case + 1, msgs, k, 1, l, random_count=k // 3)
        for i in range(k):
            row = pr[i].copy()
            row[row == 0xFFFF] = rng.integers(0, l)
            row[rng.choice(c, int(rng.integers(0, c + 1)), replace=False)] = 0xFFFF
            if rng.random() < 0.02:
                row[int(rng.integers(0, c))] = l + int(rng.integers(0, 5))
            pr[i] = row
        w, _ = oracle.store(msgs, c, l)
        net = make_net(gb, msgs, c, l)
        st, it, ss = net.decode(to_dev(pr), rule, gamma=gamma, max_iters=T, flags=flags)
        torch.cuda.synchronize()
        got = (st.cpu().numpy().view(np.uint32), it.cpu().numpy().view(np.uint16), ss.cpu().numpy())
        want = oracle.decode(w, c, l, pr, rule, gamma, T, flags=flags)
        assert_same(got, want, rule, f"mixed fuzz c={c} l={l} m={m} k={k} rule={rule} g={gamma} T={T} f={flags} "
                                     f"kernel={net.decode_kernel(rule)}")
        net.close()
