"""GPU checks of the C-ABI contract (include/gb.h) beyond single-call parity.

* Concurrency (SURVEY.md §8.b "Concurrent decodes on one handle are safe with
  distinct output buffers"): host threads on their own
  streams decode on ONE handle with different rules and gammas at once; every
  result equals the oracle.
* Host-buffer decodes larger than one staging chunk (2^19 probes) run their
  chunks on two streams: every kernel family (SOS pair, SOM shared-memory,
  hybrid list mode, L2 thread-per-probe) equals the device-pointer decode.
* gb_seal is asynchronous; gb_seal_status reports its outcome; a decode issued
  after a failed seal's outcome is known is refused; gb_weights unseals.
* gb_store falls back to scattered writes when a cluster-pair block does not
  fit the privatised tile (Lp > 1024), and the privatised path at Lp = 512.
"""
import threading

import numpy as np
import pytest

import gbgen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


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


def as_np(out):
    st, it, ss = out
    if isinstance(st, np.ndarray):
        return st.view(np.uint32), it.view(np.uint16), ss
    return st.cpu().numpy().view(np.uint32), it.cpu().numpy().view(np.uint16), ss.cpu().numpy()


def same(a, b, tag):
    for x, y, name in zip(a, b, ("state", "iters", "status")):
        bad = np.flatnonzero((x != y).reshape(x.shape[0], -1).any(axis=1))
        assert bad.size == 0, f"{tag}: {name} differs on {bad.size} probes, first {bad[:5]}"


def test_concurrent_decodes_one_handle(gb):
    """Four host threads, each with its own CUDA stream, decode on one sealed
    handle at the same time: hybrid (C=8 kernel + list mode for e > 4), SOM,
    SOS with gamma 2 and SOS with gamma 5 (two W8 + gamma*I operands built
    concurrently), repeatedly, into distinct outputs.  Every result equals
    the oracle."""
    c, l, m, k = 8, 128, 8000, 4000
    msgs = gbgen.messages(41, m, c, l)
    e = np.random.default_rng(2).integers(1, c + 1, size=k)
    pr, _ = gbgen.probes(42, msgs, k, e, l, random_count=400)
    w, _ = oracle.store(msgs, c, l)
    net = gb.Net(c, l)
    net.store(to_dev(msgs))
    net.seal()
    jobs = [(2, 1), (1, 1), (0, 2), (0, 5)]
    want = {j: oracle.decode(w, c, l, pr, j[0], gamma=j[1], max_iters=20) for j in jobs}
    prd = to_dev(pr)
    errors, results = [], {}
    start = threading.Barrier(len(jobs))

    def worker(job):
        try:
            s = torch.cuda.Stream()
            outs = []
            with torch.cuda.stream(s):
                start.wait()
                for _ in range(6):
                    outs.append(net.decode(prd, job[0], gamma=job[1], max_iters=20, stream=s))
            s.synchronize()
            results[job] = [as_np(o) for o in outs]
        except Exception as ex:   # surfaced below
            errors.append(ex)

    th = [threading.Thread(target=worker, args=(j,)) for j in jobs]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for j in jobs:
        for r, got in enumerate(results[j]):
            same(got, want[j], f"rule {j[0]} gamma {j[1]} repetition {r}")
    net.close()


@pytest.mark.parametrize("c,l,m,rule,e", [(8, 128, 5000, 0, 4), (8, 128, 5000, 1, 4), (8, 128, 20000, 2, -1),
                                          (16, 256, 20000, 2, 8)])
def test_host_buffers_multichunk_all_kernels(gb, c, l, m, rule, e):
    """Host (pinned) buffers with k = 4 * 2^19 + 4321: the library pipelines 5
    chunks of 2^19 through 3 staging slots (copy-in, compute and copy-out
    streams; slots reused), each chunk a call with its own scratch (work queue,
    overflow list, L2 state scratch).  Results equal the device-pointer decode for the
    pair SOS kernel, the SOM shared-memory kernel, the C=8 hybrid kernel with
    mixed erasure counts (list mode) and the L2 thread-per-probe kernel; a
    sample equals the oracle."""
    k = (1 << 21) + 4321
    msgs = gbgen.messages(51 + c, m, c, l)
    ee = np.random.default_rng(3).integers(0, c + 1, size=k) if e < 0 else e
    pr, _ = gbgen.probes(52 + c, msgs, k, ee, l, random_count=k // 20)
    net = gb.Net(c, l)
    net.store(to_dev(msgs))
    net.seal()
    dev = as_np(net.decode(to_dev(pr), rule, gamma=2, max_iters=20))
    torch.cuda.synchronize()
    pt = torch.from_numpy(pr.view(np.int16)).pin_memory()
    out = net.alloc_outputs(k, device=False, pin=True)
    net.decode(pt, rule, gamma=2, max_iters=20, out=out)
    same(as_np(out), dev, f"host vs device rule {rule} c={c}")
    idx = np.sort(np.random.default_rng(4).choice(k, 64, replace=False))
    idx[-1] = k - 1
    w, _ = oracle.store(msgs, c, l)
    want = oracle.decode(w, c, l, pr[idx], rule, gamma=2, max_iters=20)
    same(tuple(x[idx] for x in dev), want, "oracle sample")
    net.close()


def test_async_seal_status_and_unseal(gb):
    """gb_seal enqueues and returns; gb_seal_status reports the outcome (invalid
    messages counted once per report; broken invariants unseal); a decode after
    a known-broken seal is refused; gb_weights' writable pointer unseals."""
    c, l = 4, 16
    net = gb.Net(c, l)
    msgs = gbgen.messages(9, 40, c, l)
    bad = np.array([[1, 2, 16, 4]], np.uint16)
    net.store(to_dev(np.concatenate([msgs, bad])))
    net.seal(check=False)
    pr = to_dev(gbgen.probes(10, msgs, 16, 2, l)[0])
    net.decode(pr, 2)                               # issued before the outcome is read: allowed
    with pytest.raises(gb.GBError) as ei:
        net.seal_status()
    assert ei.value.code == gb.GB_EINVAL and "1 stored message" in str(ei.value)
    with pytest.raises(gb.GBError, match="1 stored message"):
        net.seal_status()                           # idempotent: the same seal's outcome
    net.seal()                                      # the skipped message was reported once
    w8 = net.weights()                              # writable pointer out: unsealed
    with pytest.raises(gb.GBError) as ei:
        net.decode(pr, 2)
    assert ei.value.code == gb.GB_ESTATE
    w8[0, 40] = 1                                   # asymmetric
    net.seal(check=False)
    torch.cuda.synchronize()
    with pytest.raises(gb.GBError) as ei:
        net.decode(pr, 2)                           # outcome known (seal done): refused
    assert ei.value.code == gb.GB_ESTATE
    with pytest.raises(gb.GBError, match="asymmetric"):
        net.seal_status()
    w8[0, 40] = 0
    net.seal()
    w, _ = oracle.store(msgs, c, l)
    got = as_np(net.decode(pr, 2, gamma=1))
    same(got, oracle.decode(w, c, l, pr.cpu().numpy().view(np.uint16), 2, gamma=1, max_iters=20), "after reseal")
    net.close()


def test_options_api(gb):
    net = gb.Net(8, 128)
    assert net.option("sos_pair") == 1 and net.option("hyb8_split") == -1 and net.option("som_tensor") == 0
    net.set_option("hyb8", 0)
    assert net.decode_kernel(2) == "decode_smem_kernel"
    for bad in ((99, 1), (0, 2), (0, -1), (5, -2), (7, 1), (7, 5), (7, 9), (7, -1)):
        with pytest.raises(gb.GBError):
            net.set_option(*bad)
    assert net.option("hyb8_rows") == 0 and net.option("sos_bits") == -1
    for v in (-1, 0, 1):
        net.set_option("sos_bits", v)
        assert net.option("sos_bits") == v
    with pytest.raises(gb.GBError):
        net.set_option("sos_bits", 2)
    for nr in (6, 7, 8, 0):
        net.set_option("hyb8_rows", nr)
        assert net.option("hyb8_rows") == nr
    net.close()


@pytest.mark.parametrize("c,l,m", [(4, 2048, 1_500_000), (16, 512, 100_000), (2, 4096, 9_000_000)])
def test_store_large_cluster_blocks(gb, c, l, m):
    """Privatised store at Lp = 512 (m above the scatter threshold), and the
    scattered fallback when one cluster-pair block exceeds the privatised tile
    (Lp = 2048, 4096: Lp^2/8 > 128 KiB) -- W equals the oracle's byte for byte."""
    msgs = gbgen.messages(61 + l, m, c, l)
    net = gb.Net(c, l)
    net.store(to_dev(msgs))
    net.seal()
    w, _ = oracle.store(msgs, c, l)
    got = net.weights().cpu().numpy()
    assert np.array_equal(got, w)          # L is a multiple of 32: no padding
    net.close()


@pytest.mark.parametrize("c,l,m", [(8, 128, 20000), (5, 33, 3000), (16, 256, 100000), (2, 1, 1)])
def test_upper_triangle_exchange(gb, c, l, m):
    """gb_pack_upper carries W in its C(C-1)/2 upper cluster-pair
    blocks (W symmetric); OR-ing the packed sets of message shards
    into an empty net with gb_or_upper (block + mirror) gives the W of the whole
    message set byte for byte (Eq.(1) is an OR of cliques)."""
    msgs = gbgen.messages(81 + c, m, c, l)
    whole = gb.Net(c, l)
    whole.store(to_dev(msgs))
    whole.seal()
    lp = 32 * ((l + 31) // 32)
    assert whole.upper_words() == lp * (lp // 32) * c * (c - 1) // 2
    parts = []
    for i in range(3):
        p_ = gb.Net(c, l)
        p_.store(to_dev(msgs[i::3]))
        p_.seal()
        parts.append(p_.pack_upper())
    merged = gb.Net(c, l)
    merged.or_upper(torch.stack(parts).contiguous())
    merged.seal()
    assert torch.equal(merged.weights_view(), whole.weights_view())
    assert torch.equal(merged.bits(), whole.bits())
    with pytest.raises(gb.GBError):
        gb.Net(c, l).pack_upper()                   # not sealed
    for n in (whole, merged):
        n.close()


@pytest.mark.parametrize("c,l,m,e,k", [(4, 16, 50, 2, 1000), (8, 128, 5000, 4, 3000), (8, 128, 20000, 4, 1500),
                                       (16, 256, 30000, 8, 300), (5, 100, 800, 3, 500), (16, 512, 5000, 7, 200)])
def test_decode_symbols_matches_oracle(gb, c, l, m, e, k):
    """gb_decode_symbols (the retrieved message per cluster: its only active neuron, or
    ERASED / AMBIGUOUS) equals the oracle's final state mapped by oracle.symbols, with the
    same rounds and status, for every rule and kernel family (hyb8, shared-memory, L2, SOS
    pair / streamed-A); invalid probes give ERASED rows; device buffers."""
    msgs = gbgen.messages(1000 + c + l, m, c, l)
    pr, _ = gbgen.probes(1001 + k, msgs, k, e, l, random_count=k // 5)
    pr[1, 0] = l                                   # invalid symbol
    w, _ = oracle.store(msgs, c, l)
    net = gb.Net(c, l)
    net.store(torch.from_numpy(msgs.view(np.int16)).cuda())
    net.seal()
    for rule in (0, 1, 2):
        sym, it, ss = net.decode_symbols(torch.from_numpy(pr.view(np.int16)).cuda(), rule, gamma=2, max_iters=20)
        torch.cuda.synchronize()
        ost, oit, oss = oracle.decode(w, c, l, pr, rule, gamma=2, max_iters=20)
        want = oracle.symbols(ost, c, l)
        got = sym.cpu().numpy().view(np.uint16)
        assert np.array_equal(got, want), (rule, np.flatnonzero((got != want).any(axis=1))[:5])
        assert np.array_equal(it.cpu().numpy().view(np.uint16), oit) and np.array_equal(ss.cpu().numpy(), oss)
        assert (got[1] == oracle.ERASED).all() and ss[1].item() == gb.INVALID
    net.close()


def test_decode_symbols_host_buffers_chunked(gb):
    """gb_decode_symbols with host buffers: 4 * 2^19 + 4321 probes (five staged chunks through
    three staging slots) equal the device-buffer call and gb_decode's states mapped by
    oracle.symbols; hybrid (C=8 kernel) and sum-of-sum (CTA pair)."""
    c, l, m, k = 8, 128, 5000, (1 << 21) + 4321
    msgs = gbgen.messages(77, m, c, l)
    pr, _ = gbgen.probes(78, msgs, k, 4, l)
    net = gb.Net(c, l)
    net.store(torch.from_numpy(msgs.view(np.int16)).cuda())
    net.seal()
    for rule in (2, 0):
        host = net.decode_symbols(torch.from_numpy(pr.view(np.int16)), rule, gamma=2, max_iters=20)
        dev = net.decode_symbols(torch.from_numpy(pr.view(np.int16)).cuda(), rule, gamma=2, max_iters=20)
        st, _, _ = net.decode(torch.from_numpy(pr.view(np.int16)).cuda(), rule, gamma=2, max_iters=20)
        torch.cuda.synchronize()
        for a, b in zip(host, dev):
            assert np.array_equal(a.numpy(), b.cpu().numpy())
        idx = np.arange(0, k, 997)
        want = oracle.symbols(st.cpu().numpy().view(np.uint32)[idx], c, l)
        assert np.array_equal(host[0].numpy().view(np.uint16)[idx], want)
    net.close()
