"""Raw C-ABI kernel parity against the oracle (GPU)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2604_17066_b200 import _abi as A

pytestmark = pytest.mark.gpu


def _dev(x, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(x))
    if dtype is not None:
        t = t.to(dtype)
    return t.cuda()


def test_philox_raw_and_uniform():
    for seed, gen, first, count in [(123, 0, 0, 8), (2**64 - 1, 7, 5, 1001), (9, 2**63 + 3, 12345, 777)]:
        out = torch.empty(count, dtype=torch.int64, device="cuda")
        A.call("rsr_philox_raw", seed, gen, first, count, A.ptr(out), A.stream_ptr())
        got = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, oracle.random_raw(seed, gen, first, count))
    u = torch.empty((33, 13), dtype=torch.float64, device="cuda")
    A.call("rsr_uniform_field", 5, 3, 17, 33, 13, A.ptr(u), A.stream_ptr())
    assert np.array_equal(u.cpu().numpy(), oracle.uniform_field(5, 3, 17, 33, 13))


@pytest.mark.parametrize("n,m,count,start", [(295, 2, 4099, 0), (40, 2, 1000, 3), (7, 3, 513, 11),
                                             (5, 5, 300, 1)])
def test_sample_states_and_thermo(n, m, count, start):
    rng = np.random.default_rng(n * 31 + m)
    raw = rng.random((n, m)) + 0.01
    probs = raw / raw.sum(1, keepdims=True)
    want = oracle.sample_states(probs, count, seed=77, generation_index=2, start=start)
    kpad = A.thermo_kpad(n, m)
    st = torch.empty((count, n), dtype=torch.uint8, device="cuda")
    th = torch.empty((count, kpad), dtype=torch.int8, device="cuda")
    A.call("rsr_sample", A.ptr(_dev(probs)), n, m, 77, 2, start, count, A.ptr(st), A.ptr(th), kpad,
           A.stream_ptr())
    assert np.array_equal(st.cpu().numpy(), want)
    th2 = torch.empty_like(th)
    A.call("rsr_encode_samples", A.ptr(st), count, n, m, A.ptr(th2), kpad, A.stream_ptr())
    assert torch.equal(th, th2)
    kdim = n * (m - 1)
    t = th.cpu().numpy().astype(np.int64)
    for k in range(1, m):
        assert np.array_equal(t[:, [j * (m - 1) + k - 1 for j in range(n)]], (want < k).astype(np.int64))


@pytest.mark.parametrize("n,m,count,start", [(295, 2, 4099, 0), (40, 2, 1000, 3), (7, 3, 513, 11),
                                             (5, 5, 300, 1), (295, 3, 129, 7), (64, 2, 64, 0),
                                             (1, 2, 70, 5)])
def test_sample_fp4_fused(n, m, count, start):
    # row-blocked sampler: states identical to the oracle, FP4 rows identical to the encoder's
    rng = np.random.default_rng(n * 17 + m)
    raw = rng.random((n, m)) + 0.01
    probs = raw / raw.sum(1, keepdims=True)
    want = oracle.sample_states(probs, count, seed=99, generation_index=5, start=start)
    rb = A.fp4_row_bytes(n, m)
    st = torch.empty((count, n), dtype=torch.uint8, device="cuda")
    a4 = torch.empty((count, 2 * rb), dtype=torch.uint8, device="cuda")
    A.call("rsr_sample_fp4", A.ptr(_dev(probs)), n, m, 99, 5, start, count, A.ptr(st), A.ptr(a4), rb,
           A.stream_ptr())
    assert np.array_equal(st.cpu().numpy(), want)
    assert np.array_equal(a4.cpu().numpy(), _fp4_want(want, None, n, m, None))
    only = torch.empty_like(a4)
    A.call("rsr_sample_fp4", A.ptr(_dev(probs)), n, m, 99, 5, start, count, None, A.ptr(only), rb,
           A.stream_ptr())
    assert torch.equal(only, a4)


def _refs_dev(refs, n, m, side):
    kpad = A.thermo_kpad(n, m)
    k = refs.shape[0]
    rows = max(256, (k + 255) // 256 * 256)
    st = _dev(refs.astype(np.uint8))
    out = torch.empty((rows, kpad), dtype=torch.int8, device="cuda")
    A.call("rsr_encode_refs", A.ptr(st) if k else None, k, rows, n, m, side, A.ptr(out), kpad, A.stream_ptr())
    return out


def _classify_tc(samples, lower, upper, n, m):
    kpad = A.thermo_kpad(n, m)
    s = samples.shape[0]
    st = _dev(samples.astype(np.uint8))
    a = torch.empty((s, kpad), dtype=torch.int8, device="cuda")
    A.call("rsr_encode_samples", A.ptr(st), s, n, m, A.ptr(a), kpad, A.stream_ptr())
    bl = _refs_dev(lower, n, m, A.SIDE_LOWER)
    bu = _refs_dev(upper, n, m, A.SIDE_UPPER)
    flags = torch.empty(s, dtype=torch.uint8, device="cuda")
    A.call("rsr_classify_tc", A.ptr(a), s, A.ptr(bl), lower.shape[0], A.ptr(bu), upper.shape[0], kpad,
           A.ptr(flags), 0, A.stream_ptr())
    return flags.cpu().numpy()


def _fp4_rows(bits):
    """Pack 0/1 element rows as e2m1 (1.0 = 0x2), element c in byte c // 2, low nibble first."""
    b = np.asarray(bits, dtype=np.uint8)
    return (b[:, 0::2] * 0x2) | (b[:, 1::2] * 0x20)


def _fp4_want(samples, refs, n, m, side, rows_total=None):
    """numpy restatement of the FP4 operand layout (include/rsr_b200.h)."""
    kdim = n * (m - 1)
    width = 2 * A.fp4_row_bytes(n, m)  # elements per row
    cols = [(j // (m - 1), j % (m - 1) + 1) for j in range(kdim)]
    if samples is not None:
        up = np.zeros((samples.shape[0], width), dtype=np.uint8)
        for c, (j, k) in enumerate(cols):
            up[:, c] = samples[:, j] < k
        lo = np.zeros_like(up)
        lo[:, :kdim] = 1 - up[:, :kdim]
        up[:, kdim] = lo[:, kdim] = 1
        return np.concatenate([_fp4_rows(up), _fp4_rows(lo)], axis=1)
    rows = np.zeros((rows_total, width), dtype=np.uint8)
    for c, (j, k) in enumerate(cols):
        lt = refs[:, j] < k
        rows[: refs.shape[0], c] = (~lt) if side == A.SIDE_UPPER else lt
    rows[refs.shape[0]:, kdim] = 1
    return _fp4_rows(rows)


def _fp4_refs_dev(refs, n, m, side):
    rb = A.fp4_row_bytes(n, m)
    k = refs.shape[0]
    rows = max(240, (k + 239) // 240 * 240)
    out = torch.empty((rows, rb), dtype=torch.uint8, device="cuda")
    A.call("rsr_encode_refs_fp4", A.ptr(_dev(refs.astype(np.uint8))) if k else None, k, rows, n, m,
           side, A.ptr(out), rb, A.stream_ptr())
    return out


def _classify_fp4(samples, lower, upper, n, m, first=False):
    rb = A.fp4_row_bytes(n, m)
    s = samples.shape[0]
    a = torch.empty((s, 2 * rb), dtype=torch.uint8, device="cuda")
    A.call("rsr_encode_samples_fp4", A.ptr(_dev(samples.astype(np.uint8))), s, n, m, A.ptr(a), rb,
           A.stream_ptr())
    bl = _fp4_refs_dev(lower, n, m, A.SIDE_LOWER)
    bu = _fp4_refs_dev(upper, n, m, A.SIDE_UPPER)
    flags = torch.empty(s, dtype=torch.uint8, device="cuda")
    if first:
        fl = torch.empty(s, dtype=torch.int64, device="cuda")
        fu = torch.empty(s, dtype=torch.int64, device="cuda")
        A.call("rsr_classify_fp4_explain", A.ptr(a), s, A.ptr(bl), lower.shape[0], A.ptr(bu),
               upper.shape[0], rb, A.ptr(flags), A.ptr(fl), A.ptr(fu), 0, A.stream_ptr())
        return flags.cpu().numpy(), fl.cpu().numpy(), fu.cpu().numpy()
    A.call("rsr_classify_fp4", A.ptr(a), s, A.ptr(bl), lower.shape[0], A.ptr(bu), upper.shape[0], rb,
           A.ptr(flags), 0, A.stream_ptr())
    return flags.cpu().numpy()


@pytest.mark.parametrize("n,m,s,k", [(295, 2, 300, 250), (7, 3, 33, 5), (64, 2, 10, 0), (63, 2, 5, 3),
                                     (100, 4, 17, 241)])
def test_fp4_encoders_layout(n, m, s, k):
    rng = np.random.default_rng(n + m)
    samples = rng.integers(0, m, size=(s, n))
    refs = rng.integers(0, m, size=(k, n))
    rb = A.fp4_row_bytes(n, m)
    assert rb == A.call("rsr_fp4_row_bytes", n, m) and rb % 32 == 0 and 2 * rb > n * (m - 1)
    a = torch.empty((s, 2 * rb), dtype=torch.uint8, device="cuda")
    A.call("rsr_encode_samples_fp4", A.ptr(_dev(samples.astype(np.uint8))), s, n, m, A.ptr(a), rb,
           A.stream_ptr())
    assert np.array_equal(a.cpu().numpy(), _fp4_want(samples, None, n, m, None))
    for side in (A.SIDE_LOWER, A.SIDE_UPPER):
        got = _fp4_refs_dev(refs, n, m, side).cpu().numpy()
        assert np.array_equal(got, _fp4_want(None, refs, n, m, side, got.shape[0]))


def _classify_bits(samples, lower, upper, n, m, first=False):
    w = A.thermo_words(n, m)
    s = samples.shape[0]

    def pack(x, invert):
        out = torch.zeros((max(1, x.shape[0]), w), dtype=torch.int32, device="cuda")
        if x.shape[0]:
            A.call("rsr_pack_thermo_bits", A.ptr(_dev(x.astype(np.uint8))), x.shape[0], n, m, invert,
                   A.ptr(out), w, A.stream_ptr())
        return out
    sb, lb, ub = pack(samples, 0), pack(lower, 0), pack(upper, 1)
    flags = torch.empty(s, dtype=torch.uint8, device="cuda")
    fl = torch.empty(s, dtype=torch.int64, device="cuda") if first else None
    fu = torch.empty(s, dtype=torch.int64, device="cuda") if first else None
    A.call("rsr_classify_bits", A.ptr(sb), s, A.ptr(lb), lower.shape[0], A.ptr(ub), upper.shape[0], w,
           A.ptr(flags), A.ptr(fl), A.ptr(fu), 0, A.stream_ptr())
    if first:
        return flags.cpu().numpy(), fl.cpu().numpy(), fu.cpu().numpy()
    return flags.cpu().numpy()


def _want_flags(samples, lower, upper, m):
    hl, _ = oracle.dominance_hits(samples, lower, m, oracle.LOWER)
    hu, _ = oracle.dominance_hits(samples, upper, m, oracle.UPPER)
    return hl.astype(np.uint8) | (hu.astype(np.uint8) << 1)


@pytest.mark.parametrize("n,m,s,kl,ku,p1", [
    (295, 2, 3000, 300, 260, 0.5),
    (295, 2, 1000, 1, 129, 0.9),
    (40, 2, 777, 50, 0, 0.9),
    (13, 3, 2000, 37, 41, 0.6),
    (100, 3, 600, 200, 130, 0.5),
    (9, 4, 500, 20, 20, 0.5),
    (200, 4, 300, 64, 64, 0.5),
])
@pytest.mark.parametrize("resident", ["1", "0"])
def test_classifiers_match_oracle(n, m, s, kl, ku, p1, resident, monkeypatch):
    # resident: small reference sets stay in shared memory for the whole launch
    # (RSR_FP4_RESIDENT=0 forces the streaming ring)
    monkeypatch.setenv("RSR_FP4_RESIDENT", resident)
    rng = np.random.default_rng(n + 1000 * m + s)
    samples = rng.integers(0, m, size=(s, n))
    if m == 2:
        samples = (rng.random((s, n)) < p1).astype(np.int64)
    # references near the samples so both sides get hits
    lower = np.clip(samples[rng.integers(0, s, kl)] + rng.integers(0, 2, (kl, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, s, ku)] - rng.integers(0, 2, (ku, n)), 0, m - 1)
    want = _want_flags(samples, lower, upper, m)
    # the references were drawn next to sample rows, so every non-empty side hits
    assert bool((want & 1).any()) == (kl > 0) and bool((want & 2).any()) == (ku > 0)
    got_tc = _classify_tc(samples, lower, upper, n, m)
    assert np.array_equal(got_tc, want), f"tc mismatch at {np.flatnonzero(got_tc != want)[:10]}"
    got_fp4 = _classify_fp4(samples, lower, upper, n, m)
    assert np.array_equal(got_fp4, want), f"fp4 mismatch at {np.flatnonzero(got_fp4 != want)[:10]}"
    got_bits = _classify_bits(samples, lower, upper, n, m)
    assert np.array_equal(got_bits, want)


@pytest.mark.parametrize("resident", ["1", "0"])
@pytest.mark.parametrize("chunk_tiles", ["1", "2", "3"])
def test_reference_chunked_launches(chunk_tiles, resident, monkeypatch):
    # B split across several launches (lower tail + upper head in one chunk, etc.)
    monkeypatch.setenv("RSR_TC_CHUNK_TILES", chunk_tiles)
    monkeypatch.setenv("RSR_FP4_RESIDENT", resident)
    n, m, s = 120, 2, 2500
    rng = np.random.default_rng(17)
    samples = (rng.random((s, n)) < 0.5).astype(np.int64)
    lower = np.clip(samples[rng.integers(0, s, 700)] + rng.integers(0, 2, (700, n)), 0, 1)
    upper = np.clip(samples[rng.integers(0, s, 600)] - rng.integers(0, 2, (600, n)), 0, 1)
    got = _classify_tc(samples, lower, upper, n, m)
    assert np.array_equal(got, _want_flags(samples, lower, upper, m))
    assert np.array_equal(_classify_fp4(samples, lower, upper, n, m), _want_flags(samples, lower, upper, m))


@pytest.mark.parametrize("n,m", [(295, 2), (295, 3), (440, 2), (120, 4), (831, 2)])
def test_fp4_first_match_and_widths(n, m):
    # every supported row width class (cq = 1 .. 14 chunks), first-match indices vs oracle
    rng = np.random.default_rng(n * 7 + m)
    s, kl, ku = 1100, 500, 700
    samples = rng.integers(0, m, size=(s, n))
    lower = np.clip(samples[rng.integers(0, s, kl)] + rng.integers(0, 2, (kl, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, s, ku)] - rng.integers(0, 2, (ku, n)), 0, m - 1)
    want = oracle.classify_labels(samples, lower, upper, m, want_first=True)
    flags, fl, fu = _classify_fp4(samples, lower, upper, n, m, first=True)
    assert np.array_equal(flags, _want_flags(samples, lower, upper, m))
    hl, fl_want = oracle.dominance_hits(samples, lower, m, oracle.LOWER, want_first=True)
    hu, fu_want = oracle.dominance_hits(samples, upper, m, oracle.UPPER, want_first=True)
    assert np.array_equal(fl, fl_want) and np.array_equal(fu, fu_want)
    assert want["labels"].shape == (s,)


def test_first_match_and_violation_counts():
    rng = np.random.default_rng(3)
    n, m = 9, 3
    samples = rng.integers(0, m, size=(500, n))
    refs = rng.integers(0, m, size=(200, n))
    flags, fl, fu = _classify_bits(samples, refs, refs, n, m, first=True)
    r = oracle.classify_labels(samples, refs, refs, m, want_first=True)
    assert np.array_equal(fl, r["first_lower"]) and np.array_equal(fu, r["first_upper"])
    sd, rd = _dev(samples.astype(np.uint8)), _dev(refs.astype(np.uint8))  # keep both alive
    for side, kind in ((A.SIDE_LOWER, "lower_ref"), (A.SIDE_UPPER, "upper_ref")):
        out = torch.empty((500, 200), dtype=torch.int32, device="cuda")
        A.call("rsr_violation_counts", A.ptr(sd), 500, A.ptr(rd), 200, n, side, A.ptr(out),
               A.stream_ptr())
        assert np.array_equal(out.cpu().numpy(), oracle.violation_counts(samples, refs, m, kind))


def test_finalize_and_compact():
    rng = np.random.default_rng(5)
    s = 100_003
    flags = rng.integers(0, 4, s).astype(np.uint8)
    f = _dev(flags)
    labels = torch.empty(s, dtype=torch.uint8, device="cuda")
    counts = torch.empty(4, dtype=torch.int64, device="cuda")
    A.call("rsr_finalize", A.ptr(f), s, A.ptr(labels), A.ptr(counts), A.stream_ptr())
    lab = labels.cpu().numpy()
    want = np.where(flags & 1, 0, np.where(flags & 2, 1, 2)).astype(np.uint8)
    assert np.array_equal(lab, want)
    assert counts.cpu().tolist() == [int((want == 0).sum()), int((want == 1).sum()),
                                     int((want == 2).sum()), int((flags == 3).sum())]
    scratch = torch.empty(A.call("rsr_compact_scratch", s), dtype=torch.int64, device="cuda")
    for label in (0, 1, 2):
        idx = torch.empty(s, dtype=torch.int64, device="cuda")
        cnt = torch.empty(1, dtype=torch.int64, device="cuda")
        A.call("rsr_compact", A.ptr(labels), s, label, A.ptr(idx), A.ptr(cnt), A.ptr(scratch), A.stream_ptr())
        c = int(cnt.item())
        assert np.array_equal(idx[:c].cpu().numpy(), np.flatnonzero(want == label))


def _grid(rows=5, cols=5):
    edges = [(r * cols + c, r * cols + c + 1) for r in range(rows) for c in range(cols - 1)]
    edges += [(r * cols + c, (r + 1) * cols + c) for r in range(rows - 1) for c in range(cols)]
    return rows * cols, edges


def _phi_desc(kind, n_nodes, edges, s, t, m, k=0, keep=None, flags=0):
    eu = _dev(np.array([e[0] for e in edges], dtype=np.int32))
    ev = _dev(np.array([e[1] for e in edges], dtype=np.int32))
    d = A.PhiDesc(kind, len(edges), m, n_nodes, s, t, k, 0, eu.data_ptr(), ev.data_ptr(), None, None,
                  flags)
    if keep is not None:
        keep.extend([eu, ev])
    return d


def _nn_graph():
    from paper_2604_17066_b200 import workloads as W
    g = W.cfg3(0)
    return g["n_nodes"], g["edges"], g["source"], g["target"]


# flags 0: edge-sweep label propagation (csrc/phi.cu); flags 1: bitset BFS (csrc/phi_bits.cu)
# and, for boundary searches, union-find / witness-path search (csrc/boundary_graph.cu) unless
# RSR_BOUNDARY_GRAPH=0
@pytest.mark.parametrize("graph_search", ["1", "0"])
@pytest.mark.parametrize("flags", [0, A.PHI_FLAG_SIMPLE])
@pytest.mark.parametrize("graph", ["grid", "nn119"])
@pytest.mark.parametrize("kind,m", [(A.PHI_ST, 2), (A.PHI_WIDEST, 3), (A.PHI_GLOBAL, 2),
                                    (A.PHI_ST, 3), (A.PHI_WIDEST, 4)])
def test_phi_eval_and_boundary(kind, m, graph, flags, graph_search, monkeypatch):
    monkeypatch.setenv("RSR_BOUNDARY_GRAPH", graph_search)
    if graph == "grid":
        nn, edges = _grid()
        s_node, t_node = 0, nn - 1
    else:
        nn, edges, s_node, t_node = _nn_graph()
    keep = []
    d = _phi_desc(kind, nn, edges, s_node, t_node, m, keep=keep, flags=flags)
    rng = np.random.default_rng(kind)
    xs = rng.integers(0, m, size=(2000, len(edges)))
    if m == 2:
        xs = (rng.random((2000, len(edges))) < 0.7).astype(np.int64)
    if kind == A.PHI_ST:
        ref = oracle.phi_st(nn, edges, s_node, t_node)
    elif kind == A.PHI_WIDEST:
        ref = oracle.phi_widest(nn, edges, s_node, t_node, m)
    else:
        ref = oracle.phi_global(nn, edges)
    want = np.array([ref(x) for x in xs])
    out = torch.empty(2000, dtype=torch.uint8, device="cuda")
    xd = _dev(xs.astype(np.uint8))
    A.call("rsr_phi_eval", A.ctypes.byref(d), A.ptr(xd), None, 2000, A.ptr(out), 0, None,
           A.stream_ptr())
    assert np.array_equal(out.cpu().numpy(), want)
    ms = m if kind == A.PHI_WIDEST else 2
    for thr in range(ms - 1):
        B = 64
        x0 = xs[:B]
        refs = torch.empty((B, len(edges)), dtype=torch.uint8, device="cuda")
        side = torch.empty(B, dtype=torch.uint8, device="cuda")
        calls = torch.empty(B, dtype=torch.int64, device="cuda")
        x0d = _dev(x0.astype(np.uint8))
        A.call("rsr_boundary_search", A.ctypes.byref(d), thr, A.ptr(x0d), B,
               A.ptr(refs), A.ptr(side), A.ptr(calls), A.stream_ptr())
        for b in range(0, B, 1 if graph == "grid" else 8):
            ev = oracle.CountingPhi(ref, len(edges), m, ms)
            vec, sd = oracle.boundary_search(ev, x0[b], thr)
            assert tuple(refs[b].cpu().tolist()) == vec
            assert int(side[b]) == (A.SIDE_LOWER if sd == oracle.LOWER else A.SIDE_UPPER)
            assert int(calls[b]) == ev.count


@pytest.mark.parametrize("tile_n", [160, 176, 192, 208, 224, 240])
@pytest.mark.parametrize("n,m", [(295, 2), (120, 3)])
def test_fp4_tile_widths_and_pad_rows(tile_n, n, m, monkeypatch):
    # every MMA N the launch can pick (RSR_FP4_TILE_N forces one), reference
    # counts that leave partial tiles, with the pad rows readable (avail = padded
    # rows: no masking) and without (avail = n: masked columns); first-match too
    monkeypatch.setenv("RSR_FP4_TILE_N", str(tile_n))
    rng = np.random.default_rng(tile_n + n + m)
    s, kl, ku = 700, 301, 517
    samples = rng.integers(0, m, size=(s, n))
    lower = np.clip(samples[rng.integers(0, s, kl)] + rng.integers(0, 2, (kl, n)), 0, m - 1)
    upper = np.clip(samples[rng.integers(0, s, ku)] - rng.integers(0, 2, (ku, n)), 0, m - 1)
    want = _want_flags(samples, lower, upper, m)
    _, fl_want = oracle.dominance_hits(samples, lower, m, oracle.LOWER, want_first=True)
    _, fu_want = oracle.dominance_hits(samples, upper, m, oracle.UPPER, want_first=True)
    rb = A.fp4_row_bytes(n, m)
    a = torch.empty((s, 2 * rb), dtype=torch.uint8, device="cuda")
    A.call("rsr_encode_samples_fp4", A.ptr(_dev(samples.astype(np.uint8))), s, n, m, A.ptr(a), rb,
           A.stream_ptr())
    bl = _fp4_refs_dev(lower, n, m, A.SIDE_LOWER)
    bu = _fp4_refs_dev(upper, n, m, A.SIDE_UPPER)
    for al, au in ((kl, ku), (bl.shape[0], bu.shape[0])):
        flags = torch.empty(s, dtype=torch.uint8, device="cuda")
        fl = torch.empty(s, dtype=torch.int64, device="cuda")
        fu = torch.empty(s, dtype=torch.int64, device="cuda")
        A.call("rsr_classify_fp4_ex", A.ptr(a), s, None, A.ptr(bl), kl, al, A.ptr(bu), ku, au, rb,
               A.ptr(flags), A.ptr(fl), A.ptr(fu), 0, A.stream_ptr())
        assert np.array_equal(flags.cpu().numpy(), want)
        assert np.array_equal(fl.cpu().numpy(), fl_want) and np.array_equal(fu.cpu().numpy(), fu_want)
        A.call("rsr_classify_fp4_ex", A.ptr(a), s, None, A.ptr(bl), kl, al, A.ptr(bu), ku, au, rb,
               A.ptr(flags), None, None, 0, A.stream_ptr())
        assert np.array_equal(flags.cpu().numpy(), want)


@pytest.mark.parametrize("n,m,batch", [(9, 2, 1), (9, 3, 17), (40, 2, 64), (7, 4, 300), (295, 2, 64)])
def test_refset_insert_matches_sequential_insert(n, m, batch):
    """rsr_refset_insert (csrc/refset.cu) over several batches against the oracle's
    sequential ReferenceSet.insert (boundary.py:87-108): candidates drawn near each other
    so batches contain duplicates, redundant candidates and candidates that drop
    earlier members (of the same batch and of previous batches), both sides mixed."""
    import ctypes
    rng = np.random.default_rng(n * 31 + m * 7 + batch)
    rb = A.fp4_row_bytes(n, m)
    cap = 4096
    sets = []
    for side in (A.SIDE_LOWER, A.SIDE_UPPER):
        rows = torch.zeros((cap, n), dtype=torch.uint8, device="cuda")
        fp4 = torch.empty((cap, rb), dtype=torch.uint8, device="cuda")
        A.call("rsr_encode_refs_fp4", None, 0, cap, n, m, side, A.ptr(fp4), rb, A.stream_ptr())
        alive = torch.zeros(cap, dtype=torch.uint8, device="cuda")
        ctr = torch.zeros(2, dtype=torch.int64, device="cuda")
        d = A.RefsetDev(rows.data_ptr(), fp4.data_ptr(), alive.data_ptr(), ctr.data_ptr(), cap, cap)
        sets.append((rows, fp4, alive, ctr, d))
    report = torch.zeros(8, dtype=torch.int64, device="cuda")
    scratch = torch.empty(A.call("rsr_refset_scratch", batch, rb), dtype=torch.uint8, device="cuda")
    outcome = torch.empty(batch, dtype=torch.uint8, device="cuda")
    calls = torch.arange(batch, dtype=torch.int64, device="cuda")
    want = {A.SIDE_LOWER: oracle.RefSet(oracle.LOWER, 0), A.SIDE_UPPER: oracle.RefSet(oracle.UPPER, 0)}
    base = rng.integers(0, m, size=n)
    redundant = 0
    for _ in range(4):
        cands = np.clip(base[None, :] + rng.integers(-1, 2, size=(batch, n)), 0, m - 1).astype(np.uint8)
        dup = rng.random(batch) < 0.2
        cands[1:][dup[1:]] = cands[:-1][dup[1:]]
        side = rng.integers(0, 2, size=batch).astype(np.uint8)
        want_out = []
        for c in range(batch):
            o = want[int(side[c])].insert(cands[c])
            want_out.append(1 if o == "inserted" else 2)
            redundant += o == "redundant"
        cd, sd = _dev(cands), _dev(side)
        A.call("rsr_refset_insert", A.ptr(cd), A.ptr(sd), batch, n, m, ctypes.byref(sets[0][4]),
               ctypes.byref(sets[1][4]), A.ptr(calls), A.ptr(outcome), A.ptr(report),
               A.ptr(scratch), A.stream_ptr())
        assert outcome.cpu().tolist() == want_out
        rep = report.cpu().tolist()
        assert rep[4] == redundant and rep[6] == batch * (batch - 1) // 2 and rep[7] == 0
        for k, s in ((0, A.SIDE_LOWER), (1, A.SIDE_UPPER)):
            rows, fp4, alive, ctr, _ = sets[k]
            nrow = int(ctr[0].item())
            live = alive[:nrow].cpu().numpy().astype(bool)
            got = [tuple(int(v) for v in r) for r in rows[:nrow].cpu().numpy()[live]]
            assert got == want[s].members
            assert int(ctr[1].item()) == len(want[s].members) == rep[2 * k + 1]
            # the FP4 rows of the members are the encoder's, pad rows past the count
            enc = torch.empty_like(fp4)
            A.call("rsr_encode_refs_fp4", A.ptr(rows), nrow, cap, n, m, s, A.ptr(enc), rb,
                   A.stream_ptr())
            assert torch.equal(enc, fp4)


@pytest.mark.parametrize("kl,ku", [(0, 1500), (0, 2200), (0, 2600), (0, 3000), (2000, 0), (600, 600),
                                   (900, 1000), (1300, 1400)])
@pytest.mark.parametrize("first", [False, True])
def test_fp4_mid_size_sets_resident_and_streamed(kl, ku, first):
    # one-sided launches buffer one sample half, and a set that fits only next to
    # two sample buffers drops the third: the tile width and residency the launch
    # picks change across these sizes; the hitting references sit in the last tile
    n, m, s = 295, 2, 1500
    rng = np.random.default_rng(kl * 7 + ku)
    samples = (rng.random((s, n)) < 0.9).astype(np.int64)
    # non-hitting bulk: lower refs with many zeros, upper refs with many ones
    lower = (rng.random((kl, n)) < 0.2).astype(np.int64)
    upper = (rng.random((ku, n)) < 0.98).astype(np.int64)
    for refs, sign in ((lower, 1), (upper, -1)):
        k = refs.shape[0]
        if k:
            near = samples[rng.integers(0, s, 8)]
            refs[k - 8:] = np.clip(near + sign * rng.integers(0, 2, near.shape), 0, 1)
    want = _want_flags(samples, lower, upper, m)
    assert bool((want & 1).any()) == (kl > 0) and bool((want & 2).any()) == (ku > 0)
    if first:
        got, fl, fu = _classify_fp4(samples, lower, upper, n, m, first=True)
        _, wl = oracle.dominance_hits(samples, lower, m, oracle.LOWER, want_first=True)
        _, wu = oracle.dominance_hits(samples, upper, m, oracle.UPPER, want_first=True)
        assert np.array_equal(fl, wl) and np.array_equal(fu, wu)
    else:
        got = _classify_fp4(samples, lower, upper, n, m)
    assert np.array_equal(got, want), f"mismatch at {np.flatnonzero(got != want)[:10]}"
