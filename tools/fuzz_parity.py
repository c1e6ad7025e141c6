"""Randomised parity sweep (evidence, not a unit test): FP4 tensor-core classification vs the
bit-packed CUDA-core kernel on random shapes (N, M, S, K_lower, K_upper), with and without
first matches, including sets that run as several resident-sized or L2-sized launches;
device-stream and shared-stream sampling vs the oracle on random shapes.

    python tools/fuzz_parity.py [seconds]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2604_17066_b200 as P  # noqa: E402
from paper_2604_17066_b200 import _abi  # noqa: E402
from paper_2604_17066_b200.classify import classify_host  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(os.environ.get("SEED", "1")))
t_end = time.time() + budget
n_cls = n_smp = n_host = n_enc = 0
while time.time() < t_end:
    kind = rng.integers(0, 4)
    if kind < 3:  # classification
        m = int(rng.choice([2, 2, 2, 3, 3, 4, 5]))
        n = int(rng.integers(1, 1536 // (m - 1) + 1)) if rng.random() < 0.3 else int(rng.integers(1, 320))
        s = int(rng.integers(1, 40_000))
        kl = int(rng.integers(0, 6000)) if rng.random() < 0.7 else 0
        ku = int(rng.integers(0, 6000)) if rng.random() < 0.8 else 0
        p_hi = rng.uniform(0.6, 0.97)
        probs = np.tile(np.r_[np.full(m - 1, (1 - p_hi) / (m - 1)), p_hi], (n, 1))
        b = P.sample_batch(P.ComponentDistribution(probs), s, seed=int(rng.integers(1 << 30)))
        # references: mostly high states (upper refs rarely hit unless sparse) with a few low
        up = np.where(rng.random((ku, n)) < rng.uniform(0.0, 0.12), rng.integers(1, m, (ku, n)), 0)
        lo = np.where(rng.random((kl, n)) < rng.uniform(0.0, 0.12), rng.integers(0, m - 1, (kl, n)),
                      m - 1)
        lset = P.ReferenceSet.from_array(P.Side.LOWER, 0, lo.astype(np.uint8), trusted=True)
        uset = P.ReferenceSet.from_array(P.Side.UPPER, 0, up.astype(np.uint8), trusted=True)
        explain = bool(rng.random() < 0.4)
        try:
            r = P.classify(b, lset, uset, n_states=m, explain=explain)
        except Exception as e:  # noqa: BLE001
            print("ERROR classify", dict(n=n, m=m, s=s, kl=kl, ku=ku, explain=explain,
                                         rb=_abi.fp4_row_bytes(n, m)), repr(e), flush=True)
            sys.exit(1)
        rb = P.classify(b, lset, uset, n_states=m, method="bits", explain=explain)
        ok = torch.equal(r.labels_device, rb.labels_device)
        if explain:
            ok = ok and np.array_equal(r.first_match_lower, rb.first_match_lower) and \
                np.array_equal(r.first_match_upper, rb.first_match_upper)
        plan = _abi.fp4_plan(s, kl, ku, _abi.fp4_row_bytes(n, m), explain) \
            if _abi.fp4_row_bytes(n, m) <= _abi.FP4_MAX_ROW_BYTES else None
        if not ok:
            print("MISMATCH classify", dict(n=n, m=m, s=s, kl=kl, ku=ku, explain=explain, plan=plan),
                  flush=True)
            sys.exit(1)
        if rng.random() < 0.25:  # the host-fed end-to-end path on the same samples
            method = "tc" if rng.random() < 0.7 else "tc8"
            host = b.device_states().cpu()
            chunk = int(rng.integers(1, s + 1)) if rng.random() < 0.5 else None
            try:
                lab, cnt = classify_host(host, lset, uset, m, chunk_rows=chunk, method=method)
            except ValueError as e:  # rows too wide for the tensor-core kernels: declared
                lab = None
                if "too wide" not in str(e):
                    raise
            if lab is not None and not np.array_equal(np.asarray(lab), rb.labels_device.cpu().numpy()):
                print("MISMATCH classify_host", dict(n=n, m=m, s=s, kl=kl, ku=ku, chunk=chunk,
                                                     method=method), flush=True)
                sys.exit(1)
            n_host += 1
        n_cls += 1
    elif rng.random() < 0.15:  # encodings and the full violation-count matrix vs the oracle
        m = int(rng.integers(2, 7))
        n = int(rng.integers(1, 200))
        h, r = int(rng.integers(1, 300)), int(rng.integers(1, 300))
        xs = rng.integers(0, m, (h, n))
        rs = rng.integers(0, m, (r, n))
        kind = "lower_ref" if rng.random() < 0.5 else "upper_ref"
        es = P.encode_batch(xs, m, "sample")
        er = P.encode_batch(rs, m, kind)
        eo_s, eo_r = oracle.encode(xs, m, "sample"), oracle.encode(rs, m, kind)
        if not np.array_equal(es.data, eo_s) or not np.array_equal(er.data, eo_r) or \
                not np.array_equal(er.packed, np.packbits(eo_r.astype(np.uint8), axis=1)) or \
                not np.array_equal(er.packed_complement,
                                   np.packbits((1 - eo_r).astype(np.uint8), axis=1)):
            print("MISMATCH encode", dict(n=n, m=m, h=h, r=r, kind=kind), flush=True)
            sys.exit(1)
        vc = P.violation_counts(es, er, method="packed" if rng.random() < 0.5 else "unpacked")
        if not np.array_equal(np.asarray(vc), oracle.violation_counts(xs, rs, m, kind)):
            print("MISMATCH violation_counts", dict(n=n, m=m, h=h, r=r, kind=kind), flush=True)
            sys.exit(1)
        n_enc += 1
    else:  # sampling vs the oracle
        m = int(rng.integers(2, 6))
        n = int(rng.integers(1, 400))
        h = int(rng.integers(1, 3000))
        start = int(rng.integers(0, 1 << 34)) if rng.random() < 0.3 else int(rng.integers(0, 5000))
        raw = rng.random((n, m)) + 0.01
        probs = raw / raw.sum(1, keepdims=True)
        stream = "device" if rng.random() < 0.5 else "shared"
        seed, gen = int(rng.integers(1 << 62)), int(rng.integers(1 << 40))
        fp4 = bool(rng.random() < 0.5)
        b = P.sample_batch(P.ComponentDistribution(probs), h, seed=seed, generation_index=gen,
                           start=start, fp4=fp4, rng=stream)
        want = oracle.sample_states(probs, h, seed, gen, start, rng=stream)
        if not np.array_equal(b.device_states().cpu().numpy(), want):
            print("MISMATCH sample", dict(n=n, m=m, h=h, start=start, rng=stream, fp4=fp4), flush=True)
            sys.exit(1)
        n_smp += 1
print(f"fuzz parity: {n_cls} classification cases ({n_host} also through classify_host) and "
      f"{n_smp} sampling cases and {n_enc} encoding / violation-count cases equal "
      f"({budget:.0f} s, seed {os.environ.get('SEED', '1')})")
