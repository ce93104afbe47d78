"""CPU-side checks: the C ABI library loads and exports exactly what
include/caramel.h declares (no GPU call), host arithmetic of the ABI, the
oracle against the reference's stage arithmetic (golden vectors from the
reference, tests/golden/plans.json.gz), and plan lowering."""

from __future__ import annotations

import ctypes
import gzip
import json
import re
from pathlib import Path

import numpy as np
import pytest

import oracle as O

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "caramel.h"


def _lib():
    from paper_2004_14020_b200 import _native as N

    if not N.LIB_PATH.exists():
        import __graft_entry__

        __graft_entry__.build()
    return N


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(caramel_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("caramel_init", "caramel_pack", "caramel_allreduce", "caramel_allreduce_update",
                     "caramel_finalize", "caramel_last_error", "caramel_allreduce_many", "caramel_unpack"):
        assert required in names


def test_library_exports_every_declared_symbol():
    N = _lib()
    handle = ctypes.CDLL(str(N.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(handle, n)]
    assert not missing, f"declared in caramel.h but not exported: {missing}"
    assert set(N.SIGNATURES) == set(declared_functions()), "ctypes binding out of sync with caramel.h"
    assert N.lib().caramel_abi_version() == 1


def test_chunk_bounds_match_oracle_rule():
    N = _lib()
    for n in (0, 1, 7, 4_000_012, 25_557_032):
        for k in (1, 3, 8):
            for p in (1, 2, 3, 8):
                assert N.chunk_bounds(n, k, p) == O.chunk_bounds(n, k, p)


def test_chunk_rule_agrees_with_reference_float_bytes():
    """Integer bounds equal the reference's float chunk bytes (c*d/k,
    collective.py:124) when 4*k*p divides d, and differ by < 1 element otherwise."""
    for n in (4096, 1 << 20, 1_000_003, 4_000_012 // 4):
        for k in (1, 2, 8):
            for p in (2, 4, 8):
                d = 4 * n
                for c, row in enumerate(O.chunk_bounds(n, k, p)):
                    exact = c * d / k / 4
                    assert abs(row[0] - exact) < 1.0
                    if d % (4 * k * p) == 0:
                        assert row[0] == exact
                        for s in range(p):
                            assert row[s] == exact + s * (d / k / p) / 4


def test_bucket_layout_and_errors():
    N = _lib()
    n = 4 << 20  # above the LL128 cutoff: the plain two-shot region
    ctas, bb, fb = N.bucket_layout(n, 2, N.SHUFFLE, 8)
    # packed bucket + 7 copy-engine staging slots of ceil(n/8)+3 elements (the
    # push engine's inbox region is only laid out with CARAMEL_PUSH=1)
    slot = (4 * (n // 8 + 3) + 15) & ~15
    assert 1 <= ctas <= 128 and bb == 4 * n + 7 * slot and fb > 0
    ll = (4 * 1000 + 8 * 1000 * 9 + 255) // 256 * 256  # LL region: bucket + out + 8 in-slots of 8 B words
    assert N.bucket_layout(1000, 1, N.SHUFFLE, 8)[1] == ll + 7 * ((4 * (125 + 3) + 15) & ~15)
    # LL128 (64K < n <= 512K elements): bucket, then out + 8 in-slots of 128 B lines of 30 floats
    m = 1 << 19
    lines = (m + 29) // 30
    ll128 = ((4 * m + 127) // 128 * 128 + 128 * lines * 9 + 255) // 256 * 256
    assert N.bucket_layout(m, 2, N.SHUFFLE, 8)[1] == ll128 + 7 * ((4 * (m // 8 + 3) + 15) & ~15)
    assert N.bucket_layout(1 << 20, 2, N.SHUFFLE, 1)[1] == 4 << 20  # one rank: no staging
    _, bb_ring, _ = N.bucket_layout(1 << 20, 2, N.RING, 8)
    assert bb_ring == 8 << 20  # input + output halves
    with pytest.raises(N.CaramelError, match="power-of-two"):
        N.bucket_layout(1024, 1, N.HD, 6)
    with pytest.raises(N.CaramelError, match="depth"):
        N.bucket_layout(1024, 9, N.SHUFFLE, 2)
    assert N.flag_bytes_for(3, 5, N.SHUFFLE, 4) == (3 * 5 * 2 * 4 * 4 + 255) & ~255


def _golden():
    with gzip.open(ROOT / "tests" / "golden" / "plans.json.gz", "rt") as fh:
        return json.load(fh)


def test_oracle_data_movement_matches_reference_stage_plan():
    """The oracle executes each pattern on p simulated workers and counts the
    bytes worker 0 pulls and reduces per stage; they must equal the reference's
    stage_plan (golden vectors) for divisible payloads."""
    pat = {"ring": O.RING, "hd": O.HD, "shuffle": O.SHUFFLE}
    checked = 0
    for u in _golden()["units"]["stage_plan"]:
        p, d = u["workers"], u["bytes"]
        if d % (4 * p) or d > 4 * 2**20 or p > 8:
            continue
        n = d // 4
        bufs = [np.ones(n, np.float32) for _ in range(p)]
        _, xfer, red = O.c_allreduce(pat[u["pattern"]], bufs, 1)
        assert [[4 * x, 4 * r] for x, r in zip(xfer, red)] == u["stages"], u
        checked += 1
    assert checked >= 20


def test_oracle_numpy_and_c_agree_bit_exact():
    rng = np.random.default_rng(0)
    for pattern in (O.RING, O.HD, O.SHUFFLE):
        for p in (2, 4, 8):
            for k in (1, 3):
                bufs = [rng.standard_normal(1003).astype(np.float32) for _ in range(p)]
                th = rng.standard_normal(1003).astype(np.float32)
                want = O.np_allreduce(pattern, bufs, k, O.EPI_SGD, 1.0 / p, 0.1, th)
                outs, _, _ = O.c_allreduce(pattern, bufs, k, O.EPI_SGD, 1.0 / p, 0.1, th)
                for o in outs:
                    assert np.array_equal(o.view(np.uint32), want.view(np.uint32))


def test_oracle_fixed_order_is_rank_order_for_shuffle():
    x = [np.float32(1e8), np.float32(1.0), np.float32(-1e8), np.float32(1.0)]
    bufs = [np.array([v], np.float32) for v in x]
    got = O.np_allreduce(O.SHUFFLE, bufs, 1)[0]
    assert got == np.float32(np.float32(np.float32(x[0] + x[1]) + x[2]) + x[3])


def test_oracle_bucket_step_threads_invariant():
    rng = np.random.default_rng(1)
    shapes = [(33,), (1000,), (7, 9), (4096,)]
    grads = [[rng.standard_normal(s).astype(np.float32).ravel() for s in shapes] for _ in range(4)]
    base = [rng.standard_normal(s).astype(np.float32).ravel() for s in shapes]
    outs = []
    for nt in (1, 3, 8):
        params = [b.copy() for b in base]
        O.c_bucket_step(O.SHUFFLE, 2, grads, params, O.EPI_SGD, 0.25, 0.1, nthreads=nt)
        outs.append(np.concatenate(params))
    assert all(np.array_equal(outs[0], o) for o in outs[1:])
    want = O.np_allreduce(O.SHUFFLE, [O.np_pack(g) for g in grads], 2, O.EPI_SGD, 0.25, 0.1, O.np_pack(base))
    assert np.array_equal(outs[0], want)


def test_lowering_is_rank_invariant_and_covers_the_plan():
    _lib()
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    for model in ("resnet50", "inception_v3"):
        ts = gradsets.gradient_set(model)
        numels = {gradsets.param_id(i, len(ts)): t.numel for i, t in enumerate(ts)}
        art = run_pipeline(gradsets.layered_chain_dag(model),
                           SimConfig(workers=8, network=NetworkModel(10.0, 1 / 460e3), reduce=ReduceModel(400, 10)))
        plan = lower(art, numels, 8, Pattern.SHUFFLE)
        assert plan.digest() == lower(art, numels, 8, Pattern.SHUFFLE).digest()
        # launch order = transfer schedule order; members = batch plan members
        assert [b.group_id for b in plan.buckets] == [t.group_id for t in art.transfer_schedule.transfers]
        groups = {g.group_id: g for g in art.batch_plan.groups}
        for b in plan.buckets:
            assert b.param_ids == groups[b.group_id].param_ids
            assert b.depth == art.depths[b.group_id]
            assert b.bucket_off % 256 == 0 and b.flag_off % 256 == 0 and b.param_off % 256 == 0
        assert plan.total_numel == sum(t.numel for t in ts)
        # regions never overlap
        spans = sorted((b.bucket_off, b.flag_off) for b in plan.buckets)
        assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))



def test_push_engine_layout_adds_the_inbox_region(tmp_path):
    """With CARAMEL_PUSH=1 every non-LL two-shot bucket also carries the push
    engine's region: a 256 B header, per-item flags (chunks x 128 KB ranges x
    {READY, DONE} x sources) and 2 x (p-1) inbox slots mirroring the bucket.
    Checked in a fresh process (the switch is read once per process)."""
    import subprocess
    import sys

    code = ("import sys; sys.path.insert(0, %r); from paper_2004_14020_b200 import _native as N; "
            "print(N.bucket_layout(4 << 20, 2, N.SHUFFLE, 8)[1])" % str(ROOT))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         env={**__import__("os").environ, "CARAMEL_PUSH": "1"}, check=True).stdout
    n = 4 << 20
    slot = (4 * (n // 8 + 3) + 15) & ~15
    push = 256 + 2 * 64 * 2 * 8 * 4 + 2 * 7 * (4 * n)  # 2 chunks x 64 ranges of 128 KB
    assert int(out) == 4 * n + push + 7 * slot


def test_lean_shuffle_oracle_equals_the_chunked_restatement():
    """np_shuffle_lean (used for the BASELINE-size GPU parity tests) is the
    chunked two-shot restatement without copies: equal bit for bit."""
    rng = np.random.default_rng(42)
    for p in (2, 3, 8):
        for n, k in ((1, 1), (1000, 3), (4097, 8)):
            bufs = [rng.standard_normal(n).astype(np.float32) for _ in range(p)]
            theta = rng.standard_normal(n).astype(np.float32)
            for epi in (O.EPI_SUM, O.EPI_SCALE, O.EPI_SGD):
                want = O.np_allreduce(O.SHUFFLE, bufs, k, epi, 1.0 / p, 0.1, theta)
                got = O.np_shuffle_lean(bufs, epi, 1.0 / p, 0.1, theta)
                assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_robust_calibration_ignores_an_outlier():
    """executor.calibrate_network_model fits through per-size medians
    (costmodel.fit_network_model_robust).  The round-1 failure case: one
    100.4 us sample among eight ~16 us samples at 64 B moved the plain
    least-squares latency to 26.6 us and the bucket cap 8x."""
    from paper_2004_14020_b200.costmodel import (Measurement, batching_threshold, fit_network_model,
                                                  fit_network_model_robust)

    small = [16.1, 16.3, 15.9, 16.0, 16.2, 100.4, 16.1, 15.8]
    big = [26.0, 26.2, 25.9, 26.1, 26.0, 26.3, 25.8, 26.1]
    meas = [Measurement(64, t) for t in small] + [Measurement(4 << 20, t) for t in big]
    plain = fit_network_model(meas)
    robust = fit_network_model_robust(meas)
    clean = fit_network_model([m for m in meas if m.observed_time_us < 50])
    assert plain.latency_us > 25.0                      # the outlier drags the plain fit
    assert abs(robust.latency_us - 16.05) < 0.2         # median of the 64 B samples (~16.05 us)
    assert abs(robust.latency_us - clean.latency_us) < 0.5
    t_plain, t_robust, t_clean = (batching_threshold(m) for m in (plain, robust, clean))
    assert t_plain > 1.5 * t_clean and abs(t_robust - t_clean) / t_clean < 0.05
    # two sizes: the robust line passes through both medians exactly
    assert robust.latency_us + robust.per_byte_us * 64 == pytest.approx(sorted(small)[3] / 2 + sorted(small)[4] / 2)
    # min statistic = estimate_op_times' rule
    mn = fit_network_model_robust(meas, "min")
    assert mn.latency_us + mn.per_byte_us * 64 == pytest.approx(min(small))
    assert mn.latency_us + mn.per_byte_us * (4 << 20) == pytest.approx(min(big))


def test_overlapped_engine_arguments_are_checked_before_any_device_work():
    """engine= is validated first: an unknown engine, and "ce" / "gated" on a
    configuration they cannot run (world 1, flat gradients, ring), raise
    ValueError on a CPU-only host before the Aggregator touches CUDA."""
    _lib()
    import torch

    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import Aggregator, lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    ts = gradsets.gradient_set("alexnet")
    numels = {gradsets.param_id(i, len(ts)): t.numel for i, t in enumerate(ts)}
    params = {pid: torch.zeros(1) for pid in numels}
    for workers, pattern in ((1, Pattern.SHUFFLE), (2, Pattern.RING), (2, Pattern.SHUFFLE)):
        art = run_pipeline(gradsets.layered_chain_dag(ts),
                           SimConfig(workers=max(workers, 2), network=NetworkModel(10.0, 1 / 460e3),
                                     reduce=ReduceModel(400, 10)))
        plan = lower(art, numels, workers, pattern)
        with pytest.raises(ValueError, match="engine must be"):
            Aggregator(plan, params, engine="nccl")
        for engine in ("ce", "gated"):
            grads = "flat" if (workers, pattern) == (2, Pattern.SHUFFLE) else "bucket"
            with pytest.raises(ValueError, match="needs grads='bucket', world > 1 and the SHUFFLE pattern"):
                Aggregator(plan, params, engine=engine, grads=grads)


def test_host_groups_taper_at_both_ends():
    """The host-buffer pipeline's groups (executor.host_groups): contiguous,
    covering, every group non-empty; flat groups stay under group_bytes (or
    hold one bucket); tapered groups start and end small and double / halve."""
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.executor import host_groups

    for sizes in ([4 * t.numel for t in gradsets.gradient_set("resnet50")], [1 << 20] * 100, [5, 7, 1 << 24, 3]):
        for taper in (0, 2 << 20):
            g = host_groups(sizes, 16 << 20, taper)
            assert g[0][0] == 0 and g[-1][1] == len(sizes)
            assert all(a < b for a, b in g) and all(g[k][1] == g[k + 1][0] for k in range(len(g) - 1))
            nbytes = [sum(sizes[a:b]) for a, b in g]
            assert all(n <= (16 << 20) or b - a == 1 for n, (a, b) in zip(nbytes, g))
            if taper and len(g) > 2:
                assert nbytes[0] <= max(2 << 20, sizes[0]) and nbytes[-1] <= max(2 << 20, max(sizes[g[-1][0]:]))
    g = host_groups([1 << 20] * 100, 16 << 20, 2 << 20)
    assert [sum(1 for _ in range(a, b)) for a, b in g][:4] == [2, 2, 4, 8]
    # group_bytes below the taper still bounds every group
    assert all(b - a == 1 for a, b in host_groups([1 << 20] * 10, 4096, 2 << 20))
