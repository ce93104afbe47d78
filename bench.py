"""Benchmark of the data-parallel aggregation hot path (BASELINE.json metric).

One "step" = one aggregation pass over a model's full fp32 gradient set:
every fusion bucket of the Caramel plan (launch order = TransferSchedule)
runs its sm_100a kernel -- pack the member gradients, reduce-scatter over
NVLink peer memory in fixed rank order, postponed SGD update fused into the
all-gather epilogue (stores straight into every replica's parameters).  At
N = 1 there is no exchange: the kernel is the fused pack -> update pass.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--model resnet50]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)
    python bench.py --impl reference ...   (CPU reference path, rank 0 only)

Prints ONE JSON line on rank 0.  `value` = whole-job aggregated gradient
bytes per second: N x (gradient bytes of the model) / step time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# one hardware queue per stream (set before any CUDA context): the copy-engine
# engine's stream-memory-op waits must not stall unrelated streams
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

METRIC = "exposed comm ms/iter and allreduce bus GB/s at 1/2/4/8 B200 vs NVLink roofline"
NVLINK_MODEL = (10.0, 1.0 / 460e3)      # latency us, us/B (SURVEY §8a "NVLink-ish")
REDUCE_MODEL = (400.0, 10.0)            # CLI defaults (cli.py:102-105); only shapes the modelled times
NVLINK_PEAK_GBS = 770.0                 # B200_PROFILING.md measured peer copy per direction (fallback)
NVLINK_NOMINAL_GBS = 900.0
E2E_GROUP = int(float(os.environ.get("CARAMEL_E2E_GROUP_MB", "16")) * (1 << 20))  # host-path pipelining granularity
#: first / last host group size of the e2e pipeline (host_groups taper; 0 = flat groups)
E2E_TAPER = int(float(os.environ.get("CARAMEL_E2E_TAPER_MB", "2")) * (1 << 20))
#: e2e through a captured host step (Aggregator.capture_step_host_flat) or eager calls
E2E_GRAPH = os.environ.get("CARAMEL_E2E_GRAPH", "1") != "0"
LR = 0.1
ROUNDS = 5  # paired (compute-only, aggregation) rounds of the exposed-communication measurement


def _median(xs):
    v = sorted(xs)
    n = len(v)
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])
MODEL_INDEX = {"vgg16": 0, "resnet50": 1, "inception_v3": 2, "alexnet": 3}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="caramel", choices=["caramel", "reference"])
    ap.add_argument("--model", default="resnet50", choices=sorted(MODEL_INDEX))
    ap.add_argument("--pattern", default="shuffle", choices=["shuffle", "ring", "hd"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-exposed", action="store_true", help="skip the model fwd/bwd exposed-comm measurement")
    ap.add_argument("--batch", type=int, default=64, help="per-GPU batch for the exposed-comm measurement")
    ap.add_argument("--exposed-iters", type=int, default=20)
    ap.add_argument("--exposed-grads", default="bucket", choices=["flat", "bucket"],
                    help="gradient storage of the overlapped Aggregator (bucket = zero-copy)")
    ap.add_argument("--exposed-engine", default="all", choices=["sm", "ce", "gated", "all"],
                    help="overlapped-path engine(s) measured; 'all' reports each and the fastest")
    ap.add_argument("--comm-priority", type=int, default=None,
                    help="CUDA priority of the overlapped comm stream (default: Aggregator.comm_priority)")
    ap.add_argument("--ce-min-mb", type=float, default=None,
                    help="copy-engine engine: buckets below this size use the SM kernels (default: Aggregator's)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the bucket-size sweep (N > 1)")
    ap.add_argument("--grads", default="bucket", choices=["bucket", "flat"],
                    help="gradient layout of the measured Aggregator: bucket = zero-copy (gradients live in the "
                         "symmetric buckets, like DDP gradient_as_bucket_view), flat = one flat buffer + pack")
    ap.add_argument("--no-zero-copy", action="store_true", help="skip the other gradient layout's variant")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.15)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# shared setup
# ---------------------------------------------------------------------------
def build_plan(model: str, world: int, pattern: str):
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    tensors = gradsets.gradient_set(model)
    dag = gradsets.layered_chain_dag(model)
    cfg = SimConfig(workers=max(2, world), network=NetworkModel(*NVLINK_MODEL), reduce=ReduceModel(*REDUCE_MODEL),
                    pattern=Pattern(pattern))
    t0 = time.perf_counter()
    art = run_pipeline(dag, cfg)
    plan_s = time.perf_counter() - t0
    numels = {gradsets.param_id(i, len(tensors)): t.numel for i, t in enumerate(tensors)}
    plan = lower(art, numels, world, Pattern(pattern))
    return tensors, art, plan, plan_s


def env_rank():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    return rank, world, local


# ---------------------------------------------------------------------------
# reference arm: the CPU implementation of the path (oracle port), rank 0
# ---------------------------------------------------------------------------
def cpu_pass(buckets, grads_by_worker, params_host, pattern_code, nthreads, scratch):
    """One CPU aggregation pass over every bucket (launch order, members,
    depth): pack -> collective on `len(grads_by_worker)` simulated workers ->
    SGD update -> unpack."""
    import oracle as O

    p = len(grads_by_worker)
    for members, depth in buckets:
        O.c_bucket_step(pattern_code, depth, [[grads_by_worker[r][pid] for pid in members] for r in range(p)],
                        [params_host[pid] for pid in members], O.EPI_SGD, 1.0 / p, LR, nthreads=nthreads,
                        scratch=scratch)


def reference_plan(model: str, world: int, pattern: str):
    """Buckets (members, depth) in launch order as planned by the REFERENCE
    planner (tests/golden/plans.json.gz, written by make_golden.py from
    overlapsim itself), or None if that configuration was not recorded."""
    import gzip

    path = ROOT / "tests" / "golden" / "plans.json.gz"
    if not path.exists():
        return None
    with gzip.open(path, "rt", encoding="utf-8") as fh:
        doc = json.load(fh)
    for case in doc["models"]:
        c = case["config"]
        if (case["model"] == model and c["workers"] == max(2, world) and c["pattern"] == pattern
                and c["scenario"] is None and tuple(c["network"]) == NVLINK_MODEL):
            a = case["artifacts"]
            members = {g[0]: g[1] for g in a["groups"]}
            return [(members[t[0]], a["depths"][t[0]]) for t in a["transfers"]]
    return None


def make_host_inputs(tensors, world, model, seed_base=1000):
    import numpy as np

    from paper_2004_14020_b200 import gradsets

    ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
    prng = np.random.default_rng(7)
    params = {pid: (prng.standard_normal(t.numel, dtype=np.float32) * np.float32(0.01)) for pid, t in zip(ids, tensors)}
    grads = []
    for r in range(world):
        g = np.random.default_rng(seed_base * (MODEL_INDEX[model] + 1) + r)
        grads.append({pid: g.standard_normal(t.numel, dtype=np.float32) for pid, t in zip(ids, tensors)})
    return ids, params, grads


def run_reference(args) -> int:
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import numpy as np

    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O

    from paper_2004_14020_b200 import gradsets

    tensors = gradsets.gradient_set(args.model)
    buckets = reference_plan(args.model, world, args.pattern)
    plan_src = "reference planner (tests/golden/plans.json.gz)"
    if buckets is None:
        _, _, plan, _ = build_plan(args.model, world, args.pattern)
        buckets = [(list(b.param_ids), b.depth) for b in plan.buckets]
        plan_src = "this package's planner (bit-exact with the reference, tests/test_plan_parity.py)"
    ids, params, grads = make_host_inputs(tensors, world, args.model)
    numel = {pid: t.numel for pid, t in zip(ids, tensors)}
    total = sum(numel.values())
    nthreads = os.cpu_count() or 1
    scratch = np.empty((world + 1) * max(sum(numel[p] for p in m) for m, _ in buckets), np.float32)
    code = {"ring": O.RING, "hd": O.HD, "shuffle": O.SHUFFLE}[args.pattern]
    steps, warm = max(1, args.steps), max(0, args.warmup)
    # bounded: keep the whole run to a few minutes
    t0 = time.perf_counter()
    cpu_pass(buckets, grads, params, code, nthreads, scratch)
    one = time.perf_counter() - t0
    budget = 120.0
    steps = max(1, min(steps, int(budget / max(one, 1e-6))))
    warm = min(warm, max(0, int(30.0 / max(one, 1e-6))))
    for _ in range(warm):
        cpu_pass(buckets, grads, params, code, nthreads, scratch)
    t0 = time.perf_counter()
    for _ in range(steps):
        cpu_pass(buckets, grads, params, code, nthreads, scratch)
    dt = (time.perf_counter() - t0) / steps
    nbytes = 4 * total
    value = world * nbytes / dt / 1e9
    sample = (f"full {args.model} gradient set ({len(tensors)} tensors, {nbytes / 1e6:.1f} MB per worker, "
              f"{len(buckets)} buckets, plan from the {plan_src}) x {world} simulated worker(s), "
              f"{steps} timed pass(es)")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "impl": "reference", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.model} gradient set, Caramel plan, {args.pattern}, p={world}",
                   "model": args.model, "pattern": args.pattern, "buckets": len(buckets)},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": nthreads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# caramel arm
# ---------------------------------------------------------------------------
def time_kernel_gated(agg, torch, reps=20):
    """Average duration of the step's collective launch (caramel_allreduce_many),
    CUDA events on its stream around each launch; a _sleep kernel first holds
    the stream so every launch is queued before the first runs (no host gaps
    inside the brackets)."""
    import ctypes

    from paper_2004_14020_b200 import _native as N

    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda._sleep(int(20e6))
    for a, b in evs:
        if agg._step_needs_epoch(True):  # as Aggregator.step: no advance where the launch needs none
            N.check(N.lib().caramel_epoch_advance(agg.ctx._ctx, ctypes.c_void_p(stream.cuda_stream)))
        a.record(stream)
        agg._launch_range(0, len(agg._live), stream.cuda_stream, N.MANY_FUSED, 0)
        b.record(stream)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return ts[len(ts) // 2]  # ms, median launch


def pack_unpack_bw(torch, tensors, dev, peak_gbs, reps=20):
    """K1 / K4 standalone (pack/unpack GB/s against HBM): every
    gradient of the set as its own allocation (161 tensors for resnet50),
    gathered into one bucket by caramel_pack and scattered back by
    caramel_unpack.  Algorithmic bytes 2 x 4 x elements (read + write);
    median of `reps` launches, CUDA events on the launching stream."""
    import ctypes

    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200 import comm

    grads = [torch.randn(max(1, t.numel), device=dev) for t in tensors]
    n = sum(g.numel() for g in grads)
    bucket = torch.empty(n, device=dev)
    segs = comm.segments_for(grads)
    table = comm.segment_table([segs], dev)
    st = torch.cuda.current_stream().cuda_stream

    def med(fn):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        fn()
        torch.cuda._sleep(int(20e6))
        for a, b in evs:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) for a, b in evs)
        return ts[len(ts) // 2]

    pk = med(lambda: comm.pack(table, len(segs), n, bucket.data_ptr(), st))
    up = med(lambda: comm.unpack(table, len(segs), n, bucket.data_ptr(), False, st))
    ok = all(torch.equal(g, bucket[o.offset:o.offset + o.numel]) for g, o in zip(grads, segs))
    alg = 8 * n
    return {"members": len(grads), "bytes": 4 * n, "alg_bytes_per_launch": alg,
            "pack_ms": round(pk, 4), "pack_gbs": round(alg / (pk * 1e-3) / 1e9, 1),
            "pack_frac": round(alg / (pk * 1e-3) / 1e9 / peak_gbs, 4),
            "unpack_ms": round(up, 4), "unpack_gbs": round(alg / (up * 1e-3) / 1e9, 1),
            "unpack_frac": round(alg / (up * 1e-3) / 1e9 / peak_gbs, 4), "peak_gbs": peak_gbs,
            "round_trip_exact": bool(ok), "kernels": "k_pack / k_unpack (caramel.cu)"}


def nccl_baseline(torch, dist, params, grads_dev, world, steps, warmup, bucket_bytes=25 << 20):
    """Plain bucketed NCCL all-reduce (DDP-style 25 MiB buckets in reverse
    parameter order) + SGD update with torch ops: the compared baseline."""
    ids = list(params)[::-1]
    buckets, cur, cur_b = [], [], 0
    for pid in ids:
        nb = params[pid].numel() * 4
        if cur and cur_b + nb > bucket_bytes:
            buckets.append(cur)
            cur, cur_b = [], 0
        cur.append(pid)
        cur_b += nb
    if cur:
        buckets.append(cur)
    flats = [torch.empty(sum(params[p].numel() for p in b), device=grads_dev[ids[0]].device) for b in buckets]

    def one_step():
        for b, flat in zip(buckets, flats):
            torch.cat([grads_dev[p].reshape(-1) for p in b], out=flat)
            dist.all_reduce(flat)
            off = 0
            for p in b:
                n = params[p].numel()
                params[p].reshape(-1).sub_(flat[off:off + n], alpha=LR / world)
                off += n

    for _ in range(warmup):
        one_step()
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        one_step()
    e.record()
    e.synchronize()
    t = torch.tensor([s.elapsed_time(e) / steps], device=flats[0].device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item(), len(buckets)


B200_REDUCE_MODEL = (2e6, 1.0)  # the reduction runs inside the collective kernel (~2 TB/s effective, 1 us)


def ingested_plan(args, model, compute_only, world, dist, dev, network=None, example_inputs=None):
    """The full Caramel configuration for a real model: DAG ingested from the
    model (module-level ops, device-measured durations, min of 5 runs; max over
    ranks so every rank plans identically), calibrated network model,
    fused-reduction model; lowered to the executor plan."""
    import torch
    from dataclasses import replace as _replace

    from paper_2004_14020_b200.collective import Pattern as _P
    from paper_2004_14020_b200.collective import ReduceModel as _RM
    from paper_2004_14020_b200.costmodel import NetworkModel as _NM
    from paper_2004_14020_b200.dag import DataflowDag as _DAG
    from paper_2004_14020_b200.executor import lower as _lower
    from paper_2004_14020_b200.ingest import ingest_model
    from paper_2004_14020_b200.pipeline import run_pipeline as _rp
    from paper_2004_14020_b200.sim import SimConfig as _SC

    ing = ingest_model(model, compute_only, runs=5, example_inputs=example_inputs)
    op_ids = sorted(o for o, op in ing.dag.ops.items() if op.kind.value == "compute")
    durs = torch.tensor([float(ing.dag.ops[o].duration_us) for o in op_ids], device=dev)
    if dist is not None:
        dist.all_reduce(durs, op=dist.ReduceOp.MAX)
    ops = dict(ing.dag.ops)
    for o, d in zip(op_ids, durs.tolist()):
        ops[o] = _replace(ops[o], duration_us=int(d))
    dag = _DAG(ops=ops, params=dict(ing.dag.params))
    net = network or _NM(*NVLINK_MODEL)
    art = _rp(dag, _SC(workers=max(2, world), network=net, reduce=_RM(*B200_REDUCE_MODEL), pattern=_P(args.pattern)))
    numels = {pid: p.numel() for pid, p in ing.params.items()}
    return ing, art, _lower(art, numels, world, _P(args.pattern)), net


def measure_exposed(args, plan, ids, world, rank, dev, dist, network=None):
    """Exposed communication per iteration, T - C (sim.py:155-157), measured on
    the real model: torchvision `args.model` (random init, synthetic batch,
    bf16 autocast, fp32 parameters and gradients), forward + backward on every
    GPU.  C = compute only (no aggregation, no update).  Caramel: the Aggregator
    launches each bucket from gradient hooks in the enforced order during
    backward, SGD fused.  NCCL: DistributedDataParallel (25 MiB buckets) +
    torch.optim.SGD.  CUDA events around `exposed_iters` iterations, max over ranks."""
    import torch
    import torchvision

    from paper_2004_14020_b200.executor import Aggregator

    size = 299 if args.model == "inception_v3" else 224
    B, K = args.batch, args.exposed_iters

    def make():
        torch.manual_seed(7)
        kw = {"aux_logits": True, "init_weights": False} if args.model == "inception_v3" else {}
        return getattr(torchvision.models, args.model)(**kw).to(dev)

    gen = torch.Generator(device=dev).manual_seed(1000 * (MODEL_INDEX[args.model] + 1) + rank)
    x = torch.randn(B, 3, size, size, device=dev, generator=gen)
    y = torch.randint(0, 1000, (B,), device=dev, generator=gen)
    loss_fn = torch.nn.CrossEntropyLoss()

    def fwd_bwd(m):
        with torch.autocast("cuda", dtype=torch.bfloat16):
            out = m(x)
            if isinstance(out, tuple):  # inception_v3 in training: (logits, aux_logits)
                loss = loss_fn(out[0].float(), y) + 0.4 * loss_fn(out[1].float(), y)
            else:
                loss = loss_fn(out.float(), y)
        loss.backward()

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(K):
            fn()
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / K
        if dist is not None:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = t.item()
        return ms

    model = make()
    named = list(model.named_parameters())
    from paper_2004_14020_b200 import gradsets

    if [tuple(p.shape) for _, p in named] != [t.shape for t in gradsets.gradient_set(args.model)]:
        raise RuntimeError("model parameters do not match the recorded gradient set")
    for p in model.parameters():
        p.grad = torch.zeros_like(p)

    # every arm zeroes its gradients the same way: one _foreach_zero_ over the
    # gradient list (a per-parameter zero_() loop would cost the compute-only
    # arm ~160-290 extra launches and bias T - C low)
    grads_c = [p.grad for p in model.parameters()]

    def compute_only():
        torch._foreach_zero_(grads_c)
        fwd_bwd(model)

    ing, art, mplan, net = ingested_plan(args, model, compute_only, world, dist, dev, network, example_inputs=(x,))
    placements = {}
    for b in mplan.buckets:
        placements[b.placement] = placements.get(b.placement, 0) + 1
    # engines of the overlapped path: "sm" (NVLink kernels) and, at N > 1 with
    # zero-copy gradients, "ce" (copy-engine two-shot, no SM held while bytes
    # move); each measured in 3 rounds alternating with compute-only rounds
    # (clock / thermal drift hits both alike), medians over rounds
    engines = ["sm"] + (["gated", "ce"] if world > 1 and args.exposed_grads == "bucket" else [])
    if args.exposed_engine != "all":
        engines = [args.exposed_engine]
    cs, per_engine, gated = [], {}, 0

    def run_engine(engine, cs, per_engine):
        nonlocal gated
        if args.comm_priority is not None:
            Aggregator.comm_priority = args.comm_priority
        agg = Aggregator(mplan, dict(ing.params), rank=rank, lr=LR, epilogue="sgd", grads=args.exposed_grads,
                         engine=engine)
        try:
            if args.ce_min_mb is not None:
                agg.ce_min_bytes = int(args.ce_min_mb * (1 << 20))
            gated = agg.gate_forward(ing.modules)

            def caramel_step():
                agg.zero_grad()
                agg.begin_iteration()
                fwd_bwd(model)
                agg.finish_iteration(postpone=True)

            ks, ds = [], []
            for _ in range(ROUNDS):
                c = timed(compute_only)
                agg.attach_hooks()
                k = timed(caramel_step)
                agg.detach_hooks()
                cs.append(c)
                ks.append(k)
                ds.append(k - c)
            # exposed = median over rounds of (round's Caramel - round's compute):
            # paired rounds cancel slow clock / thermal drift between rounds
            per_engine[engine] = (_median(ks), _median(ds), min(ds), max(ds))
            agg.sync()
            agg.status()
        finally:
            agg.close()  # hands the model torch-owned storage back
            grads_c[:] = [p.grad for p in model.parameters()]

    errors = {}
    for engine in engines:
        try:
            run_engine(engine, cs, per_engine)
        except Exception as exc:  # recorded in the JSON line; the other engine still runs
            errors[engine] = f"{type(exc).__name__}: {exc}"
    if not per_engine:
        raise RuntimeError(f"no engine completed: {errors}")
    c_ms = _median(cs)
    best = min(per_engine, key=lambda e: per_engine[e][1])
    k_ms, k_exp = per_engine[best][:2]
    torch.cuda.empty_cache()

    nccl_ms = nccl_exp = None
    if dist is not None and not args.no_nccl:
        from torch.nn.parallel import DistributedDataParallel as DDP

        m2 = make()
        ddp = DDP(m2, device_ids=[dev.index], bucket_cap_mb=25, gradient_as_bucket_view=True)
        opt = torch.optim.SGD(m2.parameters(), lr=LR)

        for p in m2.parameters():
            p.grad = torch.zeros_like(p)
        fwd_bwd(ddp)  # the first backward settles DDP's gradient bucket views
        grads_d = [p.grad for p in m2.parameters()]

        def ddp_step():
            torch._foreach_zero_(grads_d)
            fwd_bwd(ddp)
            opt.step()

        ns, nd = [], []
        for _ in range(ROUNDS):
            c = timed(compute_only)
            n = timed(ddp_step)
            ns.append(n)
            nd.append(n - c)
        nccl_ms, nccl_exp = _median(ns), _median(nd)
        nccl_spread = [round(min(nd), 4), round(max(nd), 4)]
        del ddp, m2, opt
        torch.cuda.empty_cache()
    del model
    out = {"compute_ms": round(c_ms, 4), "compute_spread_ms": [round(min(cs), 4), round(max(cs), 4)],
           "caramel_ms": round(k_ms, 4),
           "caramel_exposed_ms": round(k_exp, 4), "engine": best,
           "engines": {e: {"ms": round(v[0], 4), "exposed_ms": round(v[1], 4),
                           "exposed_spread_ms": [round(v[2], 4), round(v[3], 4)]} for e, v in per_engine.items()},
           "engine_errors": errors or None,
           "negative_median_is_error": k_exp < 0,
           "model": f"torchvision {args.model}, batch {B}/GPU, {size}x{size}, bf16 autocast, fp32 grads",
           "iters": K, "rounds": ROUNDS,
           "zero_grad": "torch._foreach_zero_ over the gradient list in every arm (C, Caramel, DDP)",
           "stat": f"exposed = median over {ROUNDS} rounds of (round time - paired compute-only round time); "
                   "spread = [min, max] over the rounds; a negative median is a measurement error, not a result",
           "grads": args.exposed_grads,
           "plan": {"source": "ingested model DAG: unit dataflow traced from the model (ingest.trace_units), "
                              "durations measured (min of 5 runs, max over ranks)",
                    "control_edges": len(art.control_edges),
                    "network_model": [round(net.latency_us, 3), net.per_byte_us], "reduce_model": list(B200_REDUCE_MODEL),
                    "buckets": len(mplan.buckets), "placements": placements, "gated_modules": gated,
                    "modelled_exposed_us": round(art.transfer_schedule.added_iteration_time_us, 1)}}
    if nccl_ms is not None:
        out.update({"nccl_ddp_ms": round(nccl_ms, 4), "nccl_ddp_exposed_ms": round(nccl_exp, 4),
                    "nccl_ddp_exposed_spread_ms": nccl_spread})
    return out


SWEEP_SIZES = tuple(4096 * 4 ** i for i in range(10))  # 4 KiB .. 1 GiB
SWEEP_DEPTHS = (1, 2, 4, 8)
SWEEP_REPS = 3  # repetitions of every sweep row (median reported, [min, max] kept)


def bucket_sweep(torch, dist, world, rank, dev, iters=20, network=None):
    """Config 5: one bucket of S bytes (4 KiB * 4^i up to 1 GiB), adaptive depth
    from the calibrated network model (else the NVLink model), two-shot over
    NVLink (caramel_allreduce, packed input, result in place) vs
    torch.distributed.all_reduce (NCCL) on the same bytes, plus fixed depths
    1/2/4/8 from 1 MiB up.  `iters` calls captured in a CUDA graph (both
    sides; host launch cost excluded), replayed between two CUDA events, max
    over ranks; bus GB/s = 2(p-1)/p*S/t."""
    import ctypes

    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200 import comm
    from paper_2004_14020_b200.collective import adaptive_depth
    from paper_2004_14020_b200.costmodel import NetworkModel, batching_threshold

    thr = batching_threshold(network or NetworkModel(*NVLINK_MODEL))
    big = max(SWEEP_SIZES)
    region = max(N.bucket_layout(big // 4, d, N.SHUFFLE, world)[1] for d in (1, 8))
    region = (region + (1 << 20)) // (1 << 20) * (1 << 20)
    ctx = comm.Context(rank, world, arena_bytes=region + (32 << 20))
    ctx.bootstrap()
    base, _ = ctx.arena_ptrs(0)
    comm._view_fp32(base, big // 4).normal_()
    stream = torch.cuda.current_stream()
    rows = []
    # the copy-engine two-shot on its own context (same layout)
    ce_ctx, ce_epoch = {}, {}
    if N.lib().caramel_ce_available(ctx._ctx):
        c = comm.Context(rank, world, arena_bytes=region + (32 << 20))
        c.bootstrap()
        comm._view_fp32(c.arena_ptrs(0)[0], big // 4).normal_()
        ce_ctx["ce"], ce_epoch["ce"] = c, 0
        # the gated SM engine (stream-front-end waits around a k_gated launch)
        c = comm.Context(rank, world, arena_bytes=region + (32 << 20))
        c.bootstrap()
        comm._view_fp32(c.arena_ptrs(0)[0], big // 4).normal_()
        ce_ctx["gated"], ce_epoch["gated"] = c, 0
    # the NVLS (multicast, in-switch reduction) two-shot: the non-fixed-order mode;
    # its CTAs only issue switch round trips, so it takes the whole GPU
    nvls_ok = ctx.nvls_available()

    def nvls_ctas(n):
        return int(max(1, min(148, n // world // 2048)))
    if nvls_ok:
        ctx.nvls_setup(big + (2 << 20))
        comm._view_fp32(ctx.nvls_base, big // 4).normal_()
    for k, size in enumerate(SWEEP_SIZES):
        n = size // 4
        depth = adaptive_depth(size, thr)
        ctas, _, _ = N.bucket_layout(n, depth, N.SHUFFLE, world)
        # one kernel per call: the launch takes the device epoch + 1 and its last
        # CTA advances the counter (CARAMEL_F_AUTO_EPOCH), like NCCL's one kernel
        b = comm.make_bucket(n, 0, region + k * (1 << 20), depth=depth, pattern=N.SHUFFLE, epilogue=N.EPI_SUM,
                             flags=N.F_AUTO_EPOCH, ctas=ctas)
        b_ce = comm.make_bucket(n, 0, region + k * (1 << 20), depth=depth, pattern=N.SHUFFLE, epilogue=N.EPI_SUM,
                                flags=0, ctas=ctas)

        def timed(fn, graphed=True):
            """Per-call device time of `fn`: `iters` calls captured in one CUDA
            graph (no host launch overhead in the measurement), replayed
            between two events; eager back-to-back calls if capture fails."""
            for _ in range(5):
                fn()
            torch.cuda.synchronize()
            g = None
            if graphed:
                try:
                    g = torch.cuda.CUDAGraph()
                    side = torch.cuda.Stream()
                    side.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                        for _ in range(iters):
                            fn(side)
                    torch.cuda.current_stream().wait_stream(side)
                    g.replay()
                    torch.cuda.synchronize()
                except Exception:
                    g = None
            # SWEEP_REPS repetitions (each `iters` calls, max over ranks); the
            # row reports their median and spread
            reps = []
            for _ in range(SWEEP_REPS):
                dist.barrier()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                if g is not None:
                    g.replay()
                else:
                    for _ in range(iters):
                        fn()
                e.record(stream)
                e.synchronize()
                t = torch.tensor([s.elapsed_time(e) / iters], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                reps.append(t.item() * 1e3)
            spread.append([round(min(reps), 2), round(max(reps), 2)])
            return _median(reps), g is not None  # us

        def caramel(st=None):
            st = st or stream
            ctx.allreduce(b, 0, st.cuda_stream)  # epoch 0 + AUTO_EPOCH: device counter (graph-replayable)

        x = torch.empty(n, device=dev).normal_()
        spread = []
        us_c, gc = timed(caramel)
        us_n, gn = timed(lambda st=None: dist.all_reduce(x))
        bus = 2 * (world - 1) / world * size / 1e3
        row = {"bytes": size, "depth": depth, "caramel_us": round(us_c, 2),
               "caramel_bus_gbs": round(bus / us_c, 1), "nccl_us": round(us_n, 2),
               "nccl_bus_gbs": round(bus / us_n, 1), "graphed": [gc, gn],
               "spread_us": {"caramel": spread[0], "nccl": spread[1]}, "reps": SWEEP_REPS}
        if size >= (1 << 20):
            fixed = {}
            for d in SWEEP_DEPTHS:
                cd, _, _ = N.bucket_layout(n, d, N.SHUFFLE, world)
                bd = comm.make_bucket(n, 0, region + k * (1 << 20), depth=d, pattern=N.SHUFFLE,
                                      epilogue=N.EPI_SUM, flags=N.F_AUTO_EPOCH, ctas=cd)

                def fixed_call(st=None, bd=bd):
                    ctx.allreduce(bd, 0, (st or stream).cuda_stream)

                fixed[str(d)] = round(timed(fixed_call)[0], 2)
            row["fixed_depth_us"] = fixed
        if size >= (1 << 20) and ce_ctx:
            # the copy-engine two-shot and the gated SM engine (eager: their
            # host-side tags cannot replay)
            for key, c in ce_ctx.items():
                fn = N.lib().caramel_allreduce_gated if key == "gated" else N.lib().caramel_allreduce_ce

                def ce_call(st=None, c=c, key=key, fn=fn):
                    ce_epoch[key] += 1
                    N.check(fn(c._ctx, ctypes.byref(b_ce), 1, 0, ce_epoch[key], ctypes.c_void_p(stream.cuda_stream),
                               ctypes.c_void_p(stream.cuda_stream)))
                us_e, _ = timed(ce_call, graphed=False)
                row[f"{key}_us"] = round(us_e, 2)
                row[f"{key}_bus_gbs"] = round(bus / us_e, 1)
        if nvls_ok:
            bn = comm.make_bucket(n, 0, region + k * (1 << 20), depth=depth, pattern=N.SHUFFLE,
                                  epilogue=N.EPI_SUM, flags=0, ctas=nvls_ctas(n))

            def nvls_call(st=None, bn=bn):
                st = st or stream
                N.check(N.lib().caramel_epoch_advance(ctx._ctx, ctypes.c_void_p(st.cuda_stream)))
                ctx.allreduce_nvls(bn, 0, st.cuda_stream)

            us_v, _ = timed(nvls_call)
            row["nvls_us"] = round(us_v, 2)
            row["nvls_bus_gbs"] = round(bus / us_v, 1)  # same 2(p-1)/p*S convention; NVLS moves S per direction
        rows.append(row)
    ctx.status()
    ctx.close()
    for c in ce_ctx.values():
        c.status()
        c.close()
    return rows


def run_caramel(args) -> int:
    import ctypes

    import numpy as np
    import torch

    from paper_2004_14020_b200 import _native as N
    from paper_2004_14020_b200.executor import Aggregator

    rank, world, local = env_rank()
    if world != args.gpus:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
    N.lib()  # fail loudly if the sm_100a library is missing

    tensors, art, plan, plan_s = build_plan(args.model, world, args.pattern)
    ids, params_h, grads_h = make_host_inputs(tensors, 1, args.model, seed_base=1000)
    # this rank's gradients: seed 1000*(config)+rank (mode B)
    g = np.random.default_rng(1000 * (MODEL_INDEX[args.model] + 1) + rank)
    grads_h = {pid: g.standard_normal(t.numel, dtype=np.float32) for pid, t in zip(ids, tensors)}
    shapes = {pid: t.shape for pid, t in zip(ids, tensors)}
    params = {pid: torch.from_numpy(params_h[pid]).to(dev).view(shapes[pid]) for pid in ids}
    agg = Aggregator(plan, params, rank=rank, lr=LR, epilogue="sgd", param_arena=True, grads=args.grads)
    for pid in ids:
        params[pid].grad.copy_(torch.from_numpy(grads_h[pid]).view(shapes[pid]))
    nbytes = 4 * plan.total_numel

    def barrier():
        if dist is not None:
            dist.barrier()

    # warm-up, then capture one step in a CUDA graph
    for _ in range(max(3, args.warmup)):
        agg.step()
    torch.cuda.synchronize()
    agg.status()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    barrier()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            agg.step()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    for _ in range(max(3, args.warmup)):
        graph.replay()
    torch.cuda.synchronize()
    agg.status()

    # ---- timed region: K graph replays, inputs (grads+params) > L2 --------
    barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        s.record()
        for _ in range(args.steps):
            graph.replay()
        e.record()
        e.synchronize()
    barrier()
    ms = s.elapsed_time(e) / args.steps
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    agg.status()
    value = world * nbytes / (ms * 1e-3) / 1e9

    # ---- dominant kernel: per-launch durations (events around each launch)
    barrier()
    kern_ms = time_kernel_gated(agg, torch)
    barrier()
    agg.status()
    if world == 1:
        alg_bytes = 12 * plan.total_numel  # read grad, read theta, write theta
        roof = {"bound": "hbm", "unit": "GB/s", "peak": None, "peak_source": None}
        peaks = ROOT / "MEASURED_PEAKS.json"
        if peaks.exists():
            roof["peak"] = json.loads(peaks.read_text()).get("hbm_gbs")
            roof["peak_source"] = "MEASURED_PEAKS.json hbm_gbs (measured)"
        if roof["peak"] is None:
            roof["peak"], roof["peak_source"] = 6650.0, "B200_PROFILING.md fallback"
    else:
        alg_bytes = plan.bus_bytes()  # 2(p-1)/p * S per bucket, NVLink per direction
        roof = {"bound": "nvlink", "unit": "GB/s", "peak": NVLINK_PEAK_GBS,
                "peak_source": "B200_PROFILING.md measured peer copy per direction (fallback; 900 nominal)"}
    if dist is not None:
        t = torch.tensor([kern_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        kern_ms = t.item()
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    roof.update({"achieved": round(achieved, 1), "frac": round(achieved / roof["peak"], 4),
                 "traffic": None,
                 "kernel": agg.step_kernel() + " (caramel.cu)",
                 "launches_per_step": 1,
                 "kernel_ms_per_step": round(kern_ms, 4),
                 "alg_bytes_per_step": alg_bytes,
                 "alg_bytes_rule": "12 B/elem (grad r, theta r/w)" if world == 1 else "2(p-1)/p x bucket bytes"})
    tr = ROOT / "profiles" / "traffic.json"
    if tr.exists():
        key = f"{args.model}_p{world}_{args.pattern}"
        roof["traffic"] = json.loads(tr.read_text()).get(key)

    # ---- e2e: through the public API with host buffers --------------------
    def measure_e2e(hagg):
        """Aggregator.step_host_flat on a flat-layout Aggregator (host buffers
        are flat; one H2D per group of buckets)."""
        # Aggregator.step_host_flat: pinned host gradients in, updated parameters
        # out (flat, arena layout), H2D / kernels / D2H pipelined per ~16 MB group
        pinned_g = torch.zeros(plan.param_bytes // 4).pin_memory()
        pinned_p = torch.zeros(plan.param_bytes // 4).pin_memory()
        for pid, off, n in hagg.flat_layout():
            pinned_g[off:off + n].copy_(torch.from_numpy(grads_h[pid]))
        per_step = hagg.step_host_flat(pinned_g, pinned_p, group_bytes=E2E_GROUP, taper_bytes=E2E_TAPER)
        graph = None
        if E2E_GRAPH:  # one replay per step: the same copies and launches, no host issue cost
            graph = hagg.capture_step_host_flat(pinned_g, pinned_p, group_bytes=E2E_GROUP, taper_bytes=E2E_TAPER)

        def one_step():
            if graph is not None:
                graph.replay()
                return per_step
            return hagg.step_host_flat(pinned_g, pinned_p, group_bytes=E2E_GROUP, taper_bytes=E2E_TAPER)

        for _ in range(2):
            one_step()
        torch.cuda.synchronize()
        barrier()
        e2e_steps = max(3, min(args.steps, 20))
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        e2e_launches = 0
        for _ in range(e2e_steps):
            e2e_launches += one_step()
        e2.record()
        e2.synchronize()
        e2e_ms = s2.elapsed_time(e2) / e2e_steps
        if dist is not None:
            t = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = t.item()
        hagg.status()
        e2e = {"value": round(world * nbytes / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "ms_per_step": round(e2e_ms, 4),
               "api": ("Aggregator.capture_step_host_flat + replay per step" if graph is not None else
                       "Aggregator.step_host_flat") +
                      " (pinned host grads -> fused aggregation + SGD -> pinned host params)",
               "groups": len(hagg.host_groups(E2E_GROUP, E2E_TAPER)), "taper_bytes": E2E_TAPER, "launches_per_step": e2e_launches // e2e_steps,
               "grads": hagg.grads}
        return e2e

    # ---- the other gradient layout: packed (flat buffer + K1 pack phase) or
    # zero-copy (gradients live in the symmetric buckets) -----------------------
    variant = None
    e2e = measure_e2e(agg) if args.grads == "flat" else None
    other = "flat" if args.grads == "bucket" else "bucket"
    vkey = "packed" if other == "flat" else "zero_copy"
    if not args.no_zero_copy:
        zparams = {pid: torch.from_numpy(params_h[pid]).to(dev).view(shapes[pid]) for pid in ids}
        zagg = Aggregator(plan, zparams, rank=rank, lr=LR, epilogue="sgd", param_arena=True, grads=other)
        for pid in ids:
            zparams[pid].grad.copy_(torch.from_numpy(grads_h[pid]).view(shapes[pid]))
        zg = torch.cuda.CUDAGraph()
        zs = torch.cuda.Stream()
        for _ in range(3):
            zagg.step()
        torch.cuda.synchronize()
        barrier()
        zs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(zs), torch.cuda.graph(zg, stream=zs):
            zagg.step()
        torch.cuda.current_stream().wait_stream(zs)
        for _ in range(3):
            zg.replay()
        torch.cuda.synchronize()
        barrier()
        s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s3.record()
        for _ in range(args.steps):
            zg.replay()
        e3.record()
        e3.synchronize()
        zms = s3.elapsed_time(e3) / args.steps
        if dist is not None:
            t = torch.tensor([zms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            zms = t.item()
        zagg.status()
        if other == "flat":
            e2e = measure_e2e(zagg)
        variant = {"ms_per_step": round(zms, 4), "value": round(world * nbytes / (zms * 1e-3) / 1e9, 3),
                   "bus_gbs": round(plan.bus_bytes() / (zms * 1e-3) / 1e9, 1) if world > 1 else None,
                   "what": ("Aggregator(grads='flat'): gradients in one flat buffer, packed into the buckets "
                            "by the kernel's phase 0" if other == "flat" else
                            "Aggregator(grads='bucket'): autograd writes gradients straight into the symmetric "
                            "NVLink-mapped buckets, no pack phase")}
        del zg
        zagg.close()
        del zparams
    if e2e is None:
        e2e = measure_e2e(agg)

    # ---- NCCL bucketed baseline (N > 1) -------------------------------------
    nccl = None
    if dist is not None and not args.no_nccl:
        bparams = {pid: params[pid].detach().clone() for pid in ids}
        bgrads = {pid: params[pid].grad.detach().clone() for pid in ids}
        nms, nb = nccl_baseline(torch, dist, bparams, bgrads, world, args.steps, max(3, args.warmup))
        nccl = {"ms_per_step": round(nms, 4), "value": round(world * nbytes / (nms * 1e-3) / 1e9, 3),
                "bus_gbs": round(plan.bus_bytes() / (nms * 1e-3) / 1e9, 1) if world > 1 else None,
                "buckets": nb, "bucket_mib": 25}

    # ---- calibrated network model (SURVEY §8f row 1, N > 1) --------------------
    calibrated = None
    if dist is not None:
        from paper_2004_14020_b200.costmodel import batching_threshold
        from paper_2004_14020_b200.executor import calibrate_network_model

        model, meas = calibrate_network_model(world, rank)
        from paper_2004_14020_b200 import gradsets as _gs
        from paper_2004_14020_b200.collective import Pattern as _P, ReduceModel as _RM
        from paper_2004_14020_b200.pipeline import run_pipeline as _rp
        from paper_2004_14020_b200.sim import SimConfig as _SC

        cal_art = _rp(_gs.layered_chain_dag(args.model),
                      _SC(workers=world, network=model, reduce=_RM(*REDUCE_MODEL), pattern=_P(args.pattern)))
        calibrated = {"latency_us": round(model.latency_us, 3), "per_byte_us": model.per_byte_us,
                      "threshold_bytes": batching_threshold(model), "buckets": len(cal_art.batch_plan.groups),
                      "samples": [[m.size_bytes, round(m.observed_time_us, 2)] for m in meas],
                      "fit": "fit_network_model (costmodel.py:84-108) on caramel_allreduce 64 B / 4 MB, max over ranks"}

    # ---- config 5: bucket-size sweep vs NCCL (N > 1) --------------------------
    sweep = None
    if dist is not None and not args.no_sweep:
        try:
            from paper_2004_14020_b200.costmodel import NetworkModel as _NMs

            sweep = bucket_sweep(torch, dist, world, rank, dev,
                                 network=_NMs(calibrated["latency_us"], calibrated["per_byte_us"]) if calibrated else None)
        except Exception as exc:  # recorded, never silently dropped
            sweep = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- exposed communication on the real model (T - C) --------------------
    exposed = None
    if not args.no_exposed:
        agg.close()
        for pid in ids:  # free the step's tensors before the model runs
            params[pid] = None
        torch.cuda.empty_cache()
        from paper_2004_14020_b200.costmodel import NetworkModel as _NM

        net = _NM(calibrated["latency_us"], calibrated["per_byte_us"]) if calibrated else None
        try:
            exposed = measure_exposed(args, plan, ids, world, rank, dev, dist, network=net)
        except Exception as exc:  # recorded, never silently dropped
            exposed = {"error": f"{type(exc).__name__}: {exc}", "caramel_exposed_ms": None}

    # ---- K1 / K4 standalone vs HBM --------------------------------
    hbm_peak = 6650.0
    if (ROOT / "MEASURED_PEAKS.json").exists():
        hbm_peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs") or hbm_peak
    try:
        packbw = pack_unpack_bw(torch, tensors, dev, hbm_peak)
    except Exception as exc:  # recorded, never silently dropped
        packbw = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- CPU baseline (rank 0, N = 1 only) ----------------------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle as O

        nthreads = os.cpu_count() or 1
        scratch = np.empty(2 * max(b.numel for b in plan.buckets), np.float32)
        hp = {pid: params_h[pid].copy() for pid in ids}
        cb = [(list(b.param_ids), b.depth) for b in plan.buckets]
        cpu_pass(cb, [grads_h], hp, O.SHUFFLE, nthreads, scratch)
        reps, t0 = 0, time.perf_counter()
        while reps < 3 or time.perf_counter() - t0 < 2.0:
            cpu_pass(cb, [grads_h], hp, O.SHUFFLE, nthreads, scratch)
            reps += 1
            if time.perf_counter() - t0 > 20.0:
                break
        cdt = (time.perf_counter() - t0) / reps
        cpu = {"value": round(nbytes / cdt / 1e9, 3), "unit": "GB/s", "cores": nthreads, "kind": "port",
               "sample": f"full {args.model} set ({nbytes / 1e6:.1f} MB), {len(plan.buckets)} buckets, "
                         f"{reps} passes of oracle_bucket_step (C, pthreads)"}

    kernels_per_step = agg.kernels_per_step(fused=True)
    bus = plan.bus_bytes() / (ms * 1e-3) / 1e9 if world > 1 else None
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.model} fp32 gradient set ({len(tensors)} tensors, {nbytes / 1e6:.1f} MB/GPU): "
                               f"Caramel plan -> {'pack + ' if args.grads == 'flat' else ''}{args.pattern} all-reduce + fused SGD update",
                   "model": args.model, "pattern": args.pattern, "grads": args.grads, "buckets": len(plan.buckets),
                   "depths": sorted({b.depth for b in plan.buckets}), "parallelism": f"dp{world}",
                   "l2": "working set (grads + params) > 126 MB L2; no flush", "graph": "CUDA graph per step",
                   "network_model": {"latency_us": NVLINK_MODEL[0], "per_byte_us": NVLINK_MODEL[1]},
                   "threshold_bytes": art.threshold_bytes},
        "bus_gbs": round(bus, 1) if bus is not None else None,
        "exposed_comm_ms_per_iter": exposed["caramel_exposed_ms"] if exposed else None,
        "exposed_comm": exposed,
        "bucket_sweep": sweep,
        vkey: variant,
        "calibrated_network_model": calibrated,
        "pack_unpack": packbw,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "nccl_baseline": nccl,
        "clocks": clocks.summary(),
        "gpu_launches": kernels_per_step * args.steps,
        "planner_s": round(plan_s, 3),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if exposed is None:
        agg.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main() -> int:
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_caramel(args)


if __name__ == "__main__":
    sys.exit(main())
