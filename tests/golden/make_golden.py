"""Generate the golden plan fixtures by running the REFERENCE planner.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
It imports overlapsim read-only from /root/reference/pkg/src and writes
tests/golden/plans.json.gz.  tests/test_plan_parity.py then checks this
package's planner against the file bit for bit, with no reference needed.

Contents:
  models   the four BASELINE gradient sets as layered-chain DAGs
           (gradsets.layered_chain_dag), at p in {2,4,8}, under the "cloud"
           model (1000 us, 0.001 us/B) and an NVLink-scale model
           (10 us, 1/460e3 us/B); all three patterns for resnet50 at p=8;
           the five ablation scenarios for resnet50 and inception_v3 at p=4
  fuzz     reference gen_dag graphs (both presets) with their plans
  units    stage_plan / adaptive_depth / batching_threshold / collective_time
           vectors, including non-divisible payloads
"""

from __future__ import annotations

import gzip
import json
import math
import random
import sys
from dataclasses import replace
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))

import overlapsim as R  # noqa: E402  (the reference)
from overlapsim import collective as RC  # noqa: E402
from overlapsim import costmodel as RCM  # noqa: E402
from overlapsim.dag import dag_from_json  # noqa: E402
from overlapsim.generator import gen_dag as ref_gen_dag  # noqa: E402
from overlapsim.pipeline import run_pipeline  # noqa: E402
from overlapsim.sim import DEFAULT_SCENARIOS, BASELINE  # noqa: E402

from paper_2004_14020_b200 import gradsets  # noqa: E402
from paper_2004_14020_b200.dag import dag_to_json  # noqa: E402

CLOUD = (1000.0, 0.001)
NVLINK = (10.0, 1.0 / 460e3)
REDUCE = (400.0, 10.0)


def artifacts_to_json(a) -> dict:
    return {
        "order": list(a.order.param_ids),
        "cumulative_cost_us": list(a.order.cumulative_cost_us),
        "control_edges": [[e.from_op, e.to_op] for e in a.control_edges],
        "threshold_bytes": a.threshold_bytes,
        "groups": [[g.group_id, list(g.param_ids), g.total_bytes, g.ready_time_us, g.earliest_read_us]
                   for g in a.batch_plan.groups],
        "windows": {k: [w.start_us, w.end_us] for k, w in sorted(a.windows.items())},
        "depths": dict(sorted(a.depths.items())),
        "collective_times": dict(sorted(a.collective_times.items())),
        "bp_interval": list(a.bp_interval),
        "fp_interval": list(a.fp_interval),
        "transfers": [[t.group_id, t.begin_us, t.finish_us, t.placement.value]
                      for t in a.transfer_schedule.transfers],
        "added_iteration_time_us": a.transfer_schedule.added_iteration_time_us,
        "makespan_us": a.schedule.makespan_us(),
    }


def config(workers, net, pattern="shuffle", scenario=None):
    cfg = R.SimConfig(workers=workers, network=R.NetworkModel(*net), reduce=R.ReduceModel(*REDUCE),
                      pattern=R.Pattern(pattern))
    if scenario is not None:
        cfg = replace(cfg, enforce_order=scenario.enforce_order, batching=scenario.batching,
                      fp_scheduling=scenario.fp_scheduling, depth_policy=scenario.depth_policy)
    return cfg


def cfg_json(workers, net, pattern, scenario):
    return {"workers": workers, "network": list(net), "reduce": list(REDUCE), "pattern": pattern,
            "scenario": None if scenario is None else scenario.name}


def main() -> None:
    out = {"models": [], "fuzz": [], "units": {}}
    for model in gradsets.MODELS:
        ref_dag = dag_from_json(dag_to_json(gradsets.layered_chain_dag(model)))
        cases = [(p, net, "shuffle", None) for p in (2, 4, 8) for net in (CLOUD, NVLINK)]
        if model == "resnet50":
            cases += [(8, NVLINK, "ring", None), (8, NVLINK, "hd", None), (8, CLOUD, "ring", None)]
        if model in ("resnet50", "inception_v3"):
            cases += [(4, CLOUD, "shuffle", sc) for sc in (BASELINE,) + tuple(DEFAULT_SCENARIOS)]
        for p, net, pat, sc in cases:
            art = run_pipeline(ref_dag, config(p, net, pat, sc))
            out["models"].append({"model": model, "config": cfg_json(p, net, pat, sc),
                                  "artifacts": artifacts_to_json(art)})
            print(model, p, net, pat, sc and sc.name, len(art.batch_plan.groups), flush=True)

    rng = random.Random(2004_14020)
    for seed in range(40):
        n_params = rng.randint(3, 40)
        n_ops = rng.randint(2 * n_params + 4, 2 * n_params + 120)
        preset = "small-heavy" if seed % 2 == 0 else "log-uniform"
        dag = ref_gen_dag(n_ops, n_params, seed=seed, preset=preset)
        p = rng.choice([2, 4, 8])
        net = rng.choice([CLOUD, NVLINK, (500.0, 0.002)])
        pat = rng.choice(["shuffle", "ring", "hd"])
        from overlapsim.dag import dag_to_json as ref_to_json

        art = run_pipeline(dag, config(p, net, pat))
        out["fuzz"].append({"dag": ref_to_json(dag), "config": cfg_json(p, net, pat, None),
                            "artifacts": artifacts_to_json(art)})

    units = out["units"]
    sizes = [1, 3, 4095, 4096, 1_000_000, 4_000_012, 4 * 2**20, 25_000_001, 102_760_448 * 4]
    units["stage_plan"] = [
        {"pattern": pat, "workers": p, "bytes": d,
         "stages": [[s.transfer_bytes, s.reduce_bytes] for s in RC.stage_plan(RC.CollectiveSpec(RC.Pattern(pat), p, d)).stages]}
        for pat in ("ring", "hd", "shuffle") for p in (2, 3, 4, 6, 8, 16) for d in sizes
        if not (pat == "hd" and p & (p - 1))
    ]
    units["adaptive_depth"] = [[d, t, RC.adaptive_depth(d, t)] for d in sizes + [0, 1500001, 6_900_001 * 3]
                               for t in (1, 1000, 1_500_001, 6_900_001)]
    mr = random.Random(7)
    models = [(math.exp(mr.uniform(math.log(0.1), math.log(1e5))), math.exp(mr.uniform(math.log(1e-6), 0.0)))
              for _ in range(200)] + [CLOUD, NVLINK, (0.0, 0.5), (1000.0, 0.01)]
    units["batching_threshold"] = [[a, b, RCM.batching_threshold(RCM.NetworkModel(a, b))] for a, b in models]
    ct = []
    for pat in ("ring", "hd", "shuffle"):
        for p in (2, 4, 8):
            for d in (4096, 65536, 4 * 2**20, 100 * 2**20):
                for k in (1, 2, 3, 8):
                    spec = RC.CollectiveSpec(RC.Pattern(pat), p, d, k)
                    for net in (CLOUD, NVLINK):
                        for red in ((400.0, 10.0), (1000.0, 0.0)):
                            ct.append([pat, p, d, k, list(net), list(red),
                                       RC.collective_time(spec, RCM.NetworkModel(*net), RC.ReduceModel(*red))])
    units["collective_time"] = ct
    path = HERE / "plans.json.gz"
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote", path, path.stat().st_size, "bytes")


if __name__ == "__main__":
    main()
