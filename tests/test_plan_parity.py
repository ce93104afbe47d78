"""Bit-exact plan parity against fixtures produced by the reference planner
(tests/golden/make_golden.py): activation order, control edges, bucket
membership and member order, windows, depths, modelled times, placement and
launch order -- for the four BASELINE gradient sets and 40 fuzzed graphs."""

from __future__ import annotations

import gzip
import json
from dataclasses import replace
from functools import lru_cache
from pathlib import Path

import pytest

from paper_2004_14020_b200 import collective as C
from paper_2004_14020_b200 import costmodel as CM
from paper_2004_14020_b200 import gradsets
from paper_2004_14020_b200.dag import dag_from_json
from paper_2004_14020_b200.pipeline import run_pipeline
from paper_2004_14020_b200.sim import BASELINE, DEFAULT_SCENARIOS, SimConfig

GOLDEN = Path(__file__).resolve().parent / "golden" / "plans.json.gz"
SCENARIOS = {s.name: s for s in (BASELINE,) + tuple(DEFAULT_SCENARIOS)}


@lru_cache(maxsize=1)
def golden() -> dict:
    with gzip.open(GOLDEN, "rt", encoding="utf-8") as fh:
        return json.load(fh)


def make_config(c: dict) -> SimConfig:
    cfg = SimConfig(workers=c["workers"], network=CM.NetworkModel(*c["network"]),
                    reduce=C.ReduceModel(*c["reduce"]), pattern=C.Pattern(c["pattern"]))
    if c["scenario"] is not None:
        s = SCENARIOS[c["scenario"]]
        cfg = replace(cfg, enforce_order=s.enforce_order, batching=s.batching, fp_scheduling=s.fp_scheduling,
                      depth_policy=s.depth_policy)
    return cfg


def as_json(a) -> dict:
    return json.loads(json.dumps({
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
    }))


def _compare(got: dict, want: dict, label: str) -> None:
    for key in want:
        assert got[key] == want[key], f"{label}: {key} differs"


def _model_cases():
    return [pytest.param(i, id=f"{c['model']}-p{c['config']['workers']}-{c['config']['pattern']}-"
                               f"{'cloud' if c['config']['network'][0] == 1000.0 else 'nvl'}-"
                               f"{c['config']['scenario'] or 'full'}")
            for i, c in enumerate(golden()["models"])]


@pytest.mark.parametrize("idx", _model_cases())
def test_model_plans_bitexact(idx):
    case = golden()["models"][idx]
    art = run_pipeline(gradsets.layered_chain_dag(case["model"]), make_config(case["config"]))
    _compare(as_json(art), case["artifacts"], case["model"])


def test_fuzz_plans_bitexact():
    for i, case in enumerate(golden()["fuzz"]):
        art = run_pipeline(dag_from_json(case["dag"]), make_config(case["config"]))
        _compare(as_json(art), case["artifacts"], f"fuzz[{i}]")


def test_stage_plan_vectors():
    for u in golden()["units"]["stage_plan"]:
        plan = C.stage_plan(C.CollectiveSpec(C.Pattern(u["pattern"]), u["workers"], u["bytes"]))
        assert [[s.transfer_bytes, s.reduce_bytes] for s in plan.stages] == u["stages"], u


def test_adaptive_depth_vectors():
    for d, t, k in golden()["units"]["adaptive_depth"]:
        assert C.adaptive_depth(d, t) == k


def test_batching_threshold_vectors():
    for a, b, t in golden()["units"]["batching_threshold"]:
        assert CM.batching_threshold(CM.NetworkModel(a, b)) == t


def test_collective_time_vectors():
    for pat, p, d, k, net, red, t in golden()["units"]["collective_time"]:
        spec = C.CollectiveSpec(C.Pattern(pat), p, d, k)
        assert C.collective_time(spec, CM.NetworkModel(*net), C.ReduceModel(*red)) == t
