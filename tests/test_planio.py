"""Persisted plan formats as executor input (planio).

The fixtures under tests/golden/optimize/ are the reference CLI's own
`optimize` output (tests/golden/make_optimize_golden.py).  Lowering them must
give exactly the ExecPlan this package's planner produces for the same DAG and
config, and this package's write_plan must reproduce the reference files."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

from paper_2004_14020_b200 import gradsets, planio
from paper_2004_14020_b200.collective import Pattern, ReduceModel
from paper_2004_14020_b200.costmodel import NetworkModel
from paper_2004_14020_b200.executor import lower
from paper_2004_14020_b200.pipeline import run_pipeline
from paper_2004_14020_b200.sim import DepthPolicy, SimConfig

GOLDEN = Path(__file__).resolve().parent / "golden" / "optimize"
CASES = sorted(p.name for p in GOLDEN.iterdir() if p.is_dir())


def _case(name):
    c = json.loads((GOLDEN / name / "case.json").read_text())
    tensors = gradsets.gradient_set(c["model"])
    numels = {gradsets.param_id(i, len(tensors)): t.numel for i, t in enumerate(tensors)}
    policy = DepthPolicy(adaptive=False, fixed=c["depth"]) if c["depth"] is not None else DepthPolicy()
    cfg = SimConfig(workers=c["workers"], network=NetworkModel(*c["network"]), reduce=ReduceModel(400.0, 10.0),
                    pattern=Pattern(c["pattern"]), depth_policy=policy)
    art = run_pipeline(gradsets.layered_chain_dag(c["model"]), cfg)
    return c, numels, art


def _same(a, b):
    assert a.digest() == b.digest()
    assert a.buckets == b.buckets
    assert (a.arena_bytes, a.param_bytes, a.total_numel) == (b.arena_bytes, b.param_bytes, b.total_numel)


@pytest.mark.parametrize("name", CASES)
def test_reference_optimize_output_lowers_to_our_plan(name):
    c, numels, art = _case(name)
    ours = lower(art, numels, c["workers"], Pattern(c["pattern"]))
    theirs = planio.load_exec_plan(GOLDEN / name, numels, c["workers"], c["pattern"], depth=c["depth"])
    _same(ours, theirs)


@pytest.mark.parametrize("name", CASES)
def test_write_plan_matches_reference_files_and_round_trips(name, tmp_path):
    c, numels, art = _case(name)
    paths = planio.write_plan(art, tmp_path)
    assert [p.name for p in paths] == list(planio.PLAN_FILES)
    ours_bp = json.loads((tmp_path / "batch_plan.json").read_text())
    ref_bp = json.loads((GOLDEN / name / "batch_plan.json").read_text())
    assert all("depth" in g for g in ours_bp["groups"])
    stripped = {**ours_bp, "groups": [{k: v for k, v in g.items() if k != "depth"} for g in ours_bp["groups"]]}
    assert stripped == ref_bp
    assert json.loads((tmp_path / "transfer_schedule.json").read_text()) == \
        json.loads((GOLDEN / name / "transfer_schedule.json").read_text())
    # depths are in the file now: no policy argument needed
    _same(lower(art, numels, c["workers"], Pattern(c["pattern"])),
          planio.load_exec_plan(tmp_path, numels, c["workers"], c["pattern"]))


def test_load_rejects_mismatched_files():
    name = CASES[0]
    c, numels, _ = _case(name)
    bp = json.loads((GOLDEN / name / "batch_plan.json").read_text())
    ts = json.loads((GOLDEN / name / "transfer_schedule.json").read_text())
    ts_short = {**ts, "transfers": ts["transfers"][:-1]}
    with pytest.raises(ValueError, match="disagree"):
        planio.load_exec_plan(numels=numels, world=c["workers"], batch_plan=bp, transfer_schedule=ts_short)
    bad = dict(numels)
    first = bp["groups"][0]["param_ids"][0]
    bad[first] += 1
    with pytest.raises(ValueError, match="fp32 member sizes"):
        planio.load_exec_plan(numels=bad, world=c["workers"], batch_plan=bp, transfer_schedule=ts)
