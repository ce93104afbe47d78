"""DAG ingestion from real models, on the CPU.

The unit dataflow of torchvision resnet50 and inception_v3 is traced on the
meta device (ingest.trace_units) -- no GPU, no weights.  Checked:
* the traced graphs are branchy (residual joins, Inception towers, the
  auxiliary classifier's second sink) and valid (validate_dag);
* tracing is deterministic: the DAG document equals the committed fixture;
* this package's planner on that DAG equals the REFERENCE planner's plan
  (tests/golden/ingested.json.gz, made by make_ingest_golden.py) bit for bit,
  and the enforced order carries real control edges (a pure chain has none).
"""

from __future__ import annotations

import gzip
import json
from functools import lru_cache
from pathlib import Path

import pytest

torch = pytest.importorskip("torch")
torchvision = pytest.importorskip("torchvision")

from paper_2004_14020_b200.dag import dag_from_json, dag_to_json, validate_dag  # noqa: E402
from paper_2004_14020_b200.ingest import build_dag, synthetic_durations, trace_units  # noqa: E402
from paper_2004_14020_b200.pipeline import run_pipeline  # noqa: E402

from test_plan_parity import _compare, as_json, make_config  # noqa: E402

GOLDEN = Path(__file__).resolve().parent / "golden" / "ingested.json.gz"


@lru_cache(maxsize=None)
def golden() -> list:
    with gzip.open(GOLDEN, "rt", encoding="utf-8") as fh:
        return json.load(fh)


@lru_cache(maxsize=None)
def traced(model: str):
    size = 299 if model == "inception_v3" else 224
    with torch.device("meta"):
        kw = {"aux_logits": True, "init_weights": False} if model == "inception_v3" else {}
        m = getattr(torchvision.models, model)(**kw)
    m.train()
    return trace_units(m, (torch.empty(2, 3, size, size, device="meta"),))


@pytest.mark.parametrize("model,units,sinks", [("resnet50", 107, 1), ("inception_v3", 194, 2)])
def test_traced_graph_is_branchy_and_valid(model, units, sinks):
    g = traced(model)
    assert len(g.names) == units
    assert sum(1 for c in g.consumers() if not c) == sinks
    joins = sum(1 for ins in g.inputs if len(ins) > 1)
    forks = sum(1 for c in g.consumers() if len(c) > 1)
    assert joins > 0 and forks > 0, "a real model's graph has joins and forks"
    dag = build_dag(g, *synthetic_durations(g))
    rep = validate_dag(dag)
    assert rep.ok, rep.errors
    assert sum(len(ps) for ps in g.params) == len(dag.params) == {"resnet50": 161, "inception_v3": 292}[model]


def test_traced_dag_matches_fixture():
    for model in ("resnet50", "inception_v3"):
        g = traced(model)
        doc = dag_to_json(build_dag(g, *synthetic_durations(g)))
        want = next(c["dag"] for c in golden() if c["model"] == model)
        assert doc == want, f"{model}: traced DAG differs from the committed fixture"


@pytest.mark.parametrize("idx", range(6))
def test_planner_matches_reference_on_ingested_dag(idx):
    case = golden()[idx]
    art = run_pipeline(dag_from_json(case["dag"]), make_config(case["config"]))
    got = as_json(art)
    _compare(got, case["artifacts"], f"{case['model']} p={case['config']['workers']}")
    assert len(got["control_edges"]) > 0, "branchy graph: enforce_order must add control edges"
