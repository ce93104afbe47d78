"""Golden plans for DAGs INGESTED from real models.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ingest_golden.py
For torchvision resnet50 and inception_v3 (aux logits on) the unit dataflow
is traced on the meta device (paper_2004_14020_b200.ingest.trace_units),
turned into a DataflowDag with the survey's synthetic durations, serialised
with the reference's JSON wire format, and planned by the REFERENCE planner
(imported read-only from /root/reference/pkg/src).  Writes
tests/golden/ingested.json.gz: the DAG documents and the reference's plans.
tests/test_ingest_parity.py re-traces, checks the DAG is identical, and checks
this package's planner against the reference's plans bit for bit -- including
the non-empty control edges of the branchy graphs.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))

import make_golden as G  # noqa: E402  (reference imports + artifacts_to_json)
from overlapsim.dag import dag_from_json  # noqa: E402
from overlapsim.pipeline import run_pipeline  # noqa: E402

from paper_2004_14020_b200.dag import dag_to_json  # noqa: E402

CASES = [(8, G.NVLINK), (4, G.CLOUD), (2, G.NVLINK)]


def traced_dag_json(model: str) -> dict:
    import torch
    import torchvision

    from paper_2004_14020_b200.ingest import build_dag, synthetic_durations, trace_units

    size = 299 if model == "inception_v3" else 224
    with torch.device("meta"):
        kw = {"aux_logits": True, "init_weights": False} if model == "inception_v3" else {}
        m = getattr(torchvision.models, model)(**kw)
    m.train()
    g = trace_units(m, (torch.empty(2, 3, size, size, device="meta"),))
    return dag_to_json(build_dag(g, *synthetic_durations(g)))


def main() -> None:
    out = []
    for model in ("resnet50", "inception_v3"):
        doc = traced_dag_json(model)
        ref_dag = dag_from_json(doc)
        for p, net in CASES:
            art = run_pipeline(ref_dag, G.config(p, net))
            out.append({"model": model, "dag": doc, "config": G.cfg_json(p, net, "shuffle", None),
                        "artifacts": G.artifacts_to_json(art)})
            print(model, p, net, len(art.batch_plan.groups), "groups", len(art.control_edges), "control edges")
    with gzip.open(HERE / "ingested.json.gz", "wt", encoding="utf-8") as fh:
        json.dump(out, fh)


if __name__ == "__main__":
    main()
