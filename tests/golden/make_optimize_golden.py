"""Golden persisted plans from the REFERENCE CLI (`overlapsim optimize`).

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_optimize_golden.py
For each case it writes the DAG (gradsets.layered_chain_dag) and model JSON
to a temp dir, invokes the reference's own `optimize` command (cli.py:177-216)
through click's CliRunner, and keeps the two files the executor consumes --
batch_plan.json (batching.py:41-56) and transfer_schedule.json
(transfer.py:59-73) -- under tests/golden/optimize/<case>/, plus the case's
arguments in case.json.  tests/test_planio.py lowers them with
planio.load_exec_plan and checks the result against this package's own
planner run on the same DAG.
"""

from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))

from click.testing import CliRunner  # noqa: E402
from overlapsim.cli import main as ref_cli  # noqa: E402  (the reference)

from paper_2004_14020_b200 import gradsets  # noqa: E402
from paper_2004_14020_b200.dag import dag_to_json  # noqa: E402

CASES = {
    # name: (model, workers, pattern, (latency_us, per_byte_us), fixed depth or None)
    "resnet50_p4_nvlink": ("resnet50", 4, "shuffle", (10.0, 1.0 / 460e3), None),
    "alexnet_p8_cloud_depth3": ("alexnet", 8, "ring", (1000.0, 0.001), 3),
    "vgg16_p2_nvlink": ("vgg16", 2, "shuffle", (10.0, 1.0 / 460e3), None),
}


def main() -> None:
    out_root = HERE / "optimize"
    runner = CliRunner()
    for name, (model, workers, pattern, net, depth) in CASES.items():
        with tempfile.TemporaryDirectory() as td:
            td = Path(td)
            (td / "dag.json").write_text(json.dumps(dag_to_json(gradsets.layered_chain_dag(model))))
            (td / "model.json").write_text(json.dumps({"latency_us": net[0], "per_byte_us": net[1]}))
            args = ["optimize", str(td / "dag.json"), "--model", str(td / "model.json"), "--workers", str(workers),
                    "--pattern", pattern, "--out", str(td / "out")]
            if depth is not None:
                args += ["--depth", str(depth)]
            res = runner.invoke(ref_cli, args, catch_exceptions=False)
            if res.exit_code != 0:
                raise SystemExit(f"{name}: reference optimize failed: {res.output}")
            dst = out_root / name
            dst.mkdir(parents=True, exist_ok=True)
            for f in ("batch_plan.json", "transfer_schedule.json"):
                shutil.copy(td / "out" / f, dst / f)
            (dst / "case.json").write_text(json.dumps(
                {"model": model, "workers": workers, "pattern": pattern, "network": list(net), "depth": depth,
                 "reference_stdout": res.output.strip()}, indent=2) + "\n")
        print(f"{name}: {res.output.strip()}")


if __name__ == "__main__":
    main()
