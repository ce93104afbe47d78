"""Persisted plan formats as executor input.

The reference's `optimize` command (osim/cli.py:177-216) writes the planner's
artifacts as JSON: dag_enforced.json, control_edges.json,
activation_order.json, batch_plan.json (BatchPlan.to_json, batching.py:41-56)
and transfer_schedule.json (TransferSchedule.to_json, transfer.py:59-73).
`write_plan` writes the same five files from a pipeline run, adding the one
field the reference leaves out -- each group's collective depth -- and
`load_exec_plan` lowers a batch plan + transfer schedule pair (this package's
or the reference CLI's own output) into the executor's rank-invariant
ExecPlan:

* buckets and member order come from batch_plan.json groups;
* launch order and placement from transfer_schedule.json (already sorted by
  (begin_us, group_id), transfer.py:193; the times are rounded by round_us,
  costmodel.py:69-71, which changes no order);
* depth from the group's "depth" field when present, else the depth policy
  over the file's threshold_bytes (pipeline.py:83-86): adaptive_depth, or a
  fixed depth clamped to [1, MAX_DEPTH].
"""

from __future__ import annotations

import json
from pathlib import Path

from .collective import MAX_DEPTH, Pattern, adaptive_depth
from .costmodel import round_us
from .dag import dag_to_json
from .executor import ExecPlan, lower_groups

PLAN_FILES = ("dag_enforced.json", "control_edges.json", "activation_order.json", "batch_plan.json",
              "transfer_schedule.json")


def batch_plan_json(art) -> dict:
    """BatchPlan.to_json plus each group's depth (the field the reference omits)."""
    doc = art.batch_plan.to_json()
    for g in doc["groups"]:
        g["depth"] = int(art.depths[g["group_id"]])
    return doc


def write_plan(art, out_dir: str | Path) -> list[Path]:
    """The reference `optimize` command's five artifacts (cli.py:199-212) for a
    pipeline run, batch_plan.json carrying depths."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    docs = {
        "dag_enforced.json": dag_to_json(art.enforced_dag),
        "control_edges.json": [{"from_op": e.from_op, "to_op": e.to_op} for e in art.control_edges],
        "activation_order.json": {"param_ids": list(art.order.param_ids),
                                  "cumulative_cost_us": [round_us(c) for c in art.order.cumulative_cost_us]},
        "batch_plan.json": batch_plan_json(art),
        "transfer_schedule.json": art.transfer_schedule.to_json(),
    }
    paths = []
    for name in PLAN_FILES:
        path = out / name
        path.write_text(json.dumps(docs[name], indent=2) + "\n", encoding="utf-8")
        paths.append(path)
    return paths


def group_depth(group: dict, threshold: int, depth: int | None) -> int:
    """Depth of one persisted group: its "depth" field, else the policy
    (fixed `depth` clamped like pipeline.bucket_depth, or adaptive_depth)."""
    if "depth" in group:
        return int(group["depth"])
    if depth is not None:
        return min(MAX_DEPTH, max(1, int(depth)))
    return adaptive_depth(int(group["total_bytes"]), int(threshold))


def load_exec_plan(plan_dir: str | Path | None = None, numels: dict[str, int] | None = None, world: int = 2,
                   pattern: Pattern | str = Pattern.SHUFFLE, *, depth: int | None = None,
                   batch_plan: dict | None = None, transfer_schedule: dict | None = None,
                   max_ctas: int | None = None) -> ExecPlan:
    """ExecPlan from persisted batch_plan.json + transfer_schedule.json (read
    from `plan_dir`, or passed as parsed documents).  `numels`: param id ->
    element count (fp32 gradients); `depth`: the fixed depth the plan was made
    with, for files without depths (None = adaptive, the reference default)."""
    if numels is None:
        raise ValueError("numels (param id -> element count) is required")
    if batch_plan is None or transfer_schedule is None:
        if plan_dir is None:
            raise ValueError("pass plan_dir or both documents")
        d = Path(plan_dir)
        batch_plan = batch_plan or json.loads((d / "batch_plan.json").read_text(encoding="utf-8"))
        transfer_schedule = transfer_schedule or json.loads((d / "transfer_schedule.json").read_text(encoding="utf-8"))
    groups = {g["group_id"]: g for g in batch_plan["groups"]}
    launch = transfer_schedule["transfers"]
    if len(launch) != len(groups) or {t["group_id"] for t in launch} != set(groups):
        raise ValueError("transfer schedule and batch plan disagree")
    # file order IS the launch order: written sorted by the unrounded
    # (begin_us, group_id); re-sorting rounded times could swap near-ties
    thr = int(batch_plan["threshold_bytes"])
    rows = []
    for t in launch:
        g = groups[t["group_id"]]
        rows.append((g["group_id"], tuple(g["param_ids"]), int(g["total_bytes"]), group_depth(g, thr, depth),
                     t["placement"], float(g["ready_time_us"])))
    return lower_groups(rows, numels, world, Pattern(pattern), max_ctas)
