"""Long bit-exact stress of the fused aggregation step on N GPUs (one process
per GPU, torch.distributed.run).  ResNet-50's gradient set and plan; every step
every rank writes fresh integer-valued gradients g_r(step, i) = ((7 i + 13 step
+ 5 r) mod 17) - 8 into the zero-copy buckets and runs Aggregator.step() (the
one-launch fused two-shot + SGD).  With lr = 2^-10 and p a power of two every
value is exact in fp32, so each rank checks its parameters against a closed-form
running expectation (computed on the device from the same formula for every
rank) -- bit for bit -- every `--check` steps, and all ranks' parameter
checksums against each other.  Prints one JSON line per check and a summary."""
import argparse, json, os, sys, time
from pathlib import Path
import torch
import torch.distributed as dist
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--check", type=int, default=500)
    ap.add_argument("--model", default="resnet50")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    NVLINK_MODEL = (10.0, 1.0 / 460e3)  # SURVEY §8a "NVLink-ish" network model
    from paper_2004_14020_b200 import gradsets
    from paper_2004_14020_b200.collective import Pattern, ReduceModel
    from paper_2004_14020_b200.costmodel import NetworkModel
    from paper_2004_14020_b200.executor import Aggregator, lower
    from paper_2004_14020_b200.pipeline import run_pipeline
    from paper_2004_14020_b200.sim import SimConfig

    tensors = gradsets.gradient_set(args.model)
    art = run_pipeline(gradsets.layered_chain_dag(args.model),
                       SimConfig(workers=max(2, world), network=NetworkModel(*NVLINK_MODEL),
                                 reduce=ReduceModel(400.0, 10.0)))
    ids = [gradsets.param_id(i, len(tensors)) for i in range(len(tensors))]
    plan = lower(art, {pid: t.numel for pid, t in zip(ids, tensors)}, world, Pattern.SHUFFLE)
    params = {pid: torch.zeros(t.shape, device=dev) for pid, t in zip(ids, tensors)}
    lr = 2.0 ** -10
    agg = Aggregator(plan, params, rank=rank, lr=lr, epilogue="sgd", grads="bucket")
    flat_idx = {pid: torch.arange(params[pid].numel(), device=dev, dtype=torch.int64) for pid in ids}
    expect = {pid: torch.zeros(params[pid].numel(), device=dev) for pid in ids}
    t0 = time.time()
    fails = 0
    for step in range(1, args.steps + 1):
        for pid in ids:
            base = 7 * flat_idx[pid] + 13 * step
            params[pid].grad.view(-1).copy_(((base + 5 * rank) % 17 - 8).float())
            tot = sum(((base + 5 * r) % 17 - 8) for r in range(world)).float()
            expect[pid].sub_(tot * (lr / world))
        agg.step()
        if step % args.check == 0 or step == args.steps:
            torch.cuda.synchronize()
            agg.status()
            bad = sum(int(not torch.equal(params[pid].view(-1), expect[pid])) for pid in ids)
            ck = torch.tensor([float(sum(params[pid].double().sum().item() for pid in ids))], device=dev,
                              dtype=torch.float64)
            allck = [torch.empty_like(ck) for _ in range(world)]
            dist.all_gather(allck, ck)
            same = all(float(a.item()) == float(ck.item()) for a in allck)
            fails += bad + (0 if same else 1)
            if rank == 0:
                print(json.dumps({"step": step, "tensors_mismatched": bad, "replicas_identical": same,
                                  "checksum": float(ck.item()), "elapsed_s": round(time.time() - t0, 1)}),
                      flush=True)
    t = torch.tensor([fails], device=dev)
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"summary": "stress", "world": world, "steps": args.steps, "buckets": len(plan.buckets),
                          "elements": plan.total_numel, "failures": int(t.item()),
                          "kernel": agg.step_kernel()}), flush=True)
    agg.close()
    dist.destroy_process_group()
    return 0 if int(t.item()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
