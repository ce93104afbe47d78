"""K1 / K4 standalone on the resnet50 gradient set (161 separate tensors):
a few caramel_pack / caramel_unpack launches, for ncu."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2004_14020_b200 import gradsets  # noqa: E402

dev = torch.device("cuda", 0)
r = bench.pack_unpack_bw(torch, gradsets.gradient_set("resnet50"), dev, 6524.0, reps=3)
print(r)
