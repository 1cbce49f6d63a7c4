"""Single-GPU target for ncu: the two-shot protocol kernel (allreduce_kernel)
with n emulated members as CTA groups of one cooperative launch, or the
in-process one-shot kernel.  usage: ncu_target.py [protocol|oneshot] [n] [MiB | KiB"k"] [dtype]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import ftar  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "protocol"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
size = sys.argv[3] if len(sys.argv) > 3 else "256"  # MiB, or KiB with a trailing "k"
dt = torch.bfloat16 if (len(sys.argv) > 4 and sys.argv[4] == "bf16") else torch.float32
elems = (int(size[:-1]) << 10 if size.endswith("k") else int(size) << 20) // 4
dev = torch.device("cuda", 0)
ring = ftar.LocalRing(n, device=dev, max_bucket_bytes=elems * 4, protocol=(mode == "protocol"))
bufs = [torch.randn(elems, device=dev).to(dt) for _ in range(n)]
outs = [torch.empty(elems, device=dev) for _ in range(n)]
for _ in range(4):
    ring.all_reduce(bufs, outs=outs, scale=1.0 / n)
torch.cuda.synchronize()
ring.close()
print("ok")
