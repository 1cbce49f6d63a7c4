"""Config 5's hot call in isolation: the all-reduce with the fused
normalisation + SGD-momentum step (ftar_all_reduce_sgd) on B buckets of bf16
gradients, one process per GPU, against the plain bf16 -> fp32 all-reduce of
the same buckets.  Per bucket ms (CUDA events, max over ranks) for each
FTAR_CTAS_SGD value given (buckets queued, as ftar_all_reduce_sgd_async).

    python -m torch.distributed.run --nproc-per-node N tools/sgd_bench.py [--mib 256] [--buckets 8] [--ctas 64,128]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256, help="bf16 gradient MiB per bucket")
    ap.add_argument("--buckets", type=int, default=8)
    ap.add_argument("--ctas", default="64,128")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2602_00277_b200 import _lib, ftar
    from paper_2602_00277_b200.fabric import StoreFabric

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, n = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    elems = (args.mib << 20) // 2
    fabric = StoreFabric(dist.PrefixStore("sgdb", dist.distributed_c10d._get_default_store()))
    group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=elems * 2,
                           pool_bytes=args.buckets * elems * 6 + 8192)
    group.reconfig({r: ftar.PeerAddress(r) for r in range(n)}, 1, deadline_s=60)
    grads = [group.alloc_bucket(elems, torch.bfloat16) for _ in range(args.buckets)]
    gouts = [group.alloc_bucket(elems, torch.float32) for _ in range(args.buckets)]
    for g in grads:
        g.copy_(torch.randn(elems, device=dev))
    params = [torch.randn(elems, device=dev) for _ in range(args.buckets)]
    moms = [torch.randn(elems, device=dev) for _ in range(args.buckets)]
    pouts = [torch.empty(elems, device=dev) for _ in range(args.buckets)]
    mouts = [torch.empty(elems, device=dev) for _ in range(args.buckets)]
    cfg = ftar.PipelineConfig()
    stream = torch.cuda.current_stream(dev)
    scale = 1.0 / n

    def plain():
        pend = [ftar.ftar_all_reduce_async(group, g, 0, cfg, out=o, scale=scale) for g, o in zip(grads, gouts)]
        for p in pend:
            p.wait()

    def sgd(with_grad_out):
        pend = [ftar.ftar_all_reduce_sgd_async(group, grads[i], 0, cfg, params=params[i], momentum=moms[i], lr=0.01,
                                               beta=0.9, scale=scale, params_out=pouts[i], momentum_out=mouts[i],
                                               grad_out=gouts[i] if with_grad_out else None)
                for i in range(args.buckets)]
        for p in pend:
            p.wait()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        dist.barrier()
        best = 1e9
        for _ in range(args.reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            fn()
            e.record(stream)
            torch.cuda.synchronize()
            t = torch.tensor([s.elapsed_time(e)], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            best = min(best, t.item())
        return best / args.buckets

    for c in args.ctas.split(","):
        os.environ["FTAR_CTAS_SGD"] = c
        row = {"n": n, "mib_bf16": args.mib, "buckets": args.buckets, "ctas": int(c),
               "plain_ms": round(timed(plain), 4), "sgd_ms": round(timed(lambda: sgd(False)), 4),
               "sgd_grad_out_ms": round(timed(lambda: sgd(True)), 4)}
        if rank == 0:
            print(json.dumps(row), flush=True)
    _lib.lib.ftar_set_tuning(0, 0)
    group.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
