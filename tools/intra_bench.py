"""Intra-replica reduce-scatter / all-gather throughput
vs NCCL on the same tensors.  One process per GPU (torchrun); rank 0 prints
one JSON line per (op, dtype, size).

    python -m torch.distributed.run --nproc-per-node 4 tools/intra_bench.py

busbw (NCCL convention): RS = (total * in_bytes / t) * (n-1)/n;
AG = (total * 4 / t) * (n-1)/n.  Inputs live in the registered pool
(zero-copy); queued 3 deep; 20 warm-up + 50 timed calls, CUDA events, max
over ranks.
"""

import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200.fabric import StoreFabric  # noqa: E402
from paper_2602_00277_b200.intra import IntraRank, segment_bounds  # noqa: E402


def timed(fn, iters, dev, drain=None):
    st = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(iters):
        fn()
    if drain is not None:
        drain()
    e1.record(st)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item() / 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes-mib", default="4,16,64,256")
    ap.add_argument("--dtypes", default="f32,bf16")
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    rank, n = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    store = dist.PrefixStore("intra-bench", dist.distributed_c10d._get_default_store())
    sizes = [int(s) << 20 for s in args.sizes_mib.split(",")]
    emax = max(sizes) // 2  # elements of the largest bf16 vector
    ir = IntraRank(rank, n, StoreFabric(store), device=dev, max_bytes=max(sizes),
                   pool_bytes=max(sizes) + emax * 4 // n + (8 << 20))
    vec = ir.alloc(max(sizes) // 4, torch.float32)
    vec.normal_()
    shard_buf = ir.alloc(emax // n + 64, torch.float32)
    full = torch.empty(emax, device=dev)
    for dname in args.dtypes.split(","):
        dt = torch.float32 if dname == "f32" else torch.bfloat16
        esz = 4 if dname == "f32" else 2
        for nb in sizes:
            total = nb // esz
            v = vec.view(torch.bfloat16)[:total] if dt == torch.bfloat16 else vec[:total]
            bounds = segment_bounds(total, n)
            ln = bounds[rank][1]
            shard = shard_buf[:ln]
            out_full = full[:total] if total <= emax else torch.empty(total, device=dev)
            from collections import deque
            pend = deque()

            def queued(fn):
                def step():
                    pend.append(fn())
                    while len(pend) >= 3:
                        pend.popleft().wait()
                return step

            def drain():
                while pend:
                    pend.popleft().wait()

            rs_step = queued(lambda: ir.reduce_scatter_async(v, bounds, out=shard))
            ag_step = queued(lambda: ir.all_gather_async(shard, bounds, total, out=out_full))
            for _ in range(20):
                rs_step()
            drain()
            t_rs = timed(lambda: rs_step(), args.iters, dev, drain)
            for _ in range(5):
                ag_step()
            drain()
            t_ag = timed(lambda: ag_step(), args.iters, dev, drain)
            # NCCL on the same tensors (equal shards: pad to a multiple of n)
            tn = total - total % n
            nv = v[:tn].contiguous()
            ns = torch.empty(tn // n, device=dev, dtype=dt)
            for _ in range(5):
                dist.reduce_scatter_tensor(ns, nv)
            t_nrs = timed(lambda: dist.reduce_scatter_tensor(ns, nv), args.iters, dev)
            nsf = torch.empty(tn // n, device=dev)
            nfull = torch.empty(tn, device=dev)
            for _ in range(5):
                dist.all_gather_into_tensor(nfull, nsf)
            t_nag = timed(lambda: dist.all_gather_into_tensor(nfull, nsf), args.iters, dev)
            f = (n - 1) / n
            if rank == 0:
                print(json.dumps({
                    "n": n, "dtype": dname, "bytes": nb,
                    "rs_us": round(t_rs * 1e6, 1), "rs_busbw": round(total * esz / t_rs * f / 1e9, 1),
                    "nccl_rs_us": round(t_nrs * 1e6, 1), "nccl_rs_busbw": round(tn * esz / t_nrs * f / 1e9, 1),
                    "ag_us": round(t_ag * 1e6, 1), "ag_busbw": round(total * 4 / t_ag * f / 1e9, 1),
                    "nccl_ag_us": round(t_nag * 1e6, 1), "nccl_ag_busbw": round(tn * 4 / t_nag * f / 1e9, 1),
                }), flush=True)
    ir.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
