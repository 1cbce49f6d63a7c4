"""Config 3: FTAR bucket-size sweep vs NCCL all_reduce (rank 0 prints JSON lines).

    python -m torch.distributed.run --nproc-per-node N tools/sweep.py [--max-mib 1024]

Per cell: FTAR (push one-shot <= 1 MiB, else two-shot NVLink; fused x f32(1/n), fp32 out, buckets in
the registered pool, queue depth 3) and NCCL all_reduce on a same-size
tensor of the same input dtype (NCCL reduces in the input dtype; FTAR always
accumulates and outputs fp32).  busbw = (E*in_bytes/t) * 2(n-1)/n; nvlink =
actual FTAR ingress per GPU (n-1)/n*E*(in_bytes+4) / t.  CUDA events, max
over ranks.
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
    ap.add_argument("--max-mib", type=int, default=1024)
    ap.add_argument("--dtypes", default="bf16,f32")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--min-steps", type=int, default=5, help="timed calls per cell at the largest sizes")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2602_00277_b200 import ftar
    from paper_2602_00277_b200.fabric import StoreFabric

    sys.path.insert(0, ROOT)
    from bench import _StdoutToStderr

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, n = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    store = dist.PrefixStore("sweep", dist.distributed_c10d._get_default_store())
    maxb = args.max_mib << 20
    group = ftar.RingGroup(rank, 0, StoreFabric(store), device=dev, max_bucket_bytes=maxb,
                           pool_bytes=maxb + 2 * maxb + 8192)
    group.reconfig({r: ftar.PeerAddress(r) for r in range(n)}, 1, deadline_s=60)
    pg = None
    if not args.no_nccl:
        with _StdoutToStderr():
            pg = dist.new_group(backend="nccl")
            t = torch.ones(16, device=dev)
            dist.all_reduce(t, group=pg)
            torch.cuda.synchronize()

    def mx(v):
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def timeit(fn, k, drain=None):
        for _ in range(3):
            fn()
        if drain:
            drain()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(k):
            fn()
        if drain:
            drain()
        e.record()
        torch.cuda.synchronize()
        return mx(s.elapsed_time(e) / k / 1e3)

    sizes = []
    b = 1024
    while b <= maxb:
        sizes.append(b)
        b *= 4
    if sizes[-1] != maxb:
        sizes.append(maxb)
    for dt in args.dtypes.split(","):
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        ib = 2 if dt == "bf16" else 4
        for nbytes in sizes:
            elems = nbytes // ib
            group.reset_pool()
            buf = group.alloc_bucket(elems, tdt)
            buf.copy_(torch.randn(elems, device=dev).to(tdt))
            out = group.alloc_bucket(elems, torch.float32)
            k = max(args.min_steps, min(200, int(2e9 // max(nbytes, 1) // 8)))
            pend = []

            def step():
                pend.append(ftar.ftar_all_reduce_async(group, buf, 0, out=out, scale=1.0 / n))
                while len(pend) >= 3:
                    pend.pop(0).wait()

            def drain():
                while pend:
                    pend.pop(0).wait()

            t = timeit(step, k, drain)
            row = {"n": n, "dtype": dt, "bytes": nbytes, "elems": elems, "ftar_us": round(t * 1e6, 2),
                   "ftar_busbw": round(nbytes / t * 2 * (n - 1) / n / 1e9, 2),
                   "ftar_nvlink_GBps": round((n - 1) / n * elems * (ib + 4) / t / 1e9, 2)}
            if pg is not None:
                x = torch.randn(elems, device=dev).to(tdt)
                tn = timeit(lambda: dist.all_reduce(x, group=pg), k)
                row.update({"nccl_us": round(tn * 1e6, 2),
                            "nccl_busbw": round(nbytes / tn * 2 * (n - 1) / n / 1e9, 2)})
                del x
            if rank == 0:
                print(json.dumps(row), flush=True)
            del buf, out
    group.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
