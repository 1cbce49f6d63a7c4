"""GB/s-vs-CTA curves of the two-shot all-reduce over NVLink: the bulk-copy
(TMA) reduce-scatter vs the register path, per bucket size and dtype, in the
production topology (one process per GPU, registered buckets, out of place
with the push all-gather, x f32(1/n) fused, queue depth 3).  CUDA events, max
over ranks; one JSON line per cell on rank 0.

    python -m torch.distributed.run --nproc-per-node N tools/tune_tma.py \\
        [--mib 4,16,64,256,1024] [--dtypes f32,bf16] [--tma-ctas 8,12,16,24,32,48] [--ldg-ctas 32,64,128]
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
    ap.add_argument("--mib", default="4,16,64,256,1024", help="bucket MiB per replica (input dtype)")
    ap.add_argument("--dtypes", default="f32,bf16")
    ap.add_argument("--tma-ctas", default="8,12,16,24,32,48")
    ap.add_argument("--ldg-ctas", default="32,64,128")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ag", default="push", help="comma list of all-gather modes: push (into registered outs), "
                                                  "pull (FTAR_NO_PUSH=1: members pull the reduced slices)")
    ap.add_argument("--auto", action="store_true", help="add a cell with the library's default policy")
    ap.add_argument("--env", action="append", default=[], metavar="NAME=v1,v2",
                    help="sweep an environment knob over every cell (repeatable; e.g. FTAR_PDL_EARLY=0,1)")
    ap.add_argument("--repeat", type=int, default=1, help="run every cell this many times (interleaved)")
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
    sizes = [int(x) for x in args.mib.split(",")]
    maxb = max(sizes) << 20
    fabric = StoreFabric(dist.PrefixStore("tune", dist.distributed_c10d._get_default_store()))
    group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=maxb, pool_bytes=maxb * 3 + 8192)
    group.reconfig({r: ftar.PeerAddress(r) for r in range(n)}, 1, deadline_s=60)
    cfg = ftar.PipelineConfig()
    stream = torch.cuda.current_stream(dev)

    def timed(buf, out, steps):
        pend = []

        def step():
            pend.append(ftar.ftar_all_reduce_async(group, buf, 0, cfg, out=out, scale=1.0 / n))
            while len(pend) >= 3:
                pend.pop(0).wait()

        for _ in range(3):
            step()
        while pend:
            pend.pop(0).wait()
        dist.barrier()
        step()  # device-side barrier opening the window
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(steps):
            step()
        while pend:
            pend.pop(0).wait()
        e.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / steps / 1e3], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    for dt in args.dtypes.split(","):
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        ib = 2 if dt == "bf16" else 4
        for mib in sizes:
            elems = (mib << 20) // ib
            group.reset_pool()
            buf = group.alloc_bucket(elems, tdt)
            buf.copy_(torch.randn(elems, device=dev).to(tdt))
            out = group.alloc_bucket(elems, torch.float32)
            steps = max(5, min(args.steps * 8, int(args.steps * 256 / max(mib, 1))))
            cells = [("tma", c) for c in args.tma_ctas.split(",") if c] + \
                    [("ldg", c) for c in args.ldg_ctas.split(",") if c] + ([("auto", "0")] if args.auto else [])
            combos = [{}]
            for spec in args.env:
                name, vals = spec.split("=", 1)
                combos = [{**c, name: v} for c in combos for v in vals.split(",")]
            cells = [(*cell, e) for _ in range(args.repeat) for cell in cells for e in combos]
            for ag in args.ag.split(","):
                os.environ["FTAR_NO_PUSH"] = "1" if ag == "pull" else "0"
                for path, c, env in cells:
                    os.environ.update(env)
                    os.environ["FTAR_TMA"] = "0" if path == "ldg" else "1"
                    _lib.lib.ftar_set_tuning(int(c), 0)
                    t = timed(buf, out, steps)
                    if rank == 0:
                        busbw = elems * ib / t * 2 * (n - 1) / n / 1e9
                        ingress = (n - 1) / n * elems * (ib + 4) / t / 1e9
                        print(json.dumps({"n": n, "dtype": dt, "MiB": mib, "path": path, "ag": ag, "ctas": int(c),
                                          "env": env,
                                          "us": round(t * 1e6, 2), "busbw": round(busbw, 1),
                                          "nvlink_ingress_GBps": round(ingress, 1)}), flush=True)
            os.environ["FTAR_NO_PUSH"] = "0"
    _lib.lib.ftar_set_tuning(0, 0)
    group.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
