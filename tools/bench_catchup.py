"""Config 4: non-blocking catch-up (one JSON line per pull budget on rank 0).

    python -m torch.distributed.run --nproc-per-node N tools/bench_catchup.py [--gib 8]

Ranks 0..N-2 are healthy replicas stepping: back-to-back FTAR all-reduces of
256 MiB fp32 buckets over NVLink (ring of N-1).  Rank N-1 is the recovering
replica: it pulls the donor's (rank 0, pick_donor) retention-1 snapshot of
params + momentum (GiB total, fp32) over NVLink with the catch-up kernel on a
low-priority side stream (checkpoint.start_fetch), with a CTA budget.
Reported: pull ms/GB alone and under load, and the healthy replicas' step time
without / with the concurrent pull (the "does not stall the healthy replicas"
criterion).  Times: CUDA events, max over healthy ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=8.0, help="params+momentum GiB")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--bucket-mib", type=int, default=256)
    ap.add_argument("--ctas", type=str, default="8,16,32")
    ap.add_argument("--stripe", action="store_true", help="stripe the pull over every healthy donor")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2602_00277_b200 import checkpoint as ck
    from paper_2602_00277_b200 import ftar
    from paper_2602_00277_b200.fabric import StoreFabric

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    store = dist.PrefixStore("catchup", dist.distributed_c10d._get_default_store())
    fabric = StoreFabric(store)
    rec = world - 1
    healthy = list(range(world - 1))
    donor = ck.pick_donor(healthy, rec, rank=0)
    half = int(args.gib * (1 << 30) / 2) // 4  # fp32 elements per tensor
    nbytes = 2 * half * 4
    elems = args.bucket_mib * (1 << 20) // 4

    snap = ck.SnapshotStore(capacity_bytes=nbytes, device=dev, fabric=fabric, rank=0, replica_id=rank)
    if rank != rec:  # every healthy replica holds the same retention-1 snapshot
        g = torch.Generator(device=dev).manual_seed(5)
        p = torch.randn(half, device=dev, generator=g)
        m = torch.randn(half, device=dev, generator=g)
        snap.capture(41, p, m)
        torch.cuda.synchronize()
        del p, m
    group = None
    if rank != rec and len(healthy) > 1:
        group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=elems * 4,
                               pool_bytes=2 * elems * 4 + 4096)
        group.reconfig({r: ftar.PeerAddress(r) for r in healthy}, 1, deadline_s=60)
        buf = group.alloc_bucket(elems)
        buf.normal_()
        out = group.alloc_bucket(elems)
    elif rank != rec:
        buf = torch.randn(elems, device=dev)
        out = torch.empty_like(buf)
    if rank == rec:
        p_out = torch.empty(half, device=dev)
        m_out = torch.empty(half, device=dev)
    dist.barrier()

    def healthy_steps(k):
        """k FTAR steps; returns mean ms/step (CUDA events)."""
        cfg = ftar.PipelineConfig()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        pend = []
        for _ in range(k):
            if group is not None:
                pend.append(ftar.ftar_all_reduce_async(group, buf, 0, cfg, out=out, scale=1.0 / len(healthy)))
                while len(pend) >= 3:
                    pend.pop(0).wait()
            else:
                out.copy_(buf).mul_(1.0)
        while pend:
            pend.pop(0).wait()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / k

    def pull(ctas, donors=None):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        side = ck.catchup_stream(dev)
        t0 = time.perf_counter()
        s.record(side)
        h = ck.start_fetch(snap, donor if donors is None else donors, 41, 0, p_out, m_out, timeout_s=30, ctas=ctas)
        e.record(side)
        h.wait()
        torch.cuda.synchronize()
        return s.elapsed_time(e), (time.perf_counter() - t0) * 1e3

    def mx(v):
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    if rank != rec:
        healthy_steps(5)
    if rank == rec:  # warm-up: lazy peer mapping of the donors' snapshot arenas
        pull(16)
        if args.stripe and len(healthy) > 1:
            pull(16, healthy)
    dist.barrier()
    base = mx(healthy_steps(args.steps) if rank != rec else 0.0)
    results = []
    stripe = args.stripe and len(healthy) > 1
    for ctas in [int(c) for c in args.ctas.split(",")]:
        dist.barrier()
        dl = healthy if stripe else None
        alone = pull(ctas, dl)[0] if rank == rec else 0.0
        alone = mx(alone)
        dist.barrier()
        if rank == rec:
            loaded_ms, wall = pull(ctas, dl)
            step = 0.0
        else:
            step = healthy_steps(args.steps)
            loaded_ms = 0.0
        loaded_ms, step = mx(loaded_ms), mx(step)
        ok = True
        if rank == rec:
            g = torch.Generator(device=dev).manual_seed(5)
            ok = bool(torch.equal(p_out, torch.randn(half, device=dev, generator=g)))
        ok = mx(0.0 if ok else 1.0) == 0.0
        gb = nbytes / 1e9
        results.append({"metric": "catch-up ms/GB", "gib": args.gib, "bytes": nbytes, "ctas": ctas,
                        "pull_ms_alone": round(alone, 3), "ms_per_GB_alone": round(alone / gb, 3),
                        "GBps_alone": round(gb / alone * 1e3, 1),
                        "pull_ms_under_load": round(loaded_ms, 3), "ms_per_GB_under_load": round(loaded_ms / gb, 3),
                        "healthy_step_ms_baseline": round(base, 4), "healthy_step_ms_during_pull": round(step, 4),
                        "healthy_replicas": len(healthy), "bucket_mib": args.bucket_mib,
                        "pull_bit_exact": ok, "n_gpus": world,
                        "donors": healthy if stripe else [donor]})
    if rank == 0:
        for r in results:
            print(json.dumps(r), flush=True)
    if group is not None:
        group.close()
    snap.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
