"""Persistent checkpoint throughput: an 8 GiB params +
momentum snapshot (config 4's shard) streamed from the GPU to local storage
by SnapshotStore.persist, alone and while the GPU runs back-to-back 4-replica
256 MiB all-reduce steps (in-process ring).  One JSON line.

    python tools/persist_bench.py [--gib 8] [--dir /tmp/ftar_ckpt]
"""

import argparse
import json
import os
import shutil
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=8.0)
    ap.add_argument("--dir", default="/tmp/ftar_ckpt")
    args = ap.parse_args()
    import torch

    from paper_2602_00277_b200 import checkpoint as ck
    from paper_2602_00277_b200 import ftar
    dev = torch.device("cuda", 0)
    n = int(args.gib * (1 << 30)) // 8  # fp32 params + fp32 momentum
    p = torch.randn(n, device=dev)
    m = torch.randn(n, device=dev)
    store = ck.SnapshotStore(capacity_bytes=n * 8, device=dev)
    store.capture(1, p, m)
    shutil.rmtree(args.dir, ignore_errors=True)
    t0 = time.monotonic()
    store.persist(args.dir).wait()
    alone = time.monotonic() - t0
    size = os.path.getsize(ck.shard_path(args.dir, 1, 0))

    ring = ftar.LocalRing(4, device=dev, max_bucket_bytes=256 << 20)
    bufs = [torch.randn(64 << 20, device=dev) for _ in range(4)]
    outs = [torch.empty_like(b) for b in bufs]

    def steps(k):
        torch.cuda.synchronize()
        t = time.monotonic()
        for _ in range(k):
            ring.all_reduce(bufs, outs=outs, scale=0.25)
        torch.cuda.synchronize()
        return (time.monotonic() - t) / k

    steps(5)
    base = steps(20)
    store.capture(2, p, m)
    torch.cuda.synchronize()
    shutil.rmtree(args.dir, ignore_errors=True)
    box = {}
    t0 = time.monotonic()
    job = store.persist(args.dir)
    during = []

    def watch():
        job.wait()
        box["t"] = time.monotonic() - t0

    w = threading.Thread(target=watch)
    w.start()
    while w.is_alive():
        during.append(steps(5))
    w.join()
    shutil.rmtree(args.dir, ignore_errors=True)
    print(json.dumps({"metric": "persistent checkpoint from the GPU snapshot", "bytes": size,
                      "seconds_alone": round(alone, 3), "GBps_alone": round(size / alone / 1e9, 2),
                      "seconds_while_stepping": round(box["t"], 3), "GBps_while_stepping": round(size / box["t"] / 1e9, 2),
                      "step_ms_baseline": round(base * 1e3, 3),
                      "step_ms_during_persist": round(sorted(during)[len(during) // 2] * 1e3, 3) if during else None,
                      "target": args.dir}), flush=True)
    store.close()


if __name__ == "__main__":
    main()
