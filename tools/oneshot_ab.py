"""A/B of the in-process one-shot (the N=1 bench kernel) across input data and
kernel form: register (FTAR_LOCAL_BULK=0) vs bulk-copy fed, on device-random,
host-random (numpy, as bench.py) and zero buckets.  One JSON line per cell.

    python tools/oneshot_ab.py [--mib 256] [--replicas 4] [--steps 20]
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
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--replicas", type=int, default=4)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--forms", default="reg,bulk")
    ap.add_argument("--data", default="device,host,zeros")
    ap.add_argument("--bulk-ctas", default="", help="comma list of FTAR_LOCAL_BULK_CTAS for the bulk form")
    ap.add_argument("--harness", default="plain", help="comma list: plain | events (per-launch CUDA events, as "
                                                       "bench.timed_loop) | clocks (bench.ClockSampler running) | both")
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2602_00277_b200 import ftar
    dev = torch.device("cuda", 0)
    n, elems = args.replicas, (args.mib << 20) // 4
    ring = ftar.LocalRing(n, device=dev, max_bucket_bytes=elems * 4)
    cfg = ftar.PipelineConfig()
    outs = [torch.empty(elems, device=dev) for _ in range(n)]
    stream = torch.cuda.current_stream(dev)
    for data in args.data.split(","):
        if data == "device":
            g = torch.Generator(device=dev).manual_seed(0)
            bufs = [torch.randn(elems, device=dev, generator=g) for _ in range(n)]
        elif data == "host":
            bufs = [torch.from_numpy(np.random.default_rng(r).standard_normal(elems, dtype=np.float32)).to(dev)
                    for r in range(n)]
        else:
            bufs = [torch.zeros(elems, device=dev) for _ in range(n)]
        for form in args.forms.split(","):
            os.environ["FTAR_LOCAL_BULK"] = "1" if form == "bulk" else "0"
            for c in (args.bulk_ctas.split(",") if form == "bulk" and args.bulk_ctas else [""]):
                if c:
                    os.environ["FTAR_LOCAL_BULK_CTAS"] = c
                else:
                    os.environ.pop("FTAR_LOCAL_BULK_CTAS", None)
                for harness in args.harness.split(","):
                    for _ in range(3):
                        ring.all_reduce(bufs, cfg, outs=outs, scale=1.0 / n)
                    torch.cuda.synchronize()
                    sampler = None
                    if harness in ("clocks", "both"):
                        import bench
                        sampler = bench.ClockSampler(0).__enter__()
                    pend = []
                    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                          for _ in range(args.steps)]
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record(stream)
                    for i in range(args.steps):
                        if harness in ("events", "both"):
                            ev[i][0].record(stream)
                        pend.append(ring.launch(bufs, cfg, outs=outs, scale=1.0 / n))
                        while len(pend) >= 3:
                            ring.wait(pend.pop(0), cfg)
                        if harness in ("events", "both"):
                            ev[i][1].record(stream)
                    while pend:
                        ring.wait(pend.pop(0), cfg)
                    e.record(stream)
                    torch.cuda.synchronize()
                    if sampler is not None:
                        sampler.__exit__(None, None, None)
                    ms = s.elapsed_time(e) / args.steps
                    print(json.dumps({"data": data, "form": form, "ctas": c or "default", "harness": harness,
                                      "ms": round(ms, 4), "hbm_gbs": round(n * elems * 8 / ms / 1e6, 1)}), flush=True)
        del bufs
    ring.close()


if __name__ == "__main__":
    main()
