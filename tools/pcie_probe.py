"""PCIe ceiling for the e2e path: 256 MiB pinned H2D alone, D2H alone and
both at once (separate streams), on one GPU and on every GPU at the same time
(one thread per GPU).  Prints one JSON line per case.

    python tools/pcie_probe.py [--gpus N] [--mib 256]
"""

import argparse
import json
import threading

import torch


def run(dev, mib, mode, iters, out, barrier):
    torch.cuda.set_device(dev)
    n = mib << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device=dev)
    d_b = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def once():
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    once()
    barrier.wait()
    ts = []
    for _ in range(iters):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize(dev)
        e[0].record(torch.cuda.current_stream(dev))
        once()
        e[1].record(torch.cuda.current_stream(dev))
        torch.cuda.synchronize(dev)
        ts.append(e[0].elapsed_time(e[1]) / 1e3)
    t = min(ts)
    out[dev] = round(n / t / 1e9, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=torch.cuda.device_count())
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    for ngpu in sorted({1, args.gpus}):
        for mode in ("h2d", "d2h", "both"):
            out = {}
            barrier = threading.Barrier(ngpu)
            th = [threading.Thread(target=run, args=(d, args.mib, mode, args.iters, out, barrier)) for d in range(ngpu)]
            for t in th:
                t.start()
            for t in th:
                t.join()
            print(json.dumps({"gpus_at_once": ngpu, "mode": mode, "GBps_per_direction_per_gpu": out}), flush=True)


if __name__ == "__main__":
    main()
