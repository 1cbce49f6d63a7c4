"""NVLink access-pattern probe between cuda:0 and cuda:1 in one process.
uni: only GPU0 runs (reads GPU1); bi: both GPUs run the mirror pattern at
once (as in the real all-reduce).  One JSON line per configuration."""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib  # noqa: E402

N = 32 << 20  # fp32 elements per buffer (128 MiB)


def main():
    _lib.check(_lib.lib.ftar_peer_enable(0, 1))
    _lib.check(_lib.lib.ftar_peer_enable(1, 0))
    bufs = {}
    for d in (0, 1):
        bufs[d] = [torch.randn(N, device=f"cuda:{d}") for _ in range(3)]
    streams = {d: torch.cuda.Stream(device=d) for d in (0, 1)}

    def launch(d, mode, layout, unroll, ctas):
        a, c, _ = bufs[d]
        b = bufs[1 - d][2]
        _lib.check(_lib.lib.ftar_probe_pattern(c.data_ptr(), a.data_ptr(), b.data_ptr(), N, mode, layout, unroll,
                                               ctas, d, streams[d].cuda_stream))

    def run(devs, mode, layout, unroll, ctas, reps=5):
        for d in devs:
            launch(d, mode, layout, unroll, ctas)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        ev = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in devs}
        for d in devs:
            with torch.cuda.device(d):
                ev[d][0].record(streams[d])
        for _ in range(reps):
            for d in devs:
                launch(d, mode, layout, unroll, ctas)
        for d in devs:
            with torch.cuda.device(d):
                ev[d][1].record(streams[d])
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        return max(ev[d][0].elapsed_time(ev[d][1]) for d in devs) / reps / 1e3

    for mode, layout, unroll, ctas, devs in itertools.product((0, 1), (0, 1), (4, 8), (32, 64, 128),
                                                              ((0, 1),)):
        t = run(devs, mode, layout, unroll, ctas)
        print(json.dumps({"mode": ["a+b", "copy b", "loads only", "local"][mode], "layout": ["stride", "span"][layout],
                          "unroll": unroll, "ctas": ctas, "dir": "bi" if len(devs) == 2 else "uni",
                          "remote_GBps": round(N * 4 / t / 1e9, 1)}), flush=True)
    for layout, unroll, ctas in itertools.product((0, 1), (4, 8), (32, 128)):
        t = run((0,), 3, layout, unroll, ctas)
        print(json.dumps({"mode": "local", "layout": ["stride", "span"][layout], "unroll": unroll, "ctas": ctas,
                          "local_rw_GBps": round(3 * N * 4 / t / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
