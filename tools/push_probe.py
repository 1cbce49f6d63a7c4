"""Bidirectional NVLink: both GPUs pull (read peer) or push (write peer) at
once, and mixed; per-direction GB/s.  Uses the diagnostic streaming copy."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib  # noqa: E402

NB = 256 << 20


def main():
    _lib.check(_lib.lib.ftar_peer_enable(0, 1))
    _lib.check(_lib.lib.ftar_peer_enable(1, 0))
    loc = {d: torch.randn(NB // 4, device=f"cuda:{d}").view(torch.uint8) for d in (0, 1)}
    rem = {d: torch.empty(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)}
    st = {d: torch.cuda.Stream(device=d) for d in (0, 1)}

    def go(kind, ctas, reps=6):
        def launch(d):
            o = 1 - d
            if kind == "pull":   # c (local) = b (remote); a = local dummy read
                c, a, b = rem[d], rem[d], loc[o]
            else:                # push: c (remote) = b (local)
                c, a, b = rem[o], loc[d], loc[d]
            _lib.check(_lib.lib.ftar_probe_pattern(c.data_ptr(), a.data_ptr(), b.data_ptr(), NB // 4, 1, 0, 8,
                                                   ctas, d, st[d].cuda_stream))
        for d in (0, 1):
            launch(d)
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        ev = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in (0, 1)}
        for d in (0, 1):
            with torch.cuda.device(d):
                ev[d][0].record(st[d])
        for _ in range(reps):
            for d in (0, 1):
                launch(d)
        for d in (0, 1):
            with torch.cuda.device(d):
                ev[d][1].record(st[d])
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        t = max(ev[d][0].elapsed_time(ev[d][1]) for d in (0, 1)) / reps / 1e3
        return NB / t / 1e9

    for kind in ("pull", "push"):
        for ctas in (32, 64, 128):
            print(json.dumps({"bidir": kind, "ctas": ctas, "GBps_per_direction": round(go(kind, ctas), 1)}), flush=True)


if __name__ == "__main__":
    main()
