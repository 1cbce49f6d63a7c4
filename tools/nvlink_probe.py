"""Characterise NVLink between cuda:0 and cuda:1 from one process:
copy-engine peer copy, SM pull (remote src) and SM push (remote dst) at
several CTA counts.  Prints one JSON line per measurement."""
import json
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib  # noqa: E402

NB = 512 << 20


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps / 1e3


def main():
    _lib.check(_lib.lib.ftar_peer_enable(0, 1))
    _lib.check(_lib.lib.ftar_peer_enable(1, 0))
    a0 = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
    a1 = torch.empty(NB, dtype=torch.uint8, device="cuda:1")
    b0 = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream(0).cuda_stream
    t = timed(lambda: a0.copy_(a1))
    print(json.dumps({"what": "copy engine peer->local", "GBps": NB / t / 1e9}))
    t = timed(lambda: b0.copy_(a0))
    print(json.dumps({"what": "copy engine local->local (r+w)", "GBps": 2 * NB / t / 1e9}))
    for ctas in (8, 16, 32, 64, 96, 148, 296):
        t = timed(lambda: _lib.check(_lib.lib.ftar_probe_copy(a0.data_ptr(), a1.data_ptr(), NB, ctas, st)))
        t2 = timed(lambda: _lib.check(_lib.lib.ftar_probe_copy(a1.data_ptr(), a0.data_ptr(), NB, ctas, st)))
        t3 = timed(lambda: _lib.check(_lib.lib.ftar_probe_copy(b0.data_ptr(), a0.data_ptr(), NB, ctas, st)))
        print(json.dumps({"ctas": ctas, "pull_GBps": round(NB / t / 1e9, 1), "push_GBps": round(NB / t2 / 1e9, 1),
                          "local_copy_GBps(r+w)": round(2 * NB / t3 / 1e9, 1)}))


if __name__ == "__main__":
    main()
