"""Does NVLink pull bandwidth depend on data content / stream?  Same kernel
(probe_copy) on never-written, zero-filled and random buffers."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib  # noqa: E402

NB = 256 << 20


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize(0)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize(0)
    return s.elapsed_time(e) / reps / 1e3


def main():
    _lib.check(_lib.lib.ftar_peer_enable(0, 1))
    _lib.check(_lib.lib.ftar_peer_enable(1, 0))
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream(0).cuda_stream
    dst = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
    srcs = {"empty": torch.empty(NB, dtype=torch.uint8, device="cuda:1"),
            "zeros": torch.zeros(NB, dtype=torch.uint8, device="cuda:1"),
            "ones": torch.full((NB,), 7, dtype=torch.uint8, device="cuda:1"),
            "randn": torch.randn(NB // 4, device="cuda:1").view(torch.uint8),
            "randint": torch.randint(0, 255, (NB,), dtype=torch.uint8, device="cuda:1")}
    torch.cuda.synchronize(1)
    for name, src in srcs.items():
        for ctas in (32, 64, 128):
            t = timed(lambda: _lib.check(_lib.lib.ftar_probe_copy(dst.data_ptr(), src.data_ptr(), NB, ctas, st)))
            tp = timed(lambda: _lib.check(_lib.lib.ftar_probe_pattern(dst.data_ptr(), dst.data_ptr(), src.data_ptr(),
                                                                      NB // 4, 1, 0, 8, ctas, 0, st)))
            print(json.dumps({"src": name, "ctas": ctas, "probe_copy_GBps": round(NB / t / 1e9, 1),
                              "probe_pattern_copy_GBps": round(NB / tp / 1e9, 1)}), flush=True)
    t = timed(lambda: dst.copy_(srcs["randn"]))
    print(json.dumps({"src": "randn", "copy_engine_GBps": round(NB / t / 1e9, 1)}))


if __name__ == "__main__":
    main()
