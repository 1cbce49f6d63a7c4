"""Sweep the two-shot kernel's launch shape on all visible GPUs from one
process (DeviceRing).  Env knobs are read by libftar_b200 at launch:
FTAR_CTAS, FTAR_RS_LAYOUT.  One JSON line per configuration."""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib, ftar  # noqa: E402

MIB = 1 << 20


def bench(ring, bufs, outs, reps=10):
    ring.all_reduce(bufs, outs=outs, scale=0.5)
    for d in ring.devices:
        torch.cuda.synchronize(d)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in ring.devices]
    for (s, _), d in zip(ev, ring.devices):
        with torch.cuda.device(d):
            s.record()
    for _ in range(reps):
        ring.all_reduce(bufs, outs=outs, scale=0.5)
    for (_, e), d in zip(ev, ring.devices):
        with torch.cuda.device(d):
            e.record()
    for d in ring.devices:
        torch.cuda.synchronize(d)
    return max(s.elapsed_time(e) for s, e in ev) / reps / 1e3


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else torch.cuda.device_count()
    mib = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    ctas_list = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "32,48,64").split(",")]
    dtypes = (sys.argv[4] if len(sys.argv) > 4 else "f32,bf16").split(",")
    layouts = [int(x) for x in (sys.argv[5] if len(sys.argv) > 5 else "0,1").split(",")]
    elems = mib * MIB // 4
    ring = ftar.DeviceRing(list(range(n)), max_bucket_bytes=elems * 4)
    for dt in dtypes:
        tdt = torch.bfloat16 if dt == "bf16" else torch.float32
        ib = 2 if dt == "bf16" else 4
        bufs = [torch.randn(elems, device=d).to(tdt) for d in ring.devices]
        outs = [torch.empty(elems, device=d) for d in ring.devices]
        for layout, ctas in itertools.product(layouts, ctas_list):
            os.environ["FTAR_CTAS"] = str(ctas)
            os.environ["FTAR_RS_LAYOUT"] = str(layout)
            _lib.lib.ftar_set_tuning(ctas, 0)
            t = bench(ring, bufs, outs)
            busbw = elems * ib / t * 2 * (n - 1) / n / 1e9
            nv = (n - 1) / n * elems * (ib + 4) / t / 1e9
            import ctypes as C
            t0 = (C.c_uint64 * 6)()
            _lib.lib.ftar_phase_times(ring.ctxs[0], t0, 6)
            rs = (C.c_uint64 * 260)()
            ag = (C.c_uint64 * 260)()
            _lib.lib.ftar_debug_cta_times(ring.ctxs[0], rs, ag, 260)
            base = t0[1]
            rsl = sorted((rs[i] - base) / 1e3 for i in range(ctas))
            agl = sorted((ag[i] - base) / 1e3 for i in range(ctas))
            cta = {"rs_end_us": [round(rsl[0], 1), round(rsl[len(rsl) // 2], 1), round(rsl[-1], 1)],
                   "ag_end_us": [round(agl[0], 1), round(agl[len(agl) // 2], 1), round(agl[-1], 1)],
                   "fence_us": [round((rs[257] - rs[256]) / 1e3, 1), round((rs[259] - rs[258]) / 1e3, 1)],
                   "rs_pub_us": round((t0[2] - base) / 1e3, 1)}
            print(json.dumps({"n": n, "MiB": mib, "dtype": dt, "layout": layout, "ctas": ctas, "cta": cta,
                              "ms": round(t * 1e3, 4), "busbw": round(busbw, 1), "nvlink_GBps": round(nv, 1),
                              "phases": ring.phase_us(0)}), flush=True)
    ring.close()


if __name__ == "__main__":
    main()
