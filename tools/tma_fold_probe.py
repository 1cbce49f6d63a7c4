"""Per-CTA throughput of the two-shot kernel's reduce-scatter paths on ONE GPU:
members emulated as CTA groups (every load local HBM), bulk-copy (TMA) path vs
register path, across CTA budgets.  Separates pipeline issues from NVLink.

    python tools/tma_fold_probe.py [--n 2,4] [--ctas 8,16,32,64] [--mib 256]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib, ftar  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="2,4")
    ap.add_argument("--ctas", default="8,16,32,64")
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    elems = args.mib * (1 << 20) // 4
    for n in [int(x) for x in args.n.split(",")]:
        ring = ftar.LocalRing(n, device=dev, max_bucket_bytes=elems * 4, protocol=True)
        bufs = [torch.randn(elems, device=dev) for _ in range(n)]
        outs = [torch.empty(elems, device=dev) for _ in range(n)]
        for ctas in [int(x) for x in args.ctas.split(",")]:
            if ctas * n > 148:
                continue
            rec = {"n": n, "ctas_per_member": ctas, "mib": args.mib}
            for tma in ("1", "0"):
                os.environ["FTAR_TMA"] = tma
                _lib.lib.ftar_set_tuning(0, ctas)
                ring.all_reduce(bufs, outs=outs, scale=1.0 / n)
                torch.cuda.synchronize()
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                for _ in range(args.reps):
                    ring.all_reduce(bufs, outs=outs, scale=1.0 / n)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e) / args.reps
                # every member reads its slice of every input and writes its slice
                # to every output: n*E*(4+4) bytes of HBM traffic per call
                rec["tma" if tma == "1" else "ldg"] = {"ms": round(ms, 4),
                                                       "hbm_GBps": round(n * elems * 8 / ms / 1e6, 1)}
            if os.environ.get("FTAR_DIAG", "0") in ("3", "4"):
                import ctypes as C
                os.environ["FTAR_TMA"] = "1"
                ring.all_reduce(bufs, outs=outs, scale=1.0 / n)
                t = (C.c_uint64 * 512)()
                _lib.lib.ftar_debug_trace(ring.groups[0].ctx, t, 512)
                t = list(t)
                base = t[256]
                rec["trace_us"] = {k: [round((x - base) / 1e3, 2) if x else None for x in t[o:o + 24]]
                                   for k, o in (("refill_start", 0), ("refill_issued", 128), ("landed_w0", 256),
                                                ("landed_w1", 384))}
            print(json.dumps(rec), flush=True)
        _lib.lib.ftar_set_tuning(0, 0)
        ring.close()


if __name__ == "__main__":
    main()
