"""Where does a mid-size all-reduce spend its device time?  One process per
GPU (torchrun).  For each bucket size: queued per-call time (CUDA events, the
sweep's method) and the mean device phases of blocking calls, read from the
kernel's %globaltimer stamps (ftar_phase_times):

    entry   t1-t0  kernel start -> every member's entry record seen
    rs      t2-t1  my slice folded (and pushed to every peer in push mode)
    wait    t3-t2  every peer's slice arrived (ag_in flags / rs_done)
    tail    t4-t3  all-gather pull (pull mode) + completion fence

    python -m torch.distributed.run --nproc-per-node 4 tools/phase_probe.py [--dtype f32]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib, ftar  # noqa: E402
from paper_2602_00277_b200.fabric import StoreFabric  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--sizes-mib", default="1,2,4,8,16,32,64,256")
    ap.add_argument("--sizes-kib", default=None, help="overrides --sizes-mib")
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, n = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    sizes = ([int(s) << 10 for s in args.sizes_kib.split(",")] if args.sizes_kib
             else [int(s) << 20 for s in args.sizes_mib.split(",")])
    dt = torch.float32 if args.dtype == "f32" else torch.bfloat16
    esz = 4 if dt == torch.float32 else 2
    emax = max(sizes) // esz
    store = dist.PrefixStore("phase", dist.distributed_c10d._get_default_store())
    g = ftar.RingGroup(rank, 0, StoreFabric(store), device=dev, max_bucket_bytes=emax * 4,
                       pool_bytes=emax * esz + emax * 4 + (1 << 20))
    g.reconfig({r: ftar.PeerAddress(r) for r in range(n)}, 1, deadline_s=30)
    buf = g.alloc_bucket(emax, dt)
    out = g.alloc_bucket(emax, torch.float32)
    buf.normal_()
    cfg = ftar.PipelineConfig()
    st = torch.cuda.current_stream(dev)
    off = C.c_int64()
    _lib.lib.ftar_probe_clock(dev.index, 200, C.byref(off))  # this GPU's timer -> host CLOCK_MONOTONIC
    for nb in sizes:
        e = nb // esz
        b, o = buf[:e], out[:e]
        for _ in range(10):
            ftar.ftar_all_reduce(g, b, 0, cfg, out=o)
        # queued per-call time (one untimed call first: a device-side barrier,
        # so host-side skew out of dist.barrier() stays out of the window)
        dist.barrier()
        ftar.ftar_all_reduce(g, b, 0, cfg, out=o)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(st)
        pend = []
        h0 = time.perf_counter()
        for _ in range(args.iters):
            pend.append(ftar.ftar_all_reduce_async(g, b, 0, cfg, out=o))
            if len(pend) >= 3:
                pend.pop(0).wait()
        while pend:
            pend.pop(0).wait()
        ev1.record(st)
        host_call = (time.perf_counter() - h0) * 1e6 / args.iters  # host time per call incl. its wait
        torch.cuda.synchronize()
        per_call = ev0.elapsed_time(ev1) * 1e3 / args.iters
        t = (C.c_uint64 * 6)()
        _lib.lib.ftar_phase_times(g.ctx, t, 6)  # the last queued call
        q_ph = [round((t[i + 1] - t[i]) / 1e3, 2) for i in range(4)]
        q_t0 = int(t[0])
        q_host = [int(t[i]) + off.value for i in range(5)]  # stamps on the shared host clock
        # device phases of blocking calls
        acc = [0.0] * 4
        k = 20
        t = (C.c_uint64 * 6)()
        for _ in range(k):
            ftar.ftar_all_reduce(g, b, 0, cfg, out=o)
            _lib.lib.ftar_phase_times(g.ctx, t, 6)
            for i in range(4):
                acc[i] += (t[i + 1] - t[i]) / 1e3
        ph = [round(a / k, 2) for a in acc]
        # breakdown of the last blocking call, relative to the fan-out (t1):
        # per-CTA end of the reduce-scatter fold, the RS sys fence, t2
        rs_end, ag_end = (C.c_uint64 * 260)(), (C.c_uint64 * 256)()
        _lib.lib.ftar_debug_cta_times(g.ctx, rs_end, ag_end, 260)
        t1 = t[1]
        ends = sorted((rs_end[i] - t1) / 1e3 for i in range(256) if rs_end[i] >= t[0])
        det = {"ctas": len(ends),
               "rs_end_us_min_med_max": [round(ends[0], 2), round(ends[len(ends) // 2], 2), round(ends[-1], 2)]
               if ends else None,
               "rs_fence_start_us": round((rs_end[256] - t1) / 1e3, 2),
               "rs_fence_us": round((rs_end[257] - rs_end[256]) / 1e3, 2),
               "t2_us": round((t[2] - t1) / 1e3, 2)}
        slice_e, ctas, thr = C.c_uint64(), C.c_int(), C.c_int()
        _lib.lib.ftar_geometry(e, n, C.byref(slice_e), C.byref(ctas), C.byref(thr))
        rows = [None] * n
        dist.all_gather_object(rows, {"rank": rank, "phases_us": ph, "per_call_us": round(per_call, 2),
                                      "host_per_call_us": round(host_call, 2),
                                      "queued_phases_us": q_ph, "queued_t0": q_t0, "detail": det,
                                      "queued_host_ns": q_host})
        if rank == 0:
            busbw = nb / (per_call * 1e-6) * 2 * (n - 1) / n / 1e9
            print(json.dumps({"n": n, "dtype": args.dtype, "bytes": nb, "per_call_us": round(per_call, 2),
                              "host_per_call_us": [r["host_per_call_us"] for r in rows],
                              "busbw": round(busbw, 1), "slice_elems": slice_e.value,
                              "phases_entry_rs_wait_tail_us": [r["phases_us"] for r in rows],
                              "queued_phases_us": [r["queued_phases_us"] for r in rows],
                              "detail_rank0": rows[0]["detail"],
                              # the last queued call on one clock (host CLOCK_MONOTONIC via
                              # ftar_probe_clock, ~1-2 us): [start, published, all peers in,
                              # -, end] per rank, us after the earliest start
                              "timeline_us": [[round((v - min(x["queued_host_ns"][0] for x in rows)) / 1e3, 2)
                                               for v in r["queued_host_ns"]] for r in rows]}), flush=True)
    g.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
