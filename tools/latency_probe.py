"""Where does a small all-reduce spend its time?  (2 GPUs, one process per GPU)
Prints host-side microseconds per phase of the Python call and device phases."""
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
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, n = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    store = dist.PrefixStore("lat", dist.distributed_c10d._get_default_store())
    g = ftar.RingGroup(rank, 0, StoreFabric(store), device=dev, max_bucket_bytes=1 << 20, pool_bytes=4 << 20)
    g.reconfig({r: ftar.PeerAddress(r) for r in range(n)}, 1, deadline_s=30)
    buf = g.alloc_bucket(256)
    out = g.alloc_bucket(256)
    cfg = ftar.PipelineConfig()
    res = {}
    for mode in ("blocking", "async3"):
        for _ in range(50):
            ftar.ftar_all_reduce(g, buf, 0, cfg, out=out)
        dist.barrier()
        k = 2000
        t0 = time.perf_counter()
        pend = []
        t_call = 0.0
        for _ in range(k):
            a = time.perf_counter()
            if mode == "blocking":
                ftar.ftar_all_reduce(g, buf, 0, cfg, out=out)
            else:
                pend.append(ftar.ftar_all_reduce_async(g, buf, 0, cfg, out=out))
                if len(pend) >= 3:
                    pend.pop(0).wait()
            t_call += time.perf_counter() - a
        while pend:
            pend.pop(0).wait()
        res[mode] = round((time.perf_counter() - t0) / k * 1e6, 2)
    # raw C launch + wait without Python wrapper
    st = torch.cuda.current_stream(dev).cuda_stream
    dist.barrier()
    k = 2000
    t0 = time.perf_counter()
    for _ in range(k):
        _lib.lib.ftar_allreduce_launch(g.ctx, buf.data_ptr(), 0, out.data_ptr(), 256, 8 << 20, 4, 1.0, 0, st)
        _lib.lib.ftar_wait(g.ctx, 5.0, None)
    res["raw_ctypes_blocking"] = round((time.perf_counter() - t0) / k * 1e6, 2)
    t = (C.c_uint64 * 6)()
    _lib.lib.ftar_phase_times(g.ctx, t, 6)
    res["device_phases_us"] = [round((t[i + 1] - t[i]) / 1e3, 2) for i in range(4)]
    res["device_total_us"] = round((t[4] - t[0]) / 1e3, 2)
    # python overhead of the wrapper (no GPU work): time _check_buffers + stream lookup
    a = time.perf_counter()
    for _ in range(k):
        ftar._check_buffers(buf, out)
        ftar._stream_ptr(dev)
    res["py_checks_us"] = round((time.perf_counter() - a) / k * 1e6, 2)
    if rank == 0:
        print(json.dumps(res), flush=True)
    g.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
