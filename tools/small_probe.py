"""Where does a small-bucket call (the push one-shot, <= 1 MiB) spend its
device time?  Runs the diagnostic library (FTAR_LIB_VARIANT=diag), whose
small kernel stamps %globaltimer at each step of CTA 0:

    0 start  1 zombie+epoch checks  2 griddepcontrol.wait  3 pushes issued
    4 flags raised  5 all peers' flags seen  6 folded  7 re-checked
    8 arrived  9 done (last CTA)

and prints the mean step durations (us) per rank, queued (depth 3) and
blocking.  One process per GPU:

    python -m torch.distributed.run --nproc-per-node N tools/small_probe.py [--kib 1,64,1024]
"""
import argparse
import ctypes as C
import json
import os
import sys

os.environ["FTAR_LIB_VARIANT"] = "diag"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_00277_b200 import _lib, ftar  # noqa: E402
from paper_2602_00277_b200.fabric import StoreFabric  # noqa: E402

STEPS = ["checks", "pdl_wait", "push", "flags", "peers_in", "fold", "recheck", "arrive", "commit",
         "load_peer_slot", "load_my_input", "fold_thread0", "fold_again (FTAR_DIAG=5)"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kib", default="1,64,1024")
    ap.add_argument("--iters", type=int, default=50)
    args = ap.parse_args()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rank, n = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rank)))
    torch.cuda.set_device(dev)
    sizes = [int(k) << 10 for k in args.kib.split(",")]
    emax = max(sizes) // 4
    g = ftar.RingGroup(rank, 0, StoreFabric(dist.PrefixStore("sp", dist.distributed_c10d._get_default_store())),
                       device=dev, max_bucket_bytes=emax * 4, pool_bytes=emax * 8 + (1 << 20))
    g.reconfig({r: ftar.PeerAddress(r) for r in range(n)}, 1, deadline_s=30)
    buf, out = g.alloc_bucket(emax), g.alloc_bucket(emax)
    buf.normal_()
    cfg = ftar.PipelineConfig()
    tr = (C.c_uint64 * 16)()
    for nb in sizes:
        e = nb // 4
        b, o = buf[:e], out[:e]
        for _ in range(10):
            ftar.ftar_all_reduce(g, b, 0, cfg, out=o)
        acc = [0.0] * 13
        for _ in range(args.iters):
            ftar.ftar_all_reduce(g, b, 0, cfg, out=o)
            _lib.lib.ftar_debug_trace(g.ctx, tr, 16)
            for i in range(9):
                acc[i] += (tr[i + 1] - tr[i]) / 1e3
            acc[9] += tr[10] / 1e3  # one load of a peer-written slot
            acc[10] += tr[11] / 1e3  # one load of my input
            acc[11] += (tr[12] - tr[5]) / 1e3  # step 5 -> fold_tiles returned (thread 0)
            acc[12] += (tr[13] - tr[12]) / 1e3 if os.environ.get("FTAR_DIAG") == "5" else 0.0  # the fold again
        blocking = [round(a / args.iters, 2) for a in acc]
        rows = [None] * n
        dist.all_gather_object(rows, blocking)
        if rank == 0:
            print(json.dumps({"n": n, "bytes": nb, "steps": STEPS, "blocking_us_per_rank": rows,
                              "total_us_per_rank": [round(sum(r[:9]), 2) for r in rows]}), flush=True)
    g.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
