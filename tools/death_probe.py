"""Member death mid-collective (2 GPUs): rank 1 launches its all-reduce on a
big bucket and exits with os._exit while its kernel is running; rank 0 must
get a Recoverable error (not a CUDA fault) and its CUDA context must stay
usable afterwards.  Prints one JSON line from rank 0."""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import errors, ftar  # noqa: E402
from paper_2602_00277_b200.fabric import StoreFabric  # noqa: E402


def main():
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    from datetime import timedelta
    store = dist.TCPStore("127.0.0.1", int(os.environ["MASTER_PORT"]) + 7, world, rank == 0,
                          timeout=timedelta(seconds=60))
    fab = StoreFabric(dist.PrefixStore("death", store))
    e = 128 << 20  # 512 MiB fp32
    g = ftar.RingGroup(rank, 0, fab, device=dev, max_bucket_bytes=e * 4, pool_bytes=2 * e * 4 + 4096)
    g.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
    buf = g.alloc_bucket(e)
    buf.fill_(1.0)
    out = g.alloc_bucket(e)
    ftar.ftar_all_reduce(g, buf, 0, out=out)  # warm: both sides mapped
    torch.cuda.synchronize()
    store.set(f"ready{rank}", b"1")
    store.wait([f"ready{r}" for r in range(world)])
    cfg = ftar.PipelineConfig(per_chunk_timeout_s=1.0)
    if rank == 1:
        p = ftar.ftar_all_reduce_async(g, buf, 1, cfg, out=out)
        time.sleep(0.0002)
        os._exit(0)  # die with the kernel in flight and the arena still mapped by rank 0
    t0 = time.monotonic()
    res = {"survivor": rank}
    try:
        for i in range(3):  # the peer dies during one of these
            ftar.ftar_all_reduce(g, buf, 2 + i, cfg, out=out)
        res["outcome"] = "completed"
    except errors.FtdpError as exc:
        res["outcome"] = f"{type(exc).__name__}:{exc.reason}"
    except Exception as exc:  # noqa: BLE001
        res["outcome"] = f"OTHER:{exc!r}"
    res["seconds"] = round(time.monotonic() - t0, 3)
    try:
        x = torch.ones(1 << 20, device=dev)
        res["context_usable_after"] = float(x.sum().item()) == float(1 << 20)
        g.reconfig({0: ftar.PeerAddress(0)}, 2)
        y = torch.ones(1000, device=dev)
        ftar.ftar_all_reduce(g, y, 9, cfg)
        res["solo_ring_after"] = float(y.sum().item()) == 1000.0
    except Exception as exc:  # noqa: BLE001
        res["context_usable_after"] = f"FAULT:{exc!r}"[:200]
    print(json.dumps(res), flush=True)
    os._exit(0)


if __name__ == "__main__":
    main()
