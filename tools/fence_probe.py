"""How long do gpu/sys fences take after a CTA streamed remote (NVLink) loads?"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib  # noqa: E402

N = 32 << 20


def main():
    _lib.check(_lib.lib.ftar_peer_enable(0, 1))
    _lib.check(_lib.lib.ftar_peer_enable(1, 0))
    bufs = {d: [torch.randn(N, device=f"cuda:{d}") for _ in range(3)] for d in (0, 1)}
    streams = {d: torch.cuda.Stream(device=d) for d in (0, 1)}
    for kind in (0, 1, 2):
        for ctas in (32, 64):
            for remote in (True, False):
                stamps = {d: torch.zeros(ctas * 4, dtype=torch.int64, device=f"cuda:{d}") for d in (0, 1)}
                for rep in range(3):
                    for d in (0, 1):
                        a, c, _ = bufs[d]
                        b = bufs[1 - d][2] if remote else bufs[d][2]
                        _lib.check(_lib.lib.ftar_probe_fence(c.data_ptr(), a.data_ptr(), b.data_ptr(), N, kind, ctas,
                                                             stamps[d].data_ptr(), d, streams[d].cuda_stream))
                    torch.cuda.synchronize(0)
                    torch.cuda.synchronize(1)
                st = stamps[0].view(ctas, 4).cpu().double()
                t0 = st[:, 0].min()
                res = {"kind": ["no_allocate", "default", "nc"][kind], "ctas": ctas, "remote": remote,
                       "loop_end_us": [round(float(st[:, 0].min() - t0) / 1e3, 1), round(float(st[:, 0].max() - t0) / 1e3, 1)],
                       "sync_us_max": round(float((st[:, 1] - st[:, 0]).max()) / 1e3, 1),
                       "gpu_fence_us": [round(float((st[:, 2] - st[:, 1]).median()) / 1e3, 1), round(float((st[:, 2] - st[:, 1]).max()) / 1e3, 1)],
                       "sys_fence_us": [round(float((st[:, 3] - st[:, 2]).median()) / 1e3, 1), round(float((st[:, 3] - st[:, 2]).max()) / 1e3, 1)]}
                print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
