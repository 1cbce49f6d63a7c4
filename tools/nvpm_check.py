"""Validate the CUPTI PM-sampling NVLink counters (tools/nvlink_pm.cpp)
against known traffic: GPU 0 pulls 4 x 512 MiB from GPU 1 with the bulk-copy
probe; GPU 0 RX / GPU 1 TX must be ~2 GiB of user data (+ packet overhead)."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import NvlinkPM  # noqa: E402
from paper_2602_00277_b200 import _lib  # noqa: E402

NB = 512 << 20
_lib.check(_lib.lib.ftar_peer_enable(0, 1))
src = torch.randn(NB // 4, device="cuda:1").view(torch.uint8)
dst = torch.empty(NB, dtype=torch.uint8, device="cuda:0")
pms = [NvlinkPM(0), NvlinkPM(1)]
print(json.dumps({"pm_errors": [p.err for p in pms]}), flush=True)
for reps in (1, 4):
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    for p in pms:
        p.start()
    for _ in range(reps):
        with torch.cuda.device(0):
            _lib.check(_lib.lib.ftar_probe_bulk(dst.data_ptr(), src.data_ptr(), NB, 32, 32768, 4,
                                                torch.cuda.current_stream(0).cuda_stream))
    torch.cuda.synchronize(0)
    out = [p.stop() for p in pms]
    print(json.dumps({"pulled_bytes": reps * NB, "gpu0": out[0], "gpu1": out[1],
                      "errors": [p.err for p in pms]}), flush=True)
for p in pms:
    p.close()
