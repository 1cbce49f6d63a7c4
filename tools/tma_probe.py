"""NVLink copy bandwidth per CTA budget: register-staged LDG/STG copy
(ftar_probe_copy) vs the TMA bulk-copy pipeline (ftar_probe_bulk), pull
(read peer) and push (write peer), one direction or both GPUs at once.
Also checks that NVML's NVLink data counters (field values 138/139, KiB,
summed over links) see the bytes a run moved.  One process, 2 GPUs.

    python tools/tma_probe.py [--ctas 1,2,4,...] [--quick]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00277_b200 import _lib  # noqa: E402

NB = 512 << 20


class NvlinkCounters:
    """Per-GPU NVLink TX/RX data bytes from NVML field values (KiB counters,
    aggregated over links with scopeId = UINT_MAX)."""

    def __init__(self, devs):
        import pynvml as nv
        nv.nvmlInit()
        self.nv = nv
        self.h = {}
        for d in devs:
            pr = torch.cuda.get_device_properties(d)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self.h[d] = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())

    def read(self):
        nv = self.nv
        out = {}
        for d, h in self.h.items():
            vals = nv.nvmlDeviceGetFieldValues(h, [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF),
                                                   (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)])
            r = []
            for v in vals:
                if v.nvmlReturn != 0:
                    r.append(None)
                else:
                    r.append(int(v.value.ullVal) * 1024)
            out[d] = r
        return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctas", default="1,2,4,8,16,32,64,128,148")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    ctas_list = [int(x) for x in args.ctas.split(",")]
    _lib.check(_lib.lib.ftar_peer_enable(0, 1))
    _lib.check(_lib.lib.ftar_peer_enable(1, 0))
    loc = {d: torch.randn(NB // 4, device=f"cuda:{d}").view(torch.uint8) for d in (0, 1)}
    rem = {d: torch.empty(NB, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)}
    st = {d: torch.cuda.Stream(device=d) for d in (0, 1)}

    def go(engine, kind, ctas, bidir, tile=32768, stages=4, reps=4):
        devs = (0, 1) if bidir else (0,)

        def launch(d):
            o = 1 - d
            if kind == "pull":   # local dst <- remote src
                dst, src = rem[d], loc[o]
            else:                # remote dst <- local src
                dst, src = rem[o], loc[d]
            with torch.cuda.device(d):
                if engine == "ldg":
                    _lib.check(_lib.lib.ftar_probe_copy(dst.data_ptr(), src.data_ptr(), NB, ctas, st[d].cuda_stream))
                else:
                    _lib.check(_lib.lib.ftar_probe_bulk(dst.data_ptr(), src.data_ptr(), NB, ctas, tile, stages,
                                                        st[d].cuda_stream))
        for d in devs:
            launch(d)
        for d in (0, 1):
            torch.cuda.synchronize(d)
        ev = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in devs}
        for d in devs:
            with torch.cuda.device(d):
                ev[d][0].record(st[d])
        for _ in range(reps):
            for d in devs:
                launch(d)
        for d in devs:
            with torch.cuda.device(d):
                ev[d][1].record(st[d])
        for d in (0, 1):
            torch.cuda.synchronize(d)
        t = max(ev[d][0].elapsed_time(ev[d][1]) for d in devs) / reps / 1e3
        return round(NB / t / 1e9, 1)

    # correctness of the bulk path (pull and push)
    for kind in ("pull", "push"):
        rem[0].zero_(); rem[1].zero_()
        torch.cuda.synchronize(0); torch.cuda.synchronize(1)
        if kind == "pull":
            _lib.check(_lib.lib.ftar_probe_bulk(rem[0].data_ptr(), loc[1].data_ptr(), NB, 16, 32768, 4,
                                                st[0].cuda_stream))
            torch.cuda.synchronize(0)
            ok = torch.equal(rem[0].cpu(), loc[1].cpu())
        else:
            _lib.check(_lib.lib.ftar_probe_bulk(rem[1].data_ptr(), loc[0].data_ptr(), NB, 16, 32768, 4,
                                                st[0].cuda_stream))
            torch.cuda.synchronize(0)
            ok = torch.equal(rem[1].cpu(), loc[0].cpu())
        print(json.dumps({"check": kind, "bit_exact": ok}), flush=True)

    try:
        ctr = NvlinkCounters((0, 1))
        c0 = ctr.read()
        reps = 4
        bw = go("bulk", "pull", 64, True, reps=reps)
        c1 = ctr.read()
        moved = (reps + 1) * NB
        delta = {d: [(b - a) if (a is not None and b is not None) else None for a, b in zip(c0[d], c1[d])]
                 for d in c0}
        print(json.dumps({"nvml_check": "bidir bulk pull 64 CTAs", "GBps": bw, "bytes_each_way": moved,
                          "nvml_tx_rx_delta": delta}), flush=True)
    except Exception as exc:  # noqa: BLE001
        print(json.dumps({"nvml_check": "failed", "error": str(exc)[:200]}), flush=True)

    try:
        import pynvml as nv
        h = ctr.h[0]
        rep = {}
        for fid in (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
                    nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, nv.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
                    nv.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES):
            vals = nv.nvmlDeviceGetFieldValues(h, [(fid, link) for link in range(18)] + [(fid, 0xFFFFFFFF)])
            rep[fid] = [(v.nvmlReturn, int(v.value.ullVal)) for v in vals]
        print(json.dumps({"nvml_fields_gpu0": rep}), flush=True)
    except Exception as exc:  # noqa: BLE001
        print(json.dumps({"nvml_fields": "failed", "error": str(exc)[:200]}), flush=True)

    shapes = [(32768, 4)] if args.quick else [(16384, 8), (16384, 12), (32768, 4), (32768, 6), (65536, 2)]
    for bidir in (False, True):
        for kind in ("pull", "push"):
            for ctas in ctas_list:
                rec = {"bidir": bidir, "kind": kind, "ctas": ctas, "ldg": go("ldg", kind, ctas, bidir)}
                for tile, stages in shapes:
                    rec[f"bulk_{tile // 1024}k_x{stages}"] = go("bulk", kind, ctas, bidir, tile, stages)
                print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
