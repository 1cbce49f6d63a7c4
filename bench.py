#!/usr/bin/env python
"""FTAR bus bandwidth on B200 (driver contract; one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ftar|reference]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N

Workload (BASELINE.json metric "FTAR bus GB/s vs bucket size at 2/4/8 B200"):
  * N >= 2: one replica per GPU (north_star), a 256 MiB fp32 gradient bucket
    per replica in the group's registered pool, reduced out of place (fp32
    out=, --inplace for the reference's in-place shape) with the fused
    normalisation x f32(1/N) (replica.py:622-626) — the bucket class the
    >= 64 MB target names; the two-shot NVLink kernel (reduce-scatter by peer
    pulls, all-gather by pushes into the peers' registered outputs).
  * N = 1: the metric's multi-replica configs do not fit one GPU, so the
    replicas are emulated: 4 replicas (config 1's replica count) of the same
    bucket on cuda:0, reduced by the in-process one-shot kernel.  That number
    is HBM-bound, and its roofline says so.
  value = busbw = (E*in_bytes / t_step) * 2(n-1)/n (NCCL convention), t_step
  from CUDA events over the K timed steps, max over ranks.
  e2e   = the same metric through the public API with host buffers: pinned
  host -> device copy of the step's bucket(s), the all-reduce, and the
  device -> host read of the reduced bucket(s), all inside the timed region.
  The reference arm (--impl reference) times the C port of the reference's
  CPU ring (oracle/ftar_ref.c) on this host with all its threads.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


class _StdoutToStderr:
    """Rank 0's stdout must be exactly one JSON line: route fd 1 to stderr
    while NCCL initialises (its version banner is printed from C)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)

MIB = 1024 * 1024
NVLINK_PEER_GBS = 770.0   # B200_PROFILING.md measured peer copy per direction (fallback; 900 nominal)
NVLINK_NOMINAL_GBS = 900.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region through
    NVML (polled every ~2 ms on a thread; the timed region can be a few ms)."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, cuda_index: int, interval_s: float | None = None):
        self.cuda_index = cuda_index
        self.interval_s = float(os.environ.get("FTAR_CLOCK_INTERVAL_S", 0.002)) if interval_s is None else interval_s
        self.samples = []
        self.stop = threading.Event()
        self.err = None
        self.max_mhz = None

    def __enter__(self):
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            pr = torch.cuda.get_device_properties(self.cuda_index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            try:
                self.h = nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
            except Exception:  # noqa: BLE001
                self.h = nv.nvmlDeviceGetHandleByIndex(self.cuda_index)
            self.nv = nv
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception as exc:  # noqa: BLE001
            self.err = str(exc)[:120]
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception as exc:  # noqa: BLE001
                self.err = str(exc)[:120]
                return
            time.sleep(self.interval_s)

    def __exit__(self, *exc):
        self.stop.set()
        if hasattr(self, "thread"):
            self.thread.join(timeout=1)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"], "samples": 0,
                    "error": self.err}
        reasons = set()
        for _, rs in self.samples:
            for name, attr in self.REASONS:
                if rs & getattr(self.nv, attr, 0):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm for sm, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(self.samples), "source": "nvml"}


def busbw(elem_bytes_total: float, t: float, n: int) -> float:
    return (elem_bytes_total / t) * (2 * (n - 1) / n) / 1e9 if n > 1 else (elem_bytes_total / t) / 1e9


# --------------------------------------------------------------------------- CPU


def cpu_ring_rate(n: int, elems: int, seconds: float = 10.0, steps: int | None = None, warmup: int = 0):
    """The C port of the reference ring on this host (oracle/ftar_ref.c)."""
    import numpy as np
    from oracle import cref
    cref.build()
    cores = os.cpu_count() or 1
    tpm = max(1, cores // n)
    rng = np.random.default_rng(0)
    bufs = [rng.standard_normal(elems).astype(np.float32) for _ in range(n)]
    for b in bufs:
        b *= np.float32(1e-3)
    for _ in range(warmup):
        cref.ring_allreduce(bufs, 8 * MIB, 4, tpm)
    times = []
    t_end = time.perf_counter() + seconds
    while (steps is not None and len(times) < steps) or (steps is None and (time.perf_counter() < t_end or len(times) < 3)):
        t0 = time.perf_counter()
        cref.ring_allreduce(bufs, 8 * MIB, 4, tpm)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    return {"value": round(busbw(elems * 4, t, n), 3), "unit": "GB/s", "cores": n * tpm, "kind": "port",
            "sample": f"{n} replicas x {elems} fp32 (the full bucket) through the C port of the reference ring "
                      f"(oracle/ftar_ref.c: staging copy, N-1 RS + N-1 AG ring steps, per-partition commit; "
                      f"TCP hop replaced by shared memory), {len(times)} calls, {t * 1e3:.2f} ms/call",
            "ms_per_call": t * 1e3, "calls": len(times)}


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = max(args.gpus, 1) if args.gpus > 1 else args.replicas
    r = cpu_ring_rate(n, args.bucket_mib * MIB // 4, steps=args.steps, warmup=min(args.warmup, 1))
    cfg = workload_config(args, n)
    line = {"metric": METRIC, "value": r["value"], "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(r["ms_per_call"], 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": cfg,
            "impl": "reference",
            "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": r["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- inputs / parity


def member_bucket(rank: int, elems: int, dtype: str):
    """Replica `rank`'s synthetic gradient bucket:
    default_rng((0, rank)).standard_normal(E) as fp32, bf16 buckets rounded
    to nearest even.  A CPU tensor; the oracle regenerates the same bits."""
    import numpy as np
    import torch
    x = torch.from_numpy(np.random.default_rng((0, rank)).standard_normal(elems).astype(np.float32))
    return x.to(torch.bfloat16) if dtype == "bf16" else x


def expected_digest(n: int, elems: int, dtype: str) -> str:
    """sha256 of the reference result for the bench bucket: the oracle's fold
    (tests/test_ftar.py:20-40 restated in oracle/ftar_oracle.py) of every
    replica's bucket with the default geometry, times f32(1/n)
    (replica.py:622-626).  The checker only: it never produces a timed
    result."""
    import hashlib
    from oracle import ftar_oracle as orc  # checker (test infrastructure)
    arrays = [member_bucket(r, elems, dtype).float().numpy() for r in range(n)]
    want = orc.normalize(orc.oracle_reduce(arrays, 8 * MIB, 4), n)
    return hashlib.sha256(want.tobytes()).hexdigest()


def digest(t) -> str:
    import hashlib
    return hashlib.sha256(t.detach().float().cpu().numpy().tobytes()).hexdigest()


def device_digest(t) -> tuple:
    """Position-weighted 64-bit sums of a large fp32 tensor's bit patterns,
    computed on the device in 64 Mi-element chunks (a host sha256 of GiBs
    would take seconds)."""
    import torch
    x = t.detach().reshape(-1).view(torch.int32)
    s1 = s2 = 0
    step = 64 << 20
    w = (torch.arange(step, device=t.device, dtype=torch.int64) % 65521) + 1
    for i in range(0, x.numel(), step):
        c = x[i:i + step].to(torch.int64)
        s1 += int(c.sum())
        s2 += int((c * w[:c.numel()]).sum())
    return (s1, s2)


# --------------------------------------------------------------------------- GPU

METRIC = "FTAR bus GB/s vs bucket size at 2/4/8 B200 (% NVLink peak); catch-up ms/GB"


def workload_config(args, n):
    elems = args.bucket_mib * MIB // 4
    emu = args.gpus <= 1
    return {"workload": ("config3-class bucket, replicas emulated on one GPU (N=1)" if emu
                         else "config3-class bucket, one replica per GPU over NVLink"),
            "replicas": n, "bucket_elems_per_replica": elems,
            "bucket_bytes_per_replica": elems * (2 if args.dtype == "bf16" else 4),
            "in_dtype": args.dtype, "out_dtype": "f32", "chunk_bytes": 8 * MIB, "max_in_flight": 4,
            "fused": "x f32(1/n) normalisation" + (", bf16->fp32 cast" if args.dtype == "bf16" else ""),
            "result": "in place" if args.inplace else "out-of-place fp32 (out=)",
            "buffers": ("torch.empty tensors, " + ("registered (RingGroup.register)" if args.register
                                                    else "staged per call") if args.unregistered
                        else "registered pool (RingGroup.alloc_bucket)"),
            "kernel": "in-process one-shot" if emu else "two-shot NVLink (push all-gather)",
            "queue_depth": args.depth,
            "l2": "inputs larger than L2 (126 MB) per GPU; no flush needed",
            "parallelism": f"dp{n}" + (" (emulated)" if emu else "")}


def _ncu_traffic(args):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the N=1
    kernel, from the committed ncu --set full capture of this exact default
    workload (profiles/r01/ncu/summary.json); None for any other workload."""
    if args.dtype != "f32" or args.bucket_mib != 256 or args.replicas != 4 or args.inplace:
        return None
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "ncu",
                               "summary.json")) as f:
            return json.load(f)["per_launch"]["traffic_bytes"]
    except (OSError, KeyError, ValueError):
        return None


def timed_loop(fn, steps, stream, torch, drain=None):
    """The timed region: fn() `steps` times between two CUDA events on the
    launching stream (nothing else on the stream: an event recorded between
    two launches costs ~5 us, 1.5% of a 0.37 ms step).  Returns (total s,
    total / steps)."""
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for _ in range(steps):
        fn()
    if drain is not None:
        drain()
    t_end.record(stream)
    torch.cuda.synchronize()
    total = t_start.elapsed_time(t_end) / 1e3
    return total, total / steps


def launch_times(fn, steps, stream, torch, drain=None):
    """Average launch duration (s) of the dominant kernel: a second pass of
    `steps` calls right after the timed region with a CUDA event pair around
    every launch (the roofline's denominator).  The events themselves add a
    few us per launch, so this is an upper bound on the kernel time."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record(stream)
        fn()
        ev[i][1].record(stream)
    if drain is not None:
        drain()
    torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in ev]
    if os.environ.get("FTAR_BENCH_VERBOSE"):
        print(json.dumps({"rank": int(os.environ.get("RANK", 0)), "per_launch_ms": [round(x, 4) for x in per]}),
              file=sys.stderr, flush=True)
    return sum(per) / len(per) / 1e3


class NvlinkPM:
    """This GPU's NVLink bytes over a window from CUPTI PM sampling
    (tools/nvlink_pm.cpp): device-level nvlrx/nvltx counters sampled on a
    timer while the kernels run concurrently.  The measured traffic behind
    roofline.traffic for N >= 2 (NVML's NVLink fields are N/A on this driver)."""

    NVLINK = ("nvlrx__bytes.sum", "nvltx__bytes.sum", "nvlrx__bytes_data_user.sum", "nvltx__bytes_data_user.sum")
    KEYS = ("rx", "tx", "rx_user", "tx_user")

    def __init__(self, cuda_index: int, interval_ns: int = 50_000, metrics=None, keys=None):
        import ctypes as C
        self.dev, self.lib, self.err = cuda_index, None, None
        self.metrics = tuple(metrics or self.NVLINK)
        self.keys = tuple(keys or self.KEYS)
        path = os.path.join(ROOT, "tools", "_build", "libnvlink_pm.so")
        try:
            if not os.path.exists(path):
                os.makedirs(os.path.dirname(path), exist_ok=True)
                subprocess.run(["g++", "-O2", "-shared", "-fPIC", "-I/usr/local/cuda/include",
                                os.path.join(ROOT, "tools", "nvlink_pm.cpp"), "-L/usr/local/cuda/lib64", "-lcupti",
                                "-o", path], check=True, capture_output=True, timeout=120)
            lib = C.CDLL(path)
            lib.nvpm_error.restype = C.c_char_p
            lib.nvpm_open.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_char_p]
            lib.nvpm_stop.argtypes = [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_int)]
            if lib.nvpm_open(cuda_index, interval_ns, 200_000, ",".join(self.metrics).encode()):
                self.err = lib.nvpm_error().decode()
            else:
                self.lib = lib
        except Exception as exc:  # noqa: BLE001
            self.err = str(exc)[:200]

    def start(self):
        if self.lib is not None and self.lib.nvpm_start(self.dev):
            self.err = self.lib.nvpm_error().decode()
            self.lib = None

    def stop(self):
        """{rx, tx, rx_user, tx_user} bytes of the window, or None."""
        import ctypes as C
        if self.lib is None:
            return None
        out = (C.c_double * 8)()
        n, span, ovf = C.c_int(), C.c_uint64(), C.c_int()
        if self.lib.nvpm_stop(self.dev, out, C.byref(n), C.byref(span), C.byref(ovf)):
            self.err = self.lib.nvpm_error().decode()
            return None
        r = {k: out[i] for i, k in enumerate(self.keys)}
        r.update({"samples": n.value, "span_ms": span.value / 1e6, "overflow": bool(ovf.value)})
        return r

    def close(self):
        if self.lib is not None:
            self.lib.nvpm_close(self.dev)


class NvlinkBytes:
    """This GPU's NVLink data bytes (TX, RX) from NVML field values
    (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB counters summed over all
    links with scopeId = UINT_MAX), read around the timed region: the
    measured traffic behind roofline.traffic for N >= 2."""

    def __init__(self, cuda_index: int):
        self.h = None
        try:
            import pynvml as nv
            import torch
            nv.nvmlInit()
            pr = torch.cuda.get_device_properties(cuda_index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self.nv, self.h = nv, nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception as exc:  # noqa: BLE001
            self.err = str(exc)[:120]

    def read(self):
        if self.h is None:
            return None
        nv = self.nv
        try:
            vals = nv.nvmlDeviceGetFieldValues(self.h, [(nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF),
                                                        (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)])
        except Exception as exc:  # noqa: BLE001
            self.err = str(exc)[:120]
            return None
        if any(v.nvmlReturn != 0 for v in vals):
            return None
        return [int(v.value.ullVal) * 1024 for v in vals]


def run_single(args):
    import torch
    from paper_2602_00277_b200 import ftar
    dev = torch.device("cuda", 0)
    n = args.replicas
    elems = args.bucket_mib * MIB // 4
    in_bytes = 2 if args.dtype == "bf16" else 4
    ring = ftar.LocalRing(n, device=dev, max_bucket_bytes=elems * in_bytes)
    hosts = [member_bucket(r, elems, args.dtype) for r in range(n)]
    bufs = [h.to(dev) for h in hosts]
    outs = bufs if args.inplace else [torch.empty(elems, device=dev) for _ in range(n)]
    cfg = ftar.PipelineConfig()
    scale = 1.0 / n
    stream = torch.cuda.current_stream(dev)

    # queued like the N>=2 path (--depth buckets in flight, as a bucketed
    # backward pass issues them); each launch is still waited and checked
    from collections import deque
    pend = deque()

    def collect():
        for st in ring.wait(pend.popleft(), cfg):
            if st:
                raise RuntimeError(f"all-reduce failed with status {st}")

    def step():
        pend.append(ring.launch(bufs, cfg, outs=outs, scale=scale))
        while len(pend) >= max(1, args.depth):
            collect()

    def drain():
        while pend:
            collect()

    for _ in range(args.warmup):
        step()
    drain()
    # self-check outside the timed region: one call from the pristine inputs
    # against the oracle's digest (in place: restore the inputs afterwards)
    if args.inplace:
        for b, h in zip(bufs, hosts):
            b.copy_(h)
    step()
    drain()
    got = [digest(o) for o in outs]
    want = None if args.no_check else expected_digest(n, elems, args.dtype)
    if args.inplace:
        for b, h in zip(bufs, hosts):
            b.copy_(h)
    torch.cuda.synchronize()
    # live DRAM traffic of the launch pass (CUPTI PM sampling; the window
    # holds only this kernel: inputs are resident, nothing else runs)
    pm = None if args.no_pm else NvlinkPM(0, metrics=("dram__bytes_read.sum", "dram__bytes_write.sum"),
                                          keys=("read", "write"))
    with ClockSampler(0) as clk:
        total, _ = timed_loop(step, args.steps, stream, torch, drain=drain)
        # the launch pass: per-launch events and the PM counters (sampling at
        # 50 us perturbs the kernel by ~1.5%, so neither is in the timed region)
        if pm is not None:
            pm.start()
        per_launch = launch_times(step, args.steps, stream, torch, drain=drain)
        pmw = pm.stop() if pm is not None else None
    if pm is not None:
        pm.close()
    t_step = total / args.steps
    after = None if args.inplace else [digest(o) for o in outs]
    parity = {"checked": "every replica's output of one call (before the timed region) vs the oracle digest"
                         + ("" if args.inplace else "; outputs after the timed steps identical"),
              "oracle_sha256": want, "ok": (want is not None and all(g == want for g in got)
                                           and (after is None or after == got))}
    value = busbw(elems * in_bytes, t_step, n)
    peaks = measured_peaks()
    alg_bytes = n * elems * (in_bytes + 4)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    roof = {"bound": "hbm", "achieved": round(alg_bytes / per_launch / 1e9, 1), "peak": hbm_peak,
            "unit": "GB/s", "frac": round(alg_bytes / per_launch / 1e9 / hbm_peak, 4),
            "traffic": (round((pmw["read"] + pmw["write"]) / args.steps) if pmw is not None
                        else args.traffic if args.traffic is not None else _ncu_traffic(args)),
            "traffic_source": ("dram__bytes_read.sum + dram__bytes_write.sum per launch over the K-launch pass after the timed region, "
                               "CUPTI PM sampling (live)" if pmw is not None
                               else "committed ncu capture (profiles/r01/ncu): " + str(pm.err if pm else "pm off")),
            "pm_window": pmw,
            "kernel": ("local_oneshot_kernel" if os.environ.get("FTAR_LOCAL_BULK", "1") == "0" or args.inplace
                       or os.environ.get("FTAR_TMA", "1") == "0" else "local_bulk_kernel"),
            "algorithmic_bytes_per_launch": alg_bytes,
            "definition": "n*E*(in_bytes+4): every replica's bucket read once, every replica's fp32 result "
                          "written once; peak = MEASURED_PEAKS.json hbm_gbs (measured copy)",
            "avg_launch_ms": round(per_launch * 1e3, 4),
            "launch_timing": "CUDA events around each of K launches, in a pass right after the timed region "
                             "(events between launches cost ~5 us each, so they stay out of the timed region)"}
    # the same replicas through the multi-GPU protocol kernel (allreduce_kernel,
    # members as CTA groups of one cooperative launch): the product kernel's
    # code path, timed here for the record (not the headline)
    proto = None
    if not args.no_protocol:
        pring = ftar.LocalRing(n, device=dev, max_bucket_bytes=elems * in_bytes, protocol=True)
        pout = [torch.empty(elems, device=dev) for _ in range(n)]
        for _ in range(2):
            pring.all_reduce(bufs, cfg, outs=pout, scale=scale)
        pok = want is not None and all(digest(o) == want for o in pout)
        tp, pl = timed_loop(lambda: pring.all_reduce(bufs, cfg, outs=pout, scale=scale), max(3, args.steps // 2),
                            stream, torch)
        proto = {"kernel": "allreduce_kernel (emulated: members as CTA groups)", "ms_per_call": round(pl * 1e3, 4),
                 "busbw_gbs": round(busbw(elems * in_bytes, pl, n), 3),
                 "hbm_gbs": round(alg_bytes / pl / 1e9, 1), "parity_ok": pok}
        pring.close()
    # e2e through the public API with HOST buffers (the reference's call
    # shape): LocalRing.all_reduce_host pipelines chunked H2D, the range
    # all-reduce and D2H; every step moves the replicas' buckets in and the
    # reduced buckets out over PCIe inside the timed region
    e2e = None
    if not args.no_e2e:
        phost = [h.pin_memory() for h in hosts]
        hout = [torch.empty(elems, dtype=torch.float32).pin_memory() for _ in range(n)]

        def e2e_step():
            ring.all_reduce_host(phost, cfg, outs=hout, scale=scale, chunk_elems=args.host_chunk_elems)

        for _ in range(2):
            e2e_step()
        ke = max(3, min(args.steps, 10))
        tot, _ = timed_loop(e2e_step, ke, stream, torch)
        e2e = {"value": round(busbw(elems * in_bytes, tot / ke, n), 3), "unit": "GB/s",
               "h2d_bytes_per_step": n * elems * in_bytes, "d2h_bytes_per_step": n * elems * 4,
               "ms_per_step": round(tot / ke * 1e3, 3), "steps": ke,
               "api": "LocalRing.all_reduce_host (pinned host buffers; chunked H2D/reduce/D2H pipeline)"}
        if want is not None:
            e2e["parity_ok"] = all(digest(h) == want for h in hout)
    cpu = None if args.no_cpu_baseline else cpu_ring_rate(n, elems, seconds=args.cpu_seconds)
    line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32" if args.dtype == "f32" else "bf16->f32", "data": "synthetic (numpy default_rng normal buckets)",
            "config": workload_config(args, n), "roofline": roof,
            "cpu_baseline": None if cpu is None else {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": e2e, "gpu_launches": args.steps, "clocks": clk.summary(),
            "parity": parity["ok"], "parity_detail": parity,
            "protocol_kernel_emulated": proto,
            "algbw_gbs": round(elems * in_bytes / t_step / 1e9, 3)}
    ring.close()
    print(json.dumps(line), flush=True)


def run_multi(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2602_00277_b200 import ftar
    from paper_2602_00277_b200.fabric import StoreFabric
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = world
    elems = args.bucket_mib * MIB // 4
    tdtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    in_bytes = 2 if args.dtype == "bf16" else 4
    store = dist.PrefixStore("ftar_bench", dist.distributed_c10d._get_default_store())
    fabric = StoreFabric(store)
    group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=elems * in_bytes,
                           pool_bytes=elems * (in_bytes + 4) + 4096)
    group.reconfig({r: ftar.PeerAddress(r) for r in range(n)}, 1, deadline_s=60.0)
    host = member_bucket(rank, elems, args.dtype)
    if args.unregistered:
        # the reference call shape on an ordinary caching-allocator tensor:
        # staged into the arena per call, or (--register) registered with the
        # ring once and then reduced in place / pushed into zero-copy
        buf = host.to(dev)
        out = buf if args.inplace else torch.empty(elems, device=dev)
        if args.register:
            group.register(buf)
            if out is not buf:
                group.register(out)
    else:
        buf = group.alloc_bucket(elems, tdtype)
        buf.copy_(host)
        out = buf if args.inplace else group.alloc_bucket(elems, torch.float32)
    cfg = ftar.PipelineConfig()
    scale = 1.0 / n
    stream = torch.cuda.current_stream(dev)

    # buckets are enqueued asynchronously (queue depth args.depth), the way a
    # bucketed backward pass issues them; every step is still one complete
    # all-reduce of the whole bucket and all of them finish inside the region
    pend = []

    def step():
        pend.append(ftar.ftar_all_reduce_async(group, buf, 0, cfg, out=None if out is buf else out, scale=scale))
        while len(pend) >= args.depth:
            pend.pop(0).wait()

    def drain():
        while pend:
            pend.pop(0).wait()

    for _ in range(args.warmup):
        step()
    drain()
    # self-check outside the timed region (in place: from the pristine inputs)
    if args.inplace:
        buf.copy_(host)
    step()
    drain()
    got = digest(out)
    want = None
    if not args.no_check:
        box = [expected_digest(n, elems, args.dtype) if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        want = box[0]
    if args.inplace:
        buf.copy_(host)
    torch.cuda.synchronize()
    dist.barrier()
    nvl = NvlinkBytes(local_rank)
    pm = NvlinkPM(local_rank) if not args.no_pm else None
    with ClockSampler(local_rank) as clk:
        c0 = nvl.read()  # (the counters cover the untimed collective below too: steps + 1 calls)
        # One untimed collective right before the window: it is a device-side
        # barrier, so the timed region starts on every rank when all streams
        # reach the same point, instead of absorbing the ranks' host-side exit
        # skew from dist.barrier() (and the sampler's start) into the first
        # timed launch (measured: 0.7-1.5 ms vs 0.64 ms steady at 256 MiB, N=4;
        # host work between this call and the window would reopen the skew).
        step()
        total, _ = timed_loop(step, args.steps, stream, torch, drain)
        c1 = nvl.read()
        # the launch pass: per-launch events and the PM counters (neither in
        # the timed region); the untimed call after the sampler's start is
        # the device-side barrier that absorbs the ranks' start skew
        if pm is not None:
            pm.start()
        step()
        per_launch = launch_times(step, args.steps, stream, torch, drain)
        pmw = pm.stop() if pm is not None else None
    if pm is not None:
        pm.close()
    dist.barrier()
    after = None if args.inplace else digest(out)
    phases = phase_us(group)
    tt = torch.tensor([total, per_launch], dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    total, per_launch = tt.tolist()
    oks = [None] * n
    dist.all_gather_object(oks, bool(want is not None and got == want and (after is None or after == got)))
    nv_meas = None
    if c0 is not None and c1 is not None:
        nv_meas = [(b - a) / (args.steps + 1) for a, b in zip(c0, c1)]
    if nv_meas is None and pmw is not None:
        # user data bytes (what the kernels moved; the link also carries
        # packet headers: nvlrx__bytes ~1.25x, reported beside)
        nv_meas = [pmw["tx_user"] / (args.steps + 1), pmw["rx_user"] / (args.steps + 1)]
    all_nv = [None] * n
    dist.all_gather_object(all_nv, nv_meas)
    all_pm = [None] * n
    dist.all_gather_object(all_pm, pmw if pmw is not None else {"error": pm.err if pm is not None else "off"})
    t_step = total / args.steps
    value = busbw(elems * in_bytes, t_step, n)
    nv_bytes = (n - 1) / n * elems * (in_bytes + 4)
    rx = [m[1] for m in all_nv if m is not None]
    tx = [m[0] for m in all_nv if m is not None]
    roof = {"bound": "nvlink", "achieved": round(nv_bytes / per_launch / 1e9, 1), "peak": NVLINK_PEER_GBS,
            "unit": "GB/s", "frac": round(nv_bytes / per_launch / 1e9 / NVLINK_PEER_GBS, 4),
            "traffic": round(max(rx)) if rx else None,
            "traffic_source": ("NVLink RX user-data bytes per launch (nvlrx__bytes_data_user.sum, all links) from "
                               "CUPTI PM sampling of each GPU across the K-launch pass after the timed region (+1 untimed call), max over ranks; "
                               "nvlink_pm_window has the totals incl. packet overhead (nvlrx__bytes.sum)"
                               if rx else "NVLink counters unavailable: " + json.dumps(all_pm[0])[:200]),
            "traffic_over_algorithmic": round(max(rx) / nv_bytes, 4) if rx else None,
            "nvlink_pm_window": all_pm,
            "nvlink_rx_bytes_per_launch": [round(x) for x in rx] if rx else None,
            "nvlink_tx_bytes_per_launch": [round(x) for x in tx] if tx else None,
            "kernel": "allreduce_kernel (two-shot: RS by NVLink pulls, AG by pushes)",
            "algorithmic_bytes_per_launch": int(nv_bytes),
            "definition": "NVLink ingress per GPU (n-1)/n*E*(in_bytes+4): RS pulls every peer's slice of my "
                          "segment, AG receives every peer's fp32 result; peak = 770 GB/s measured peer copy "
                          "per direction (B200_PROFILING.md fallback; MEASURED_PEAKS.json has no NVLink entry)",
            "frac_of_nominal_900": round(nv_bytes / per_launch / 1e9 / NVLINK_NOMINAL_GBS, 4),
            "avg_launch_ms": round(per_launch * 1e3, 4),
            "launch_timing": "CUDA events around each of K launches, in a pass right after the timed region "
                             "(events between launches cost ~5 us each, so they stay out of the timed region)"}
    e2e = None
    if not args.no_e2e:
        phost = host.pin_memory()
        hout = torch.empty(elems, dtype=torch.float32).pin_memory()

        def e2e_step():
            ftar.ftar_all_reduce(group, phost, 0, cfg, out=hout, scale=scale)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        ke = max(3, min(args.steps, 10))
        tot, _ = timed_loop(e2e_step, ke, stream, torch)
        t = torch.tensor([tot], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ok = [None] * n
        dist.all_gather_object(e_ok, bool(want is not None and digest(hout) == want))
        e2e = {"value": round(busbw(elems * in_bytes, t.item() / ke, n), 3), "unit": "GB/s",
               "h2d_bytes_per_step": elems * in_bytes, "d2h_bytes_per_step": elems * 4,
               "ms_per_step": round(t.item() / ke * 1e3, 3), "steps": ke,
               "per": "rank (each GPU its own PCIe)", "parity_ok": all(e_ok),
               "api": "ftar_all_reduce(group, pinned host tensor, out=host tensor): chunked H2D/reduce/D2H"}
    nccl = None
    if not args.no_nccl:
        nccl = nccl_busbw(args, n, elems, tdtype, dev, stream)
    group.close()
    del buf, out
    catchup = None
    if args.catchup_gib > 0:
        catchup = catchup_ms_per_gb(args, rank, n, dev, fabric)
    if rank == 0:
        parity = {"checked": "every rank's output of one call (before the timed region) vs the oracle digest"
                             + ("" if args.inplace else "; outputs after the timed steps identical"),
                  "oracle_sha256": want, "ranks_ok": oks}
        line = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": n, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f32" if args.dtype == "f32" else "bf16->f32",
                "data": "synthetic (numpy default_rng normal buckets)",
                "config": workload_config(args, n), "roofline": roof, "cpu_baseline": None,
                "e2e": e2e, "gpu_launches": args.steps, "clocks": clk.summary(),
                "parity": all(oks), "parity_detail": parity,
                "algbw_gbs": round(elems * in_bytes / t_step / 1e9, 3),
                "pct_nvlink_nominal": round(100 * value / NVLINK_NOMINAL_GBS, 2),
                "phases_us_rank0": phases,
                "nccl_allreduce": nccl, "catchup": catchup}
        print(json.dumps(line), flush=True)


def catchup_ms_per_gb(args, rank, n, dev, fabric):
    """The metric's second half: catch-up ms/GB.  Ranks 0..n-2 hold the same
    retention-1 snapshot (params + momentum, fp32, --catchup-gib in total);
    rank n-1 pulls it striped over all of them with the catch-up kernel on
    its side stream (checkpoint.start_fetch), alone on the GPUs (config 4's
    'pull alone' number; tools/bench_catchup.py measures it inside a running
    ring).  CUDA events on the pulling stream around each pull, best of 3,
    bytes checked against the donors' digest."""
    import torch
    import torch.distributed as dist
    from paper_2602_00277_b200 import checkpoint as ck
    rec, donors = n - 1, list(range(n - 1))
    half = int(args.catchup_gib * (1 << 30) / 2) // 4
    nbytes = 2 * half * 4
    snap = ck.SnapshotStore(capacity_bytes=nbytes, device=dev, fabric=fabric, rank=0, replica_id=rank)
    want = None
    if rank != rec:
        g = torch.Generator(device=dev).manual_seed(7)
        p = torch.randn(half, device=dev, generator=g)
        m = torch.randn(half, device=dev, generator=g)
        snap.capture(3, p, m)
        torch.cuda.synchronize()
        want = (device_digest(p), device_digest(m))
        del p, m
    dist.barrier()
    res = None
    if rank == rec:
        p_out = torch.empty(half, device=dev)
        m_out = torch.empty(half, device=dev)
        side = ck.catchup_stream(dev)
        times = []
        for i in range(4):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(side)
            h = ck.start_fetch(snap, donors, 3, 0, p_out, m_out, timeout_s=60, ctas=args.catchup_ctas,
                               refresh=(i == 0))
            h.wait()
            e.record(side)
            torch.cuda.synchronize()
            if i:
                times.append(s.elapsed_time(e))
        got = (device_digest(p_out), device_digest(m_out))
        ms = min(times)
        res = {"gib": args.catchup_gib, "bytes": nbytes, "ms": round(ms, 3),
               "ms_per_gb": round(ms / (nbytes / 1e9), 3), "gbs": round(nbytes / ms / 1e6, 1),
               "ctas": args.catchup_ctas, "donors": donors, "recovering_rank": rec, "got": got,
               "how": "rank n-1 pulls params+momentum striped over ranks 0..n-2 (checkpoint.start_fetch), "
                      "alone on the GPUs; CUDA events on the pulling stream, best of 3"}
        del p_out, m_out
    box = [None] * n
    dist.all_gather_object(box, res if rank == rec else want)
    dist.barrier()
    snap.close()
    if rank == 0:
        res = box[rec]
        res["bit_exact"] = res.pop("got") == box[0]
        return res
    return None


def phase_us(group):
    """Durations of the last call's kernel phases from its %globaltimer stamps."""
    import ctypes as C
    from paper_2602_00277_b200 import _lib
    t = (C.c_uint64 * 6)()
    _lib.lib.ftar_phase_times(group.ctx, t, 6)
    t = list(t)
    if not t[0] or not t[4]:
        return None
    names = ["entry_wait", "reduce_scatter", "rs_to_ag_barrier", "all_gather"]
    return {k: round((t[i + 1] - t[i]) / 1e3, 1) for i, k in enumerate(names) if t[i + 1] >= t[i]}


def nccl_busbw(args, n, elems, tdtype, dev, stream):
    """NCCL all_reduce on the same bucket (comparison only, never on the FTAR path)."""
    import torch
    import torch.distributed as dist
    try:
        with _StdoutToStderr():
            pg = dist.new_group(backend="nccl")
            x = torch.randn(elems, device=dev).to(tdtype)
            for _ in range(max(2, args.warmup)):
                dist.all_reduce(x, group=pg)
            torch.cuda.synchronize()
        dist.barrier()
        total, _ = timed_loop(lambda: dist.all_reduce(x, group=pg), args.steps, stream, torch)
        t = torch.tensor([total], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        in_bytes = 2 if tdtype == torch.bfloat16 else 4
        return {"busbw_gbs": round(busbw(elems * in_bytes, t.item() / args.steps, n), 3),
                "dtype": str(tdtype).replace("torch.", ""), "ms_per_step": round(t.item() / args.steps * 1e3, 4)}
    except Exception as exc:  # noqa: BLE001
        return {"error": str(exc)[:200]}


def _reexec_under_torchrun(n: int) -> None:
    """`bench.py --gpus N` (N > 1) outside torchrun: one rank per GPU is the
    only meaningful shape, so re-launch this command under
    torch.distributed.run with N local ranks (never emulate silently)."""
    import socket
    try:
        import torch
        have = torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        have = 0
    if have < n:
        log(f"bench.py --gpus {n}: only {have} CUDA device(s) visible; refusing to emulate {n} GPUs")
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("bench.py: re-launching under torchrun:", " ".join(cmd))
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ftar", "reference"], default="ftar")
    ap.add_argument("--dtype", choices=["f32", "bf16"], default="f32")
    ap.add_argument("--bucket-mib", type=int, default=256, help="fp32-equivalent MiB per replica (E = MiB*2^20/4)")
    ap.add_argument("--replicas", type=int, default=4, help="emulated replicas at N=1")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--traffic", type=float, default=None, help="ncu dram bytes per launch, if captured")
    ap.add_argument("--inplace", action="store_true", help="reduce fp32 buckets in place (reference API shape)")
    ap.add_argument("--depth", type=int, default=3, help="queued all-reduces per rank (1 = blocking)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--host-chunk-elems", type=int, default=8 << 20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the oracle self-check")
    ap.add_argument("--catchup-gib", type=float, default=8.0,
                    help="N>=2: also time the catch-up pull of this many GiB of params+momentum (0: skip)")
    ap.add_argument("--catchup-ctas", type=int, default=32, help="CTAs of the catch-up pull in that measurement")
    ap.add_argument("--no-pm", action="store_true", help="no CUPTI PM sampling (N=1: DRAM bytes, N>=2: NVLink bytes)")
    ap.add_argument("--no-protocol", action="store_true", help="N=1: skip the protocol-kernel record")
    ap.add_argument("--unregistered", action="store_true",
                    help="N>=2: buckets are ordinary torch.empty tensors (reference call shape), not pool buffers")
    ap.add_argument("--register", action="store_true",
                    help="with --unregistered: RingGroup.register the tensors (zero-copy) instead of staging")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _reexec_under_torchrun(args.gpus)
    args.warmup = max(args.warmup, 3) if args.impl == "ftar" else args.warmup
    if args.dtype == "bf16":
        args.inplace = False
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif world > 1:
        run_multi(args, rank, world, local_rank)
    else:
        run_single(args)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
