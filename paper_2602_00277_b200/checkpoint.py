"""Catch-up state transfer on B200 — drop-in for the snapshot/fetch half of
``ftdp.checkpoint`` (pkg/src/ftdp/checkpoint.py:48-154).

* ``SnapshotStore``  retention-1 copy of one rank shard's (params, momentum)
  for the last committed step (checkpoint.py:56-80), held in a device arena
  that other replicas can map (CUDA IPC).  ``capture`` is a stream-ordered
  seqlock + copy kernel on the donor (replica.py:645-648).
* ``fetch_shard``    the recovering replica pulls the donor's snapshot over
  NVLink with a rate-limited kernel (``ctas`` SMs) on a low-priority side
  stream, so the donor's and everyone else's FTAR steps keep running
  (checkpoint.py:117-144, replica.py:452-493).  Called with the reference's
  arguments ``fetch_shard(addr, step, rank, replica_id, incarnation,
  timeout_s, plan)`` it resolves the caller's own store from a per-process
  registry keyed by (replica_id, rank) and the donor from ``addr.replica_id``
  (in this process, or through the store's fabric), and returns
  ``(params, momentum)`` as device byte tensors.  A donor that holds another
  step — or re-captures during the pull — yields ``SnapshotUnavailable``
  with the step it has (checkpoint.py:132-133); a donor that never published
  or whose process is gone yields ``Recoverable(PEER_DOWN)``.
* ``pick_donor``     round-robin donor choice (checkpoint.py:147-154).
* ``serve_fetches``  the reference's server thread target: on NVLink the
  donor serves by publishing its snapshot arena once, so the thread only
  waits for ``stop``.

* Persistent checkpoints (checkpoint.py:155-230): the
  reference's shard file and manifest format byte for byte (``write_shard``,
  ``read_shard``, ``write_manifest``, ``find_latest``), written straight from
  the device snapshot by ``SnapshotStore.persist`` (chunked D2H through pinned
  buffers, seqlock-validated, atomic rename) without stopping the step.

The loader ledger (checkpoint.py:233-316) is data-loader bookkeeping, not
this path, and is out of scope.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import re
import struct
import threading
import time

import weakref

import torch

from . import _lib
from .errors import INTERNAL_INVARIANT, PEER_DOWN, PROTOCOL_VIOLATION, Fatal, Recoverable, from_status
from .fabric import ArenaInfo, LocalFabric


class SnapshotUnavailable(Exception):
    """The donor no longer (or does not yet) hold the requested step."""

    def __init__(self, available):
        super().__init__(f"snapshot unavailable (donor holds {available})")
        self.available = available


def _as_bytes_tensor(t: torch.Tensor) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda or not t.is_contiguous():
        raise Fatal(INTERNAL_INVARIANT, "snapshot tensors must be contiguous CUDA tensors")
    return t


# Every SnapshotStore of this process by (replica_id, rank): how the
# reference-shaped fetch_shard(addr, step, rank, replica_id, ...) finds the
# caller's own store and in-process donors.
_STORES: "weakref.WeakValueDictionary[tuple[int, int], SnapshotStore]" = weakref.WeakValueDictionary()


class SnapshotStore:
    """Latest committed (params, momentum) shard of this rank on its GPU."""

    def __init__(self, capacity_bytes: int = 0, device=None, fabric=None, rank: int = 0,
                 replica_id: int = 0, incarnation: int = 0):
        if not torch.cuda.is_available():
            raise Fatal(INTERNAL_INVARIANT, "SnapshotStore needs a CUDA device")
        self.device = torch.device(device if device is not None else torch.cuda.current_device())
        self.device_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.fabric = fabric
        self.rank = rank
        self.replica_id = replica_id
        self.incarnation = incarnation
        self._lock = threading.Lock()
        self._snap = None
        self._cap = 0
        self._step = None
        self._lens = (0, 0)
        # donor snapshot mappings by (donor replica, incarnation); slots from a
        # free list, a donor's older incarnation is unmapped when a newer one
        # is mapped, and retain() drops donors that left the decision
        self._peers: dict[tuple[int, int], int] = {}
        self._free_slots: list[int] = list(range(255, -1, -1))
        self.map_log: list[tuple] = []
        _STORES[(replica_id, rank)] = self
        # the pull's side streams exist before any pull: creating them inside
        # a recovering replica's first catch-up step cost 17.6 ms of host time
        # right between two of its collective launches (config 5, N=4)
        catchup_stream(self.device, 0)
        catchup_stream(self.device, 1)
        if capacity_bytes:
            self._alloc(capacity_bytes)

    def _alloc(self, capacity: int) -> None:
        s = C.c_void_p()
        exportable = self.fabric is not None and not isinstance(self.fabric, LocalFabric)
        _lib.check(_lib.lib.ftar_snap_create(self.device_index, capacity, 1 if exportable else 0, C.byref(s)),
                   "ftar_snap_create")
        self._snap, self._cap = s, capacity
        if exportable:
            buf = (C.c_char * 64)()
            n = C.c_size_t()
            _lib.check(_lib.lib.ftar_snap_export(s, buf, 64, C.byref(n)), "ftar_snap_export")
            self.fabric.publish(ArenaInfo(self.replica_id, self.rank, self.incarnation, self.device_index,
                                          bytes(buf)[:n.value], capacity, pid=os.getpid()), what="snap")

    @property
    def handle(self):
        return self._snap

    def capture(self, step: int, params: torch.Tensor, momentum: torch.Tensor) -> None:
        """Replace the snapshot with `step`'s shard (stream-ordered on the
        current stream: the copy sees every prior write to params/momentum).
        Host bytes (the reference's call shape) are copied to the device
        first."""
        p, m = self._device_bytes(params), self._device_bytes(momentum)
        if p.device.index != self.device_index or m.device.index != self.device_index:
            raise Fatal(INTERNAL_INVARIANT, f"snapshot tensors must live on cuda:{self.device_index}")
        pb, mb = p.numel() * p.element_size(), m.numel() * m.element_size()
        with self._lock:
            if self._snap is None:
                self._alloc(pb + mb)
            elif pb + mb > self._cap:
                raise Fatal(INTERNAL_INVARIANT, f"snapshot of {pb + mb} bytes exceeds capacity {self._cap}")
            stream = torch.cuda.current_stream(self.device).cuda_stream
            _lib.check(_lib.lib.ftar_snap_capture(self._snap, step, p.data_ptr(), pb, m.data_ptr(), mb, stream),
                       "ftar_snap_capture")
            self._step, self._lens = step, (pb, mb)

    @property
    def step(self):
        with self._lock:
            return self._step

    def device_step(self):
        """The step recorded in the device header (synchronises)."""
        if self._snap is None:
            return None
        st, pb, mb = C.c_int64(), C.c_uint64(), C.c_uint64()
        _lib.check(_lib.lib.ftar_snap_info(self._snap, C.byref(st), C.byref(pb), C.byref(mb)), "ftar_snap_info")
        return None if st.value < 0 else st.value

    def _device_bytes(self, x):
        if isinstance(x, torch.Tensor):
            if x.is_cuda:
                return _as_bytes_tensor(x)
            x = x.contiguous().view(-1).view(torch.uint8)
        else:
            import numpy as np
            x = torch.from_numpy(np.frombuffer(bytes(x), dtype=np.uint8).copy())
        return x.to(self.device) if x.numel() else torch.empty(0, dtype=torch.uint8, device=self.device)

    def get(self, step: int):
        """The held shard if it is `step` (checkpoint.py:76-80): (params,
        momentum) as device byte tensors viewing the snapshot arena (valid
        until the next capture); SnapshotUnavailable(held step) otherwise."""
        with self._lock:
            if self._step != step:
                raise SnapshotUnavailable(self._step)
            pb, mb = self._lens
            pp, mp = C.c_void_p(), C.c_void_p()
            _lib.check(_lib.lib.ftar_snap_region(self._snap, C.byref(pp), C.byref(mp), None, None, None, None),
                       "ftar_snap_region")
            from .ftar import _CudaView

            def view(ptr, n):
                if not n:
                    return torch.empty(0, dtype=torch.uint8, device=self.device)
                t = torch.as_tensor(_CudaView(ptr, (n,), "|u1"), device=self.device)
                t._ftar_owner = self
                return t
            return view(pp.value, pb), view(mp.value, mb)

    @property
    def lengths(self) -> tuple[int, int]:
        """(params bytes, momentum bytes) of the held shard."""
        with self._lock:
            return self._lens

    def close(self) -> None:
        t = self.__dict__.get("_connecting")
        if t is not None:
            t.join()
        if self._snap is not None:
            _lib.lib.ftar_snap_destroy(self._snap)
            self._snap = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    # --- recovering side --------------------------------------------------------
    def connect(self, donors, rank: int = 0, timeout_s: float = 5.0, background: bool = False) -> None:
        """Map the donors' snapshot arenas ahead of the pull.  CUDA IPC mapping
        of a multi-GB arena costs 0.1-0.5 s per donor; a respawned replica does
        it while parked, so its first (gated) step is not late to the ring.
        ``background=True`` maps on a helper thread (the caller keeps taking
        part in quorum rounds); the next fetch joins it first."""
        if self._snap is None:
            raise Fatal(INTERNAL_INVARIANT, "connect needs a snapshot arena (capacity_bytes=)")
        todo = [int(d) for d in donors if int(d) != self.replica_id]
        if not background:
            for d in todo:
                self._map_donor(d, rank, timeout_s)
            return
        self.join_connect()
        dev = self.device_index

        def run():
            torch.cuda.set_device(dev)
            try:
                for d in todo:
                    self._map_donor(d, rank, timeout_s)
            except Exception as exc:  # noqa: BLE001 - surfaced by join_connect
                self._connect_err = exc

        self._connect_err = None
        self._connecting = threading.Thread(target=run, name="ftar-snap-connect", daemon=True)
        self._connecting.start()

    def connecting(self) -> bool:
        """True while a background connect is still mapping donors."""
        t = self.__dict__.get("_connecting")
        return t is not None and t.is_alive()

    def join_connect(self) -> None:
        """Wait for a background connect; re-raise its failure."""
        t = self.__dict__.get("_connecting")
        if t is not None:
            t.join()
            self._connecting = None
            if self._connect_err is not None:
                err, self._connect_err = self._connect_err, None
                raise err

    def _map_donor(self, donor_replica: int, rank: int, timeout_s: float, refresh: bool = True) -> int:
        """Slot of the donor's snapshot mapping.  ``refresh=False`` reuses the
        newest mapping of that donor without asking the fabric (a Store round
        trip per donor: ~4 ms each, on the recovering replica's critical path
        right before its first collective); a stale mapping (the donor
        restarted) shows up as SnapshotUnavailable, and callers then retry
        with a refresh."""
        if not refresh:
            known = sorted(k for k in self._peers if k[0] == donor_replica)
            if known:
                return self._peers[known[-1]]
        if self.fabric is None:
            raise Recoverable(PEER_DOWN, f"replica {donor_replica} is not in this process and no fabric is set")
        t0 = time.monotonic()
        info = self.fabric.lookup(rank, donor_replica, timeout_s, what="snap")
        key = (donor_replica, info.incarnation)
        if key not in self._peers:
            # an older incarnation of this donor is dead: release its snapshot
            for old in [k for k in self._peers if k[0] == donor_replica]:
                self._unmap(old)
            if not self._free_slots:
                raise Fatal(INTERNAL_INVARIANT, "no free donor slots (256 mapped)")
            t1 = time.monotonic()
            slot = self._free_slots.pop()
            rc = _lib.lib.ftar_snap_import(self._snap, slot, info.handle, len(info.handle), info.arena_bytes)
            if rc:
                self._free_slots.append(slot)
                raise Recoverable(PEER_DOWN, f"cannot map snapshot of replica {donor_replica}: {_lib.last_error()}")
            self._peers[key] = slot
            # (donor, lookup s, IPC open s, bytes): start-up cost accounting
            self.map_log.append((donor_replica, t1 - t0, time.monotonic() - t1, info.arena_bytes))
        return self._peers[key]

    def _unmap(self, key) -> None:
        slot = self._peers.pop(key)
        _lib.check(_lib.lib.ftar_snap_unmap(self._snap, slot), f"unmap snapshot of replica {key[0]}")
        self._free_slots.append(slot)

    def retain(self, live) -> None:
        """Unmap every donor snapshot whose (replica, incarnation) is not in
        `live` (a {replica: incarnation} map of the current decision, or an
        iterable of replica ids: any incarnation of those is kept)."""
        self.join_connect()
        if isinstance(live, dict):
            drop = [k for k in self._peers if live.get(k[0]) != k[1]]
        else:
            keep = {int(r) for r in live}
            drop = [k for k in self._peers if k[0] not in keep]
        for k in drop:
            self._unmap(k)

    @property
    def mapped_donors(self) -> list[tuple[int, int]]:
        return sorted(self._peers)

    def _peer_header(self, slot: int):
        st, pb, mb = C.c_int64(), C.c_uint64(), C.c_uint64()
        _lib.check(_lib.lib.ftar_snap_peer_info(self._snap, slot, C.byref(st), C.byref(pb), C.byref(mb)),
                   "ftar_snap_peer_info")
        return (None if st.value < 0 else int(st.value)), int(pb.value), int(mb.value)


class CatchupPull:
    """One in-flight pull of a donor snapshot (non-blocking catch-up)."""

    def __init__(self, local: SnapshotStore, params: torch.Tensor, momentum: torch.Tensor, stream,
                 timeout_s: float):
        self.local, self.params, self.momentum = local, params, momentum
        self.stream = stream
        self.timeout_s = timeout_s
        self.event = None

    def boost(self, ctas: int = 32) -> None:
        """Widen the pull now (e.g. once this step's collectives are done): a
        second grid on another low-priority stream takes over part of the
        remaining chunks."""
        stream = catchup_stream(self.local.device, 1)
        _lib.check(_lib.lib.ftar_snap_pull_boost(self.local.handle, ctas, stream.cuda_stream), "ftar_snap_pull_boost")
        self.streams = getattr(self, "streams", [self.stream]) + [stream]

    def poll(self):
        st, prog, avail = C.c_int(), C.c_uint64(), C.c_int64()
        _lib.lib.ftar_snap_poll(self.local.handle, C.byref(st), C.byref(prog), C.byref(avail))
        return st.value, prog.value

    def wait(self):
        avail = C.c_int64(-1)
        st = _lib.lib.ftar_snap_wait(self.local.handle, self.timeout_s, C.byref(avail))
        if st == _lib_status("UNAVAILABLE"):
            raise SnapshotUnavailable(None if avail.value < 0 else avail.value)
        if st:
            raise from_status(st, _lib.last_error() if st == 10 else "catch-up pull failed")
        # make the consumer stream see the pulled bytes
        for s in getattr(self, "streams", [self.stream]):
            torch.cuda.current_stream(self.local.device).wait_stream(s)
        return self.params, self.momentum


def _lib_status(name: str) -> int:
    return {"UNAVAILABLE": 9}[name]


_side_streams: dict[tuple[int, int], torch.cuda.Stream] = {}


def catchup_stream(device: torch.device, which: int = 0) -> torch.cuda.Stream:
    """Low-priority side streams per device for catch-up pulls (1: boost grids)."""
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if (idx, which) not in _side_streams:
        lo, hi = torch.cuda.Stream.priority_range()
        _side_streams[(idx, which)] = torch.cuda.Stream(device=idx, priority=lo if lo > hi else 0)
    return _side_streams[(idx, which)]


# CTA budget of a catch-up pull: each CTA streams ~47 GB/s (bulk copies), so 8
# CTAs cap the pull near 300 GB/s and leave the recovering GPU's NVLink
# ingress to the ring it is a member of (tools/bench_catchup.py, N=4: healthy
# steps 1.13x steady at 8 CTAs, 1.19x at 16, 1.24x at 32)
DEFAULT_PULL_CTAS = 8


def start_fetch(local: SnapshotStore, donor, step: int, rank: int, params_out: torch.Tensor,
                momentum_out: torch.Tensor, timeout_s: float = 5.0, ctas: int = DEFAULT_PULL_CTAS,
                refresh: bool = True) -> CatchupPull:
    """Launch the pull of `donor`'s snapshot of `step` into the given tensors
    without waiting.  `donor` is a SnapshotStore in this process (same device),
    a replica id resolved through ``local.fabric``, or a list of replica ids:
    the pull is then striped across all of them (every healthy replica holds
    the same retention-1 snapshot), so no single donor's NVLink egress carries
    the whole catch-up.  ``refresh=False`` reuses existing donor mappings
    without a fabric lookup (see SnapshotStore._map_donor)."""
    p, m = _as_bytes_tensor(params_out), _as_bytes_tensor(momentum_out)
    pb, mb = p.numel() * p.element_size(), m.numel() * m.element_size()
    local.join_connect()
    if local.handle is None:
        local._alloc(max(pb + mb, 16))
    if isinstance(donor, SnapshotStore):
        slots, src = [], donor.handle
        if src is None:
            raise SnapshotUnavailable(None)
        if donor.device_index != local.device_index:  # in-process donor on another GPU: peer access
            _lib.check(_lib.lib.ftar_peer_enable(local.device_index, donor.device_index), "ftar_peer_enable")
    else:
        donors = list(donor) if isinstance(donor, (list, tuple)) else [donor]
        slots, src = [local._map_donor(int(d), rank, timeout_s, refresh) for d in donors], None
    t0 = time.monotonic()
    stream = catchup_stream(local.device)
    stream.wait_stream(torch.cuda.current_stream(local.device))
    stream.wait_stream(catchup_stream(local.device, 1))  # a previous pull's boost grid has exited
    t1 = time.monotonic()
    arr = (C.c_int * max(1, len(slots)))(*slots)
    rc = _lib.lib.ftar_snap_pull_multi_launch(local.handle, arr, len(slots), src, step, p.data_ptr(), pb,
                                              m.data_ptr(), mb, ctas, stream.cuda_stream)
    _lib.check(rc, "ftar_snap_pull_launch")
    local.launch_log = (round((t1 - t0) * 1e3, 3), round((time.monotonic() - t1) * 1e3, 3))
    return CatchupPull(local, p, m, stream, timeout_s)


def _donor_id(addr) -> int:
    rid = getattr(addr, "replica_id", addr)
    return int(rid)


def _default_fabric():
    for st in list(_STORES.values()):
        if st.fabric is not None and not isinstance(st.fabric, LocalFabric):
            return st.fabric
    return None


def fetch_shard(addr, step: int, rank: int, replica_id: int = 0, incarnation: int = 0,
                timeout_s: float = 5.0, plan=None, *, local: SnapshotStore | None = None,
                out: tuple[torch.Tensor, torch.Tensor] | None = None, ctas: int = DEFAULT_PULL_CTAS):
    """Pull (params, momentum) of one rank shard of a committed step
    (checkpoint.py:117-144); the reference's signature.

    ``addr`` names the donor: a ``PeerAddress`` (its ``replica_id``), a
    replica id, a list of replica ids (striped pull), or a SnapshotStore of
    this process.  The caller's own store is ``local`` or the registered
    store of (replica_id, rank) (one is created on first use).  Returns
    (params, momentum) as device byte tensors (``out`` if given).  Raises
    SnapshotUnavailable(held step) when the donor holds another step and
    Recoverable(PEER_DOWN) when the donor never published or is gone; ``plan``
    (the reference's socket fault plan) has no NVLink analogue."""
    if local is None:
        local = _STORES.get((replica_id, rank))
        if local is None:
            local = SnapshotStore(device=torch.cuda.current_device(), fabric=_default_fabric(), rank=rank,
                                  replica_id=replica_id, incarnation=incarnation)
    if isinstance(addr, SnapshotStore):
        donor = addr
    elif isinstance(addr, (list, tuple)):
        donor = [_donor_id(a) for a in addr]
    else:
        did = _donor_id(addr)
        donor = _STORES.get((did, rank))
        if donor is None or donor is local:
            donor = did
    if isinstance(donor, SnapshotStore):
        held = donor.step
        if held != step:
            raise SnapshotUnavailable(held)
        pb, mb = donor.lengths
    else:
        ids = donor if isinstance(donor, list) else [donor]
        if local.handle is None:
            local._alloc(16)
        pb = mb = None
        for d in ids:
            held, dpb, dmb = local._peer_header(local._map_donor(d, rank, timeout_s))
            if held != step:
                raise SnapshotUnavailable(held)
            if pb is not None and (dpb, dmb) != (pb, mb):
                raise Fatal(PROTOCOL_VIOLATION, "donors disagree on the shard's lengths")
            pb, mb = dpb, dmb
    if out is None:
        out = (torch.empty(pb, dtype=torch.uint8, device=local.device),
               torch.empty(mb, dtype=torch.uint8, device=local.device))
    return start_fetch(local, donor, step, rank, out[0], out[1], timeout_s, ctas).wait()


def pick_donor(healthy, self_replica: int, rank: int, attempt: int = 0) -> int:
    """checkpoint.py:147-154: rank r pulls from donor (r + attempt) mod H."""
    donors = sorted(r for r in healthy if r != self_replica)
    if not donors:
        raise Recoverable(PEER_DOWN, "no donors available")
    return donors[(rank + attempt) % len(donors)]


def serve_fetches(router=None, store: SnapshotStore | None = None, stop=None, pred=None) -> None:
    """Thread target of checkpoint.py:83-95.  An NVLink donor serves by
    publishing its snapshot arena (done when the arena is allocated; peers
    then read it directly), so there is no per-request work: the thread
    only waits for ``stop``, as the reference's server loop does."""
    if stop is None:
        return None
    while not stop.wait(0.25):
        pass
    return None


# ------------------------------------------------------------- persistence
# checkpoint.py:155-230: one file per (step, rank) = MAGIC + header + params +
# momentum, written atomically (tmp + fsync + rename), plus a JSON manifest.

MAGIC = b"PAFTCKPT"
_SHARD_HDR = struct.Struct("<IQIQQ")  # version, step, rank, params_len, momentum_len
VERSION = 1
_CHUNK = 64 << 20  # bytes per pinned D2H staging buffer (two of them)


def shard_path(ckpt_dir: str, step: int, rank: int) -> str:
    return os.path.join(ckpt_dir, f"state_{step:08d}_rank{rank}.bin")


def manifest_path(ckpt_dir: str, step: int) -> str:
    return os.path.join(ckpt_dir, f"state_{step:08d}.json")


def _atomic_write(path: str, data: bytes) -> None:
    """Durable replace: the bytes reach the disk under a side name first, so a
    reader never sees a partial file under `path`."""
    side = f"{path}.tmp"
    fd = os.open(side, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
    try:
        view = memoryview(data)
        while view:
            view = view[os.write(fd, view):]
        os.fsync(fd)
    finally:
        os.close(fd)
    os.replace(side, path)


def _as_bytes(x) -> bytes:
    if isinstance(x, torch.Tensor):
        t = x.detach().contiguous().cpu()
        return t.view(torch.uint8).numpy().tobytes() if t.numel() else b""
    return bytes(x)


def write_shard(ckpt_dir: str, step: int, rank: int, params, momentum) -> str:
    """checkpoint.py:174-180.  params / momentum: bytes or tensors (CUDA
    tensors are copied to the host); the file is byte-identical to the
    reference's."""
    os.makedirs(ckpt_dir, exist_ok=True)
    p, m = _as_bytes(params), _as_bytes(momentum)
    path = shard_path(ckpt_dir, step, rank)
    _atomic_write(path, MAGIC + _SHARD_HDR.pack(VERSION, step, rank, len(p), len(m)) + p + m)
    return path


def _read_header(fh, path: str, step: int, rank: int):
    head = fh.read(len(MAGIC) + _SHARD_HDR.size)
    if head[:len(MAGIC)] != MAGIC:
        raise Fatal(PROTOCOL_VIOLATION, f"bad checkpoint magic in {path}")
    if len(head) < len(MAGIC) + _SHARD_HDR.size:
        raise Fatal(PROTOCOL_VIOLATION, f"truncated checkpoint shard {path}")
    version, got_step, got_rank, plen, mlen = _SHARD_HDR.unpack_from(head, len(MAGIC))
    if version != VERSION:
        raise Fatal(PROTOCOL_VIOLATION, f"unsupported checkpoint version {version}")
    if (got_step, got_rank) != (step, rank):
        raise Fatal(PROTOCOL_VIOLATION, f"checkpoint header ({got_step},{got_rank}) != ({step},{rank})")
    if len(head) + plen + mlen != os.fstat(fh.fileno()).st_size:
        raise Fatal(PROTOCOL_VIOLATION, f"truncated checkpoint shard {path}")
    return plen, mlen


def read_shard(ckpt_dir: str, step: int, rank: int) -> tuple[bytes, bytes]:
    """checkpoint.py:183-198: (params bytes, momentum bytes)."""
    path = shard_path(ckpt_dir, step, rank)
    with open(path, "rb") as fh:
        plen, mlen = _read_header(fh, path, step, rank)
        return fh.read(plen), fh.read(mlen)


def read_shard_into(ckpt_dir: str, step: int, rank: int, params_out: torch.Tensor,
                    momentum_out: torch.Tensor) -> None:
    """Restore a shard straight into device tensors (chunked H2D through
    pinned buffers)."""
    path = shard_path(ckpt_dir, step, rank)
    with open(path, "rb") as fh:
        plen, mlen = _read_header(fh, path, step, rank)
        for t, n in ((params_out, plen), (momentum_out, mlen)):
            if t.numel() * t.element_size() != n:
                raise Fatal(INTERNAL_INVARIANT, f"restore target holds {t.numel() * t.element_size()} bytes, "
                                                f"the shard {n}")
            flat = t.view(-1).view(torch.uint8)
            buf = torch.empty(min(n, _CHUNK) or 1, dtype=torch.uint8).pin_memory()
            for off in range(0, n, _CHUNK):
                k = min(_CHUNK, n - off)
                fh.readinto(memoryview(buf.numpy())[:k])
                flat[off:off + k].copy_(buf[:k], non_blocking=False)


def write_manifest(ckpt_dir: str, step: int, n_ranks: int, dims: tuple[int, ...],
                   cursors: dict[int, int]) -> str:
    """checkpoint.py:201-213 (same JSON document)."""
    doc = {"magic": MAGIC.decode(), "version": VERSION, "step": step, "n_ranks": n_ranks, "dims": list(dims),
           "cursors": {str(rid): int(cur) for rid, cur in sorted(cursors.items())}}
    path = manifest_path(ckpt_dir, step)
    _atomic_write(path, json.dumps(doc, indent=1).encode())
    return path


_MANIFEST_RE = re.compile(r"state_(\d{8})\.json")


def _manifest_ok(ckpt_dir: str, step: int):
    try:
        with open(manifest_path(ckpt_dir, step), "rb") as fh:
            doc = json.load(fh)
    except (OSError, json.JSONDecodeError):
        return None
    if doc.get("magic") != MAGIC.decode() or doc.get("step") != step:
        return None
    shards_present = all(os.path.exists(shard_path(ckpt_dir, step, r)) for r in range(doc.get("n_ranks", 0)))
    return doc if shards_present else None


def find_latest(ckpt_dir: str):
    """checkpoint.py:219-230: newest step whose manifest parses and whose shard
    files all exist, as (step, manifest)."""
    try:
        names = os.listdir(ckpt_dir)
    except (FileNotFoundError, NotADirectoryError):
        return None
    candidates = {int(m.group(1)) for m in map(_MANIFEST_RE.fullmatch, names) if m}
    for step in sorted(candidates, reverse=True):
        doc = _manifest_ok(ckpt_dir, step)
        if doc is not None:
            return step, doc
    return None
    steps = sorted((int(m.group(1)) for name in os.listdir(ckpt_dir) if (m := _MANIFEST_RE.match(name))),
                   reverse=True)
    for step in steps:
        try:
            with open(manifest_path(ckpt_dir, step), "rb") as fh:
                doc = json.load(fh)
        except (OSError, json.JSONDecodeError):
            continue
        if doc.get("magic") != MAGIC.decode() or doc.get("step") != step:
            continue
        if all(os.path.exists(shard_path(ckpt_dir, step, r)) for r in range(doc.get("n_ranks", 0))):
            return step, doc
    return None


class PersistJob:
    """A snapshot being written to storage (SnapshotStore.persist)."""

    def __init__(self, thread: threading.Thread | None, box: dict):
        self._thread, self._box = thread, box

    def done(self) -> bool:
        return self._thread is None or not self._thread.is_alive()

    def wait(self) -> str:
        """The written path; SnapshotUnavailable if a capture overwrote the
        snapshot mid-write (nothing is left behind then)."""
        if self._thread is not None:
            self._thread.join()
        if "error" in self._box:
            raise self._box["error"]
        return self._box["path"]


def _persist_snapshot(store: "SnapshotStore", ckpt_dir: str, rank: int, box: dict, hook=None) -> None:
    try:
        torch.cuda.set_device(store.device_index)
        pp, mp, pb, mb = C.c_void_p(), C.c_void_p(), C.c_uint64(), C.c_uint64()
        seq0, step0 = C.c_uint64(), C.c_int64()
        _lib.check(_lib.lib.ftar_snap_region(store.handle, C.byref(pp), C.byref(mp), C.byref(pb), C.byref(mb),
                                             C.byref(seq0), C.byref(step0)), "ftar_snap_region")
        if step0.value < 0:
            raise SnapshotUnavailable(None)
        step = int(step0.value)
        os.makedirs(ckpt_dir, exist_ok=True)
        path = shard_path(ckpt_dir, step, rank)
        tmp = path + ".tmp"
        stream = torch.cuda.Stream(device=store.device_index)
        bufs = [torch.empty(_CHUNK, dtype=torch.uint8).pin_memory() for _ in range(2)]
        events = [torch.cuda.Event(), torch.cuda.Event()]
        from .ftar import _CudaView
        regions = [torch.as_tensor(_CudaView(ptr, (n,), "|u1"), device=store.device)
                   for ptr, n in ((pp.value, pb.value), (mp.value, mb.value)) if n]
        try:
            with open(tmp, "wb") as fh:
                fh.write(MAGIC + _SHARD_HDR.pack(VERSION, step, rank, pb.value, mb.value))
                # double-buffered: chunk i+1 is copied while chunk i is written
                spans = [(r, off, min(_CHUNK, r.numel() - off)) for r in regions for off in range(0, r.numel(), _CHUNK)]

                def issue(i):
                    r, off, n = spans[i]
                    with torch.cuda.stream(stream):
                        bufs[i % 2][:n].copy_(r[off:off + n], non_blocking=True)
                        events[i % 2].record(stream)

                if spans:
                    issue(0)
                for i in range(len(spans)):
                    if i + 1 < len(spans):
                        issue(i + 1)  # its buffer's previous chunk was written to the file already
                    events[i % 2].synchronize()
                    fh.write(memoryview(bufs[i % 2].numpy())[:spans[i][2]])
                    if hook is not None:
                        hook(i)
                fh.flush()
                os.fsync(fh.fileno())
            seq1, step1 = C.c_uint64(), C.c_int64()
            _lib.check(_lib.lib.ftar_snap_region(store.handle, None, None, None, None, C.byref(seq1),
                                                 C.byref(step1)), "ftar_snap_region")
            if seq1.value != seq0.value:  # a capture ran while we copied: torn
                raise SnapshotUnavailable(None if step1.value < 0 else int(step1.value))
            os.rename(tmp, path)
        except BaseException:
            try:
                os.unlink(tmp)
            except OSError:
                pass
            raise
        box["path"] = path
    except BaseException as exc:  # noqa: BLE001 - surfaced by PersistJob.wait
        box["error"] = exc


def _persist(self, ckpt_dir: str, rank: int | None = None, background: bool = True, _hook=None) -> PersistJob:
    """Write the snapshot's step to ``ckpt_dir`` in the reference's shard
    format (§8f rank 4).  The device snapshot is streamed through two pinned
    64 MiB buffers on a side stream; the seqlock is checked after the copy,
    so a capture of the next step during the write yields
    SnapshotUnavailable instead of a torn file."""
    if self._snap is None:
        raise SnapshotUnavailable(None)
    rank = self.rank if rank is None else rank
    box: dict = {}
    if not background:
        _persist_snapshot(self, ckpt_dir, rank, box, _hook)
        return PersistJob(None, box)
    t = threading.Thread(target=_persist_snapshot, args=(self, ckpt_dir, rank, box, _hook),
                         name="ftar-snap-persist", daemon=True)
    t.start()
    return PersistJob(t, box)


SnapshotStore.persist = _persist
