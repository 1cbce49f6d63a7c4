"""Fault-tolerant all-reduce on B200 — drop-in for ``ftdp.ftar``.

Same entry points and failure contract as the reference
(pkg/src/ftdp/ftar.py): ``PipelineConfig``, ``build_partition_plan``,
``segment_bounds``, ``iter_chunks``, ``classify_error``, ``InflightMeter``,
``RingGroup(...).reconfig/close_links/links_ready`` and
``ftar_all_reduce(group, buf, step, cfg)`` which sums ``buf`` across the ring
in place and returns the same object.  Buffers are torch CUDA tensors; the data
plane is libftar_b200.so (sm_100a): members pull each other's buckets over
NVLink, reduce in the reference's fixed fold order (bit-identical to
tests/test_ftar.py:20-40) and commit all-or-nothing.

Extensions (keyword-only, reference callers never pass them):
``out=`` a separate fp32 output, which enables bf16 input buckets with the
bf16->fp32 cast fused into the reduction; ``scale=`` the normalisation factor
f32(1/(h*R)) of replica.py:622-626 fused into the same pass.

Failure semantics (ftar.py:5-16): a lost or slow member surfaces as
Recoverable (TIMEOUT / PEER_RESET / PEER_DOWN) with ``buf`` untouched and the
links closed; non-finite sums and protocol mismatches are Fatal, also with
``buf`` untouched on every member.
"""

from __future__ import annotations

import ctypes as C
from collections import deque
import logging
import os
import struct
import threading
from dataclasses import dataclass, field

import torch

from . import _lib
from .errors import (
    INTERNAL_INVARIANT,
    PEER_RESET,
    Fatal,
    FtdpError,
    Recoverable,
    from_status,
)
from .fabric import ArenaInfo, LocalFabric, StoreFabric

log = logging.getLogger(__name__)

ELEM = 4  # the reference's geometry is in float32 element units (ftar.py:46)
MIB = 1024 * 1024


# --------------------------------------------------------------- geometry


@dataclass
class PipelineConfig:
    """ftar.py:49-65.  On NVLink the chunk/window pair no longer paces a TCP
    link; it still defines the partition geometry, i.e. which member's copy
    starts each element's fold (and therefore the result bits)."""

    chunk_bytes: int = 8 * MIB
    max_in_flight: int = 4
    per_chunk_timeout_s: float = 5.0

    def __post_init__(self):
        if self.chunk_bytes < ELEM:
            raise Fatal(INTERNAL_INVARIANT, "chunk_bytes must be >= 4")
        if self.max_in_flight < 1:
            raise Fatal(INTERNAL_INVARIANT, "max_in_flight must be >= 1")
        if self.per_chunk_timeout_s <= 0:
            raise Fatal(INTERNAL_INVARIANT, "per_chunk_timeout_s must be > 0")

    @property
    def chunk_elems(self) -> int:
        return self.chunk_bytes // ELEM


@dataclass
class PartitionPlan:
    """Partition table in float32 element units (ftar.py:68-77)."""

    total_elems: int
    n_members: int
    partitions: list[tuple[int, int]]

    def partition_bytes(self) -> list[tuple[int, int]]:
        return [(o * ELEM, n * ELEM) for o, n in self.partitions]


def _balanced(total: int, parts: int) -> list[tuple[int, int]]:
    """`parts` contiguous (offset, length) pieces; the first total % parts
    pieces are one longer."""
    q, r = divmod(total, parts)
    out, off = [], 0
    for i in range(parts):
        n = q + (i < r)
        out.append((off, n))
        off += n
    return out


def build_partition_plan(total_bytes: int, cfg: PipelineConfig, n_members: int) -> PartitionPlan:
    """ftar.py:80-99: partitions of at most chunk_bytes*max_in_flight*n bytes."""
    if total_bytes % ELEM:
        raise Fatal(INTERNAL_INVARIANT, f"buffer not float32-aligned: {total_bytes}")
    if n_members < 1:
        raise Fatal(INTERNAL_INVARIANT, "n_members must be >= 1")
    total = total_bytes // ELEM
    if total == 0:
        return PartitionPlan(0, n_members, [(0, 0)])
    cap = max(1, cfg.chunk_bytes * cfg.max_in_flight * n_members // ELEM)
    return PartitionPlan(total, n_members, _balanced(total, -(-total // cap)))


def segment_bounds(part_elems: int, n: int) -> list[tuple[int, int]]:
    """ftar.py:102-112: segment j of a partition is owned by ring index j."""
    return _balanced(part_elems, n)


def iter_chunks(seg_len: int, chunk_elems: int) -> list[tuple[int, int, int]]:
    """ftar.py:115-125: (chunk_idx, offset, length) covering a segment."""
    return [(i, off, min(chunk_elems, seg_len - off))
            for i, off in enumerate(range(0, seg_len, chunk_elems))]


def classify_error(err: BaseException) -> str:
    """ftar.py:128-138."""
    if isinstance(err, FtdpError):
        return err.severity
    if isinstance(err, (TimeoutError, ConnectionError, BrokenPipeError, OSError)):
        return "recoverable"
    return "fatal"


class InflightMeter:
    """ftar.py:141-159.  On NVLink there is no ack window; the meter records,
    per call, the most bytes one peer link can have outstanding on the path
    the library takes (ftar_inflight_bound): the whole input for the small
    push one-shot, CTAs x (stages-1) x one tile for the bulk-copy
    reduce-scatter, CTAs x 512 threads x U 4-element vectors for the register
    path.  The kernel cannot exceed it; max_unacked_bytes is the largest."""

    def __init__(self):
        self.unacked_bytes = 0
        self.max_unacked_bytes = 0
        self.max_unacked_chunks = 0
        self._chunks = 0

    def sent(self, nbytes: int, chunks: int = 1) -> None:
        self.unacked_bytes += nbytes
        self._chunks += chunks
        self.max_unacked_bytes = max(self.max_unacked_bytes, self.unacked_bytes)
        self.max_unacked_chunks = max(self.max_unacked_chunks, self._chunks)

    def acked(self, nbytes: int, chunks: int = 1) -> None:
        self.unacked_bytes -= nbytes
        self._chunks -= chunks


@dataclass(frozen=True)
class PeerAddress:
    """transport.PeerAddress analogue: who a member is.  host/port are kept
    for signature compatibility; NVLink members are found through the fabric."""

    replica_id: int
    rank_id: int = 0
    host: str = ""
    port: int = 0


# --------------------------------------------------------------- tensors


class _CudaView:
    """__cuda_array_interface__ over a raw device range (arena pool)."""

    def __init__(self, ptr: int, shape: tuple, typestr: str):
        self.__cuda_array_interface__ = {
            "shape": shape, "typestr": typestr, "data": (ptr, False), "version": 3, "strides": None,
        }


_TYPESTR = {torch.float32: "<f4", torch.bfloat16: "<i2"}


def _f32(x: float) -> float:
    """Round to float32 (np.float32(x) semantics) without creating tensors."""
    return struct.unpack("f", struct.pack("f", x))[0]


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return _lib.DT_F32
    if t.dtype == torch.bfloat16:
        return _lib.DT_BF16
    raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be contiguous float32 (or bfloat16 with out=)")


# --------------------------------------------------------------- ring group


class RingGroup:
    """This rank's ring across replicas (ftar.py:162-235).

    Members are the quorum decision's replicas in ascending id order
    (ftar.py:202); ``generation`` strictly increases.  Instead of two TCP
    links, the group owns a device arena (result region, staging, registered
    pool, flag words) that the other members map, plus a pinned control block
    (live mask, contributor mask, epoch word, abort/progress/done words).

    ``router`` is the rendezvous fabric: a ``StoreFabric`` for one process per
    GPU, a ``LocalFabric`` (default) for members living in one process.
    """

    def __init__(self, self_replica: int, rank: int, router=None, plan=None, incarnation: int = 0,
                 *, device=None, max_bucket_bytes: int = 64 * MIB, pool_bytes: int = 0, keep_departed_gens: int = 4):
        if not torch.cuda.is_available():
            raise Fatal(INTERNAL_INVARIANT, "the B200 FTAR data plane needs a CUDA device")
        self.self_replica = self_replica
        self.rank = rank
        self.router = router if router is not None else LocalFabric.default()
        self.plan = plan
        self.incarnation = incarnation
        self.generation = 0
        self.members: list[int] = [self_replica]
        self.contributors: frozenset[int] = frozenset({self_replica})
        self.meter = InflightMeter()
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.device_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self._local = isinstance(self.router, LocalFabric)
        ctx = C.c_void_p()
        _lib.check(_lib.lib.ftar_ctx_create(self.device_index, max_bucket_bytes, pool_bytes,
                                            0 if self._local else 1, C.byref(ctx)), "ftar_ctx_create")
        self._ctx = ctx
        self.max_bucket_bytes = max_bucket_bytes
        self._links_up = False
        self._seq = 0
        # peer arena mappings by (replica, incarnation); slots come from a
        # free list and return to it when reconfig unmaps a departed member
        self._slots: dict[tuple[int, int], int] = {}
        self._free_slots: list[int] = list(range(255, -1, -1))
        self._absent: dict[tuple[int, int], int] = {}  # mapped but out of the ring since generation g
        self.keep_departed_gens = keep_departed_gens
        # registered user buffers: mine (rid -> tensor, kept alive) and the
        # peers' regions already mapped, by (replica, incarnation, rid, offset)
        self._regions: dict[int, torch.Tensor] = {}
        self._region_list: list[tuple] = []
        self._peer_regions: set = set()
        self._infos: dict = {}
        self._reg_round = 0
        self._pool_next = 0
        ptr, nbytes = C.c_uint64(), C.c_uint64()
        _lib.lib.ftar_ctx_pool(ctx, C.byref(ptr), C.byref(nbytes))
        self._pool_ptr, self._pool_bytes = ptr.value, nbytes.value
        self._lock = threading.Lock()
        self._pending: deque = deque()  # queued collectives, oldest first (PendingAllReduce)
        self._bound_cache: dict = {}
        if self._local:
            self.router.register(self)
        else:
            buf = (C.c_char * 64)()
            written = C.c_size_t()
            _lib.check(_lib.lib.ftar_ctx_export(ctx, buf, 64, C.byref(written)), "ftar_ctx_export")
            self.router.publish(ArenaInfo(self_replica, rank, incarnation, self.device_index,
                                          bytes(buf)[:written.value], 0, pid=os.getpid()))
        self._set_membership()

    # -- properties (ftar.py:180-186) ---------------------------------------
    @property
    def n(self) -> int:
        return len(self.members)

    @property
    def index(self) -> int:
        return self.members.index(self.self_replica)

    @property
    def ctx(self):
        return self._ctx

    # -- registered buckets ---------------------------------------------------
    def alloc_bucket(self, numel: int, dtype: torch.dtype = torch.float32) -> torch.Tensor:
        """A tensor inside the group's registered pool: reduced zero-copy
        (peers read it in place instead of a staged copy)."""
        esz = torch.empty((), dtype=dtype).element_size()
        nbytes = numel * esz
        off = (self._pool_next + 255) // 256 * 256
        if off + nbytes > self._pool_bytes:
            raise Fatal(INTERNAL_INVARIANT, f"bucket pool exhausted ({self._pool_bytes} bytes)")
        self._pool_next = off + nbytes
        view = _CudaView(self._pool_ptr + off, (numel,), _TYPESTR.get(dtype, "<f4"))
        with torch.cuda.device(self.device):
            t = torch.as_tensor(view, device=self.device)
        if dtype == torch.bfloat16:
            t = t.view(torch.bfloat16)
        t._ftar_owner = self  # keep the arena alive while the view is
        return t

    def reset_pool(self) -> None:
        self._pool_next = 0

    def register(self, t: torch.Tensor, deadline_s: float = 60.0) -> int:
        """Register an ordinary CUDA tensor (e.g. a caching-allocator gradient
        bucket) with the ring so its all-reduces run zero-copy: peers read it
        in place (no staging copy of an in-place call) and, as an ``out=``,
        write the all-gather straight into it.  The owning allocation block's
        IPC handle and the tensor's offset in it are published; every member
        maps every other member's registered buffers.

        A ring collective: every member calls it, in the same order, between
        reconfigs (like the reference's group operations).  A member that
        (re)joins later registers before its reconfig; reconfig exchanges all
        members' registrations.  The tensor is kept alive until ``close``.
        Returns this member's region id."""
        if self._local:
            return -1
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.is_contiguous()):
            raise Fatal(INTERNAL_INVARIANT, "register needs a contiguous CUDA tensor")
        if t.device.index != self.device_index:
            raise Fatal(INTERNAL_INVARIANT, f"tensor on {t.device}, ring group on cuda:{self.device_index}")
        rid, off = C.c_int(-1), C.c_uint64()
        h = (C.c_char * 64)()
        nbytes = t.numel() * t.element_size()
        _lib.check(_lib.lib.ftar_region_register(self._ctx, t.data_ptr(), nbytes, C.byref(rid), h, 64, C.byref(off)),
                   "ftar_region_register")
        self._regions[rid.value] = t
        self._region_list = [r for r in self._region_list if r[0] != rid.value] + \
            [(rid.value, bytes(h)[:64], off.value, nbytes)]
        self.router.publish_regions(self.rank, self.self_replica, self.incarnation, self._region_list)
        if self.n > 1 and self._links_up:
            self._reg_round += 1
            self.router.region_round(self.rank, self.self_replica, self.members, self.generation,
                                     self._reg_round, deadline_s)
            self._import_regions()
        return rid.value

    def _import_regions(self) -> None:
        for m in self.members:
            if m == self.self_replica or m not in self._infos:
                continue
            inc = self._infos[m].incarnation
            slot = self._slot(m, inc)
            for rid, handle, off, nbytes in self.router.lookup_regions(self.rank, m, inc):
                key = (m, inc, rid, off, handle)
                if key in self._peer_regions:
                    continue
                rc = _lib.lib.ftar_region_import(self._ctx, slot, rid, handle, len(handle), off, nbytes)
                if rc:
                    _lib.check(rc, f"map registered buffer {rid} of replica {m}")
                self._peer_regions.add(key)

    # -- membership (ftar.py:188-235) ---------------------------------------
    def _slot(self, replica_id: int, incarnation: int) -> int:
        key = (replica_id, incarnation)
        if key not in self._slots:
            if not self._free_slots:
                raise Fatal(INTERNAL_INVARIANT, "no free peer-arena slots (256 mapped)")
            self._slots[key] = self._free_slots.pop()
        return self._slots[key]

    def _release_stale(self, keep: set) -> None:
        """Unmap peer arenas that are not in `keep` (the current ring), so a
        dead incarnation does not stay pinned in its GPU's memory
        (close_links, ftar.py:226-230): at once when the replica rejoined as
        a newer incarnation (the old process is gone), otherwise once it has
        been out of the ring for ``keep_departed_gens`` generations — a
        replica parked for a few steps keeps its mapping, so re-admitting it
        costs no IPC re-map (46-870 ms for a multi-GB arena, config 5).  Its
        registered buffers are unmapped with it."""
        current = {r: inc for r, inc in keep}
        for key in list(self._slots):
            if key in keep:
                self._absent.pop(key, None)
                continue
            rid, inc = key
            first = self._absent.setdefault(key, self.generation)
            superseded = rid in current and current[rid] != inc
            if superseded or self.generation - first >= self.keep_departed_gens:
                slot = self._slots.pop(key)
                self._absent.pop(key, None)
                _lib.check(_lib.lib.ftar_ctx_unmap(self._ctx, slot), f"unmap arena of replica {rid}")
                self._free_slots.append(slot)
                self._peer_regions = {r for r in self._peer_regions if (r[0], r[1]) != key}

    @property
    def mapped_peers(self) -> list[tuple[int, int]]:
        """(replica, incarnation) of every peer arena currently mapped."""
        return sorted(self._slots)

    def _set_membership(self, infos: dict | None = None) -> None:
        n = self.n
        slots = (C.c_int * n)()
        for i, m in enumerate(self.members):
            if m == self.self_replica or self._local:
                slots[i] = -1
            else:
                slots[i] = self._slot(m, infos[m].incarnation)
        contrib = 0
        for i, m in enumerate(self.members):
            if m in self.contributors:
                contrib |= 1 << i
        if self._local:
            # in-process members are addressed directly by the launch
            slots_arg = None
            rc = _lib.lib.ftar_set_membership(self._ctx, slots_arg, 1, 0, contrib & 1 if n == 1 else 1,
                                              self.generation)
            self._contrib_mask = contrib
        else:
            rc = _lib.lib.ftar_set_membership(self._ctx, slots, n, self.index, contrib, self.generation)
            self._contrib_mask = contrib
        _lib.check(rc, "ftar_set_membership")

    def reconfig(self, addrs: dict, generation: int, deadline_s: float = 5.0,
                 contributors=None) -> None:
        """Tear down the old ring and establish the new one (ftar.py:188-224).

        ``addrs`` maps member replica ids to addresses and must include self.
        ``contributors`` (default: all members) are the replicas whose data
        enters the sum; the rest (the quorum's *behind* set, replica.py:574-577)
        fold +0.0 and issue no loads.  Unreachable members surface as
        Recoverable(PEER_DOWN)."""
        if generation <= self.generation:
            raise Fatal(INTERNAL_INVARIANT, f"generation must increase: {generation} <= {self.generation}")
        if self.self_replica not in addrs:
            raise Fatal(INTERNAL_INVARIANT, "reconfig membership must include self")
        if generation > 0xFFFFFF:
            raise Fatal(INTERNAL_INVARIANT, "generation exceeds the 24-bit epoch word")
        if self._ctx and not self._local:
            _drain_pending(self)  # collectives queued under the old membership never complete
        self.close_links()
        self.members = sorted(addrs)
        self.generation = generation
        self._seq = 0
        self.contributors = frozenset(self.members if contributors is None else contributors)
        if not self.contributors <= set(self.members):
            raise Fatal(INTERNAL_INVARIANT, "contributors must be ring members")
        if len(self.members) > 8:
            raise Fatal(INTERNAL_INVARIANT, "at most 8 replicas per NVLink ring")
        infos = None
        if self.n > 1:
            infos = self.router.join(self.rank, self.self_replica, self.members, generation, deadline_s)
            if not self._local:
                for m, info in infos.items():
                    rc = _lib.lib.ftar_ctx_import(self._ctx, self._slot(m, info.incarnation), info.handle,
                                                  len(info.handle), info.arena_bytes)
                    if rc:
                        self.close_links()
                        _lib.check(rc, f"map arena of replica {m}")
        self._set_membership(infos)
        if not self._local:
            keep = {(m, infos[m].incarnation) for m in self.members if m != self.self_replica} if infos else set()
            self._release_stale(keep)
            self._infos = dict(infos) if infos else {}
            self._reg_round = 0
            if self.n > 1:
                self._import_regions()  # every member published its registrations before joining
        self._links_up = True

    def close_links(self) -> None:
        """ftar.py:226-230: the ring is unusable until the next reconfig;
        members waiting on this one are released with PEER_RESET."""
        if self._links_up and self.n > 1:
            self.router.mark_down(self.rank, self.self_replica, self.generation)
        self._links_up = False

    def links_ready(self) -> bool:
        return self.n == 1 or self._links_up

    def close(self) -> None:
        self.close_links()
        if self._ctx:
            if self._local:
                self.router.unregister(self)
            _lib.lib.ftar_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter teardown
            pass

    def inflight_bound(self, nelems: int, dtype_code: int, cfg: "PipelineConfig", push: bool = False) -> tuple[int, int]:
        """(bytes, CTAs) one peer link can have outstanding for this call, on
        the path the library takes for it (ftar_inflight_bound: small push
        one-shot / bulk-copy reduce-scatter / register path)."""
        if self.n < 2:
            return 0, 0
        key = (self.n, nelems, dtype_code, cfg.chunk_bytes, cfg.max_in_flight, push)
        cache = self._bound_cache
        if key not in cache:
            b, g, path = C.c_uint64(), C.c_int(), C.c_int()
            _lib.check(_lib.lib.ftar_inflight_bound(self.n, nelems, dtype_code, cfg.chunk_bytes,
                                                    cfg.max_in_flight, int(push), C.byref(b), C.byref(g),
                                                    C.byref(path)),
                       "ftar_inflight_bound")
            if len(cache) > 64:
                cache.clear()
            cache[key] = (b.value, g.value)
        return cache[key]


# --------------------------------------------------------------- all-reduce


def _check_buffers(buf, out, device=None):
    if not isinstance(buf, torch.Tensor) or not buf.is_cuda:
        raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be a CUDA tensor")
    if device is not None and buf.device.index != device:
        # the kernel runs on the group's GPU: another GPU's tensor would be
        # read through a peer mapping that may not exist
        raise Fatal(INTERNAL_INVARIANT, f"buffer on {buf.device}, ring group on cuda:{device}")
    if not buf.is_contiguous():
        raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be contiguous float32")
    code = _dtype_code(buf)
    if out is None:
        if code != _lib.DT_F32:
            raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be contiguous float32 (pass out= for bf16)")
        out = buf
    else:
        if not isinstance(out, torch.Tensor) or not out.is_cuda or out.dtype != torch.float32 \
                or not out.is_contiguous() or out.numel() != buf.numel() or out.device != buf.device:
            raise Fatal(INTERNAL_INVARIANT, "out must be a contiguous float32 CUDA tensor shaped like buf")
    return code, out


def ftar_all_reduce(group: RingGroup, buf: torch.Tensor, step: int, cfg: PipelineConfig | None = None,
                    *, out: torch.Tensor | None = None, scale: float | None = None) -> torch.Tensor:
    """Sum ``buf`` across the group (ftar.py:301-326).

    In place for float32 (returns ``buf``); with ``out=`` the fp32 sum (of a
    float32 or bfloat16 bucket) lands in ``out`` and ``out`` is returned.
    ``scale`` multiplies the fp32 sum by f32(scale) in the same pass.  On a
    Recoverable error the links are closed and nothing has been written."""
    cfg = cfg or PipelineConfig()
    if not (isinstance(buf, torch.Tensor) and buf.is_cuda):
        return _host_all_reduce(group, buf, step, cfg, out, scale)
    code, dst = _check_buffers(buf, out, group.device_index)
    if group.n > 1 and not group.links_ready():
        raise Recoverable(PEER_RESET, "ring links not established")
    flags = _lib.F_SCALE if scale is not None else 0
    f_scale = _f32(scale) if scale is not None else 1.0
    bound, ctas = group.inflight_bound(buf.numel(), code, cfg, dst.data_ptr() != buf.data_ptr())
    try:
        if group._local:
            _local_all_reduce(group, buf, dst, code, cfg, f_scale, flags)
        else:
            _remote_all_reduce(group, buf, dst, code, cfg, f_scale, flags)
    except FtdpError:
        group.close_links()
        raise
    group.meter.sent(bound, ctas)
    group.meter.acked(bound, ctas)
    return dst


class PendingAllReduce:
    """A queued collective (ftar_all_reduce_async).  wait() collects it —
    and every earlier one of the same group, in launch order — and raises the
    taxonomy exception of its status (the links are then closed, as in
    ftar.py:323-325)."""

    __slots__ = ("group", "result", "cfg", "status", "detail", "done", "_keep")

    def __init__(self, group, result, cfg):
        self.group, self.result, self.cfg = group, result, cfg
        self.status, self.detail, self.done = 0, -1, False
        self._keep = None  # buffers that must outlive the queued call

    def wait(self):
        q = self.group._pending
        while not self.done:
            head = q.popleft()
            det = C.c_int(-1)
            head.status = _lib.lib.ftar_wait(self.group.ctx, head.cfg.per_chunk_timeout_s, C.byref(det))
            head.detail, head.done = det.value, True
            if head.status:
                # the step is lost: abort and collect everything queued behind
                # the failed bucket so the host and device queues stay in step
                _drain_pending(self.group)
        if self.status:
            self.group.close_links()
            blame = self.group.members[self.detail] if 0 <= self.detail < self.group.n else None
            msg = _lib.last_error() if self.status == 10 else ""
            raise from_status(self.status, (msg + f" (peer replica {blame})") if blame is not None else msg)
        return self.result


def _drain_pending(group) -> None:
    """Abort every queued collective of `group` and collect its status (each
    pending handle keeps its own: ABORTED, or OK if it had already finished)."""
    q = group._pending
    if not q:
        return
    _lib.lib.ftar_abort(group.ctx)
    while q:
        p = q.popleft()
        det = C.c_int(-1)
        p.status = _lib.lib.ftar_wait(group.ctx, p.cfg.per_chunk_timeout_s, C.byref(det))
        p.detail, p.done = det.value, True


def ftar_all_reduce_async(group: RingGroup, buf: torch.Tensor, step: int, cfg: PipelineConfig | None = None,
                          *, out: torch.Tensor | None = None, scale: float | None = None) -> PendingAllReduce:
    """Enqueue one all-reduce on the current stream and return at once (up to
    4 per group in flight; the GPU runs queued buckets back to back, as a
    bucketed backward pass would issue them).  Same semantics as
    ftar_all_reduce once .wait() returns."""
    cfg = cfg or PipelineConfig()
    if group._local or not (isinstance(buf, torch.Tensor) and buf.is_cuda):
        p = PendingAllReduce(group, ftar_all_reduce(group, buf, step, cfg, out=out, scale=scale), cfg)
        p.done = True
        return p
    code, dst = _check_buffers(buf, out, group.device_index)
    if group.n > 1 and not group.links_ready():
        raise Recoverable(PEER_RESET, "ring links not established")
    q = group._pending
    while len(q) >= 4:
        q[0].wait()
    flags = _lib.F_SCALE if scale is not None else 0
    f_scale = _f32(scale) if scale is not None else 1.0
    rc = _lib.lib.ftar_allreduce_launch(group.ctx, buf.data_ptr(), code, dst.data_ptr(), buf.numel(),
                                        cfg.chunk_bytes, cfg.max_in_flight, f_scale, flags,
                                        _stream_ptr(group.device))
    _lib.check(rc, "ftar_allreduce_launch")
    p = PendingAllReduce(group, dst, cfg)
    q.append(p)
    bound, ctas = group.inflight_bound(buf.numel(), code, cfg, dst.data_ptr() != buf.data_ptr())
    group.meter.sent(bound, ctas)
    group.meter.acked(bound, ctas)
    return p


def ftar_all_reduce_sgd(group: RingGroup, grad: torch.Tensor, step: int, cfg: PipelineConfig | None = None, *,
                        params: torch.Tensor, momentum: torch.Tensor, lr: float, beta: float,
                        scale: float | None = None, params_out: torch.Tensor | None = None,
                        momentum_out: torch.Tensor | None = None, grad_out: torch.Tensor | None = None):
    """the all-reduce with normalisation and the
    SGD-momentum step fused in.  g = sum x f32(scale) (replica.py:622-626);
    m' = f32(m * f32(beta)) + g; p' = p - f32(f32(lr) * m') (model.py:146-155),
    every fp32 op separately rounded.  Out of place: params/momentum are
    never modified (the reference applies the optimizer only after its commit
    vote, replica.py:616-633); returns (params_out, momentum_out).  grad_out
    (optional, must not alias grad) receives g."""
    return ftar_all_reduce_sgd_async(group, grad, step, cfg, params=params, momentum=momentum, lr=lr, beta=beta,
                                     scale=scale, params_out=params_out, momentum_out=momentum_out,
                                     grad_out=grad_out).wait()


def ftar_all_reduce_sgd_async(group: RingGroup, grad: torch.Tensor, step: int, cfg: PipelineConfig | None = None,
                              *, params: torch.Tensor, momentum: torch.Tensor, lr: float, beta: float,
                              scale: float | None = None, params_out: torch.Tensor | None = None,
                              momentum_out: torch.Tensor | None = None,
                              grad_out: torch.Tensor | None = None) -> PendingAllReduce:
    """ftar_all_reduce_sgd, enqueued (the same queue as ftar_all_reduce_async:
    up to 4 buckets per group in flight, collected in launch order); .wait()
    returns (params_out, momentum_out)."""
    cfg = cfg or PipelineConfig()
    if group._local:
        raise Fatal(INTERNAL_INVARIANT, "in-process groups: use LocalRing.all_reduce_sgd")
    if not (isinstance(grad, torch.Tensor) and grad.is_cuda and grad.is_contiguous()):
        raise Fatal(INTERNAL_INVARIANT, "gradient bucket must be a contiguous CUDA tensor")
    code = _dtype_code(grad)
    if grad_out is not None:
        _check_buffers(grad, grad_out, group.device_index)
    for t in (grad, params, momentum):
        if t.device.index != group.device_index:
            raise Fatal(INTERNAL_INVARIANT, f"tensor on {t.device}, ring group on cuda:{group.device_index}")
    for t in (params, momentum):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() == grad.numel()):
            raise Fatal(INTERNAL_INVARIANT, "params/momentum must be contiguous fp32 CUDA tensors shaped like grad")
    params_out = torch.empty_like(params) if params_out is None else params_out
    momentum_out = torch.empty_like(momentum) if momentum_out is None else momentum_out
    if group.n > 1 and not group.links_ready():
        raise Recoverable(PEER_RESET, "ring links not established")
    q = group._pending
    while len(q) >= 4:
        q[0].wait()
    flags = _lib.F_SCALE if scale is not None else 0
    f_scale = _f32(scale) if scale is not None else 1.0
    rc = _lib.lib.ftar_allreduce_sgd_launch(
        group.ctx, grad.data_ptr(), code, grad_out.data_ptr() if grad_out is not None else None, grad.numel(),
        cfg.chunk_bytes, cfg.max_in_flight, f_scale, flags, params.data_ptr(), momentum.data_ptr(),
        params_out.data_ptr(), momentum_out.data_ptr(), _f32(lr), _f32(beta), _stream_ptr(group.device))
    try:
        _lib.check(rc, "ftar_allreduce_sgd_launch")
    except FtdpError:
        group.close_links()
        raise
    p = PendingAllReduce(group, (params_out, momentum_out), cfg)
    p._keep = (grad, params, momentum, grad_out)
    q.append(p)
    return p


def _host_all_reduce(group, buf, step, cfg, out, scale):
    """Host (numpy / CPU tensor) buffers: the reference's exact call shape.
    One process per GPU: chunked H2D / range all-reduce / D2H pipeline.
    In-process (threaded) rings: stage through the device whole."""
    host = _as_host_tensor(buf)
    if host.dtype not in (torch.float32, torch.bfloat16):
        raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be contiguous float32")
    if out is None and host.dtype != torch.float32:
        raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be contiguous float32 (pass out= for bf16)")
    hout = _as_host_tensor(out) if out is not None else None
    if group.n > 1 and not group.links_ready():
        raise Recoverable(PEER_RESET, "ring links not established")
    q = group._pending
    while q:
        q[0].wait()
    if group._local:
        dev = host.to(group.device)
        dres = torch.empty(host.numel(), device=group.device) if out is not None else None
        ftar_all_reduce(group, dev, step, cfg, out=dres, scale=scale)
        (hout if hout is not None else host).copy_((dres if dres is not None else dev).cpu())
        return out if out is not None else buf
    pipe = group.__dict__.get("_pipe")
    if pipe is None or pipe.key != (1, host.dtype, 8 << 20):
        pipe = group._pipe = _HostPipeline(group.device, 1, host.dtype, 8 << 20)
    flags = _lib.F_SCALE if scale is not None else 0
    f_scale = _f32(scale) if scale is not None else 1.0
    code = _dtype_code(host)

    def launch(dins, douts, base, total):
        rc = _lib.lib.ftar_allreduce_launch_range(group.ctx, dins[0].data_ptr(), code, douts[0].data_ptr(),
                                                  dins[0].numel(), base, total, cfg.chunk_bytes, cfg.max_in_flight,
                                                  f_scale, flags, _stream_ptr(group.device))
        _lib.check(rc, "ftar_allreduce_launch_range")
        return None

    def wait(_tok):
        det = C.c_int(-1)
        st = _lib.lib.ftar_wait(group.ctx, cfg.per_chunk_timeout_s, C.byref(det))
        if st:
            raise from_status(st, _lib.last_error() if st == 10 else "")

    try:
        pipe.run([host], [hout] if hout is not None else None, launch, wait)
    except FtdpError:
        group.close_links()
        raise
    return out if out is not None else buf


def _remote_all_reduce(group, buf, dst, code, cfg, f_scale, flags):
    q = group._pending
    while q:
        q[0].wait()
    with group._lock:
        group._seq += 1
        rc = _lib.lib.ftar_allreduce_launch(group.ctx, buf.data_ptr(), code, dst.data_ptr(), buf.numel(),
                                            cfg.chunk_bytes, cfg.max_in_flight, f_scale, flags,
                                            _stream_ptr(group.device))
        _lib.check(rc, "ftar_allreduce_launch")
        detail = C.c_int(-1)
        st = _lib.lib.ftar_wait(group.ctx, cfg.per_chunk_timeout_s, C.byref(detail))
    if st:
        blame = group.members[detail.value] if 0 <= detail.value < group.n else None
        msg = _lib.last_error() if st == 10 else ""
        raise from_status(st, (msg + f" (peer replica {blame})") if blame is not None else msg)


def _local_all_reduce(group, buf, dst, code, cfg, f_scale, flags):
    fabric: LocalFabric = group.router
    group._seq += 1
    key = (group.rank, group.generation, group._seq)
    params = (buf.numel(), code, cfg.chunk_bytes, cfg.max_in_flight, flags, f_scale, str(buf.device))
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(group.device))
    deposit = {"buf": buf, "out": dst, "event": ev, "timeout": cfg.per_chunk_timeout_s}

    def launch(call):
        members = call.members
        n = len(members)
        groups = [fabric.group_of(group.rank, m) for m in members]
        stream = torch.cuda.current_stream(group.device)
        for i in range(n):
            stream.wait_event(call.deposits[i]["event"])
        fault_member, fault_after = -1, 0
        with fabric.cond:
            for i, m in enumerate(members):
                if (group.rank, m) in fabric.faults:
                    fault_member, fault_after = i, fabric.faults.pop((group.rank, m))
        ctxs = (C.c_void_p * n)(*[g.ctx for g in groups])
        ins = (C.c_void_p * n)(*[call.deposits[i]["buf"].data_ptr() for i in range(n)])
        outs = (C.c_void_p * n)(*[call.deposits[i]["out"].data_ptr() for i in range(n)])
        contrib = groups[0]._contrib_mask if n > 1 else 1
        lflags = flags | (_lib.F_PROTOCOL if _local_protocol() else 0)
        rc = _lib.lib.ftar_local_allreduce_launch(ctxs, n, ins, code, outs, buf.numel(), cfg.chunk_bytes,
                                                  cfg.max_in_flight, f_scale, lflags, contrib, fault_member,
                                                  fault_after, stream.cuda_stream)
        _lib.check(rc, "ftar_local_allreduce_launch")
        sts = (C.c_int * n)()
        dets = (C.c_int * n)()
        timeout = min(call.deposits[i]["timeout"] for i in range(n))
        _lib.check(_lib.lib.ftar_wait_local(ctxs, n, timeout, sts, dets), "ftar_wait_local")
        return {i: (sts[i], dets[i]) for i in range(n)}

    st, det = fabric.rendezvous(group, key, deposit, params, cfg.per_chunk_timeout_s, launch)
    if st:
        blame = group.members[det] if 0 <= det < group.n else None
        raise from_status(st, f"peer replica {blame}" if blame is not None else "")


def _as_host_tensor(b) -> torch.Tensor:
    if isinstance(b, torch.Tensor):
        if b.is_cuda:
            raise Fatal(INTERNAL_INVARIANT, "expected a host buffer")
        return b
    import numpy as np
    if isinstance(b, np.ndarray):
        if not b.flags.c_contiguous:
            raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be contiguous float32")
        return torch.from_numpy(b)
    raise Fatal(INTERNAL_INVARIANT, "all-reduce buffer must be a tensor or numpy array")


class _HostPipeline:
    """Double-buffered device staging for host-buffer all-reduces: chunk c+1
    is copied in while chunk c is reduced and chunk c-1 is copied out."""

    def __init__(self, device: torch.device, n: int, dtype: torch.dtype, chunk_elems: int):
        self.key = (n, dtype, chunk_elems)
        self.device = device
        self.chunk = chunk_elems
        self.din = [[torch.empty(chunk_elems, dtype=dtype, device=device) for _ in range(n)] for _ in range(2)]
        self.dout = [[torch.empty(chunk_elems, dtype=torch.float32, device=device) for _ in range(n)]
                     for _ in range(2)]
        self.h2d = torch.cuda.Stream(device=device)
        self.d2h = torch.cuda.Stream(device=device)
        self.staging = None

    def run(self, hosts, outs, launch, wait):
        n = len(hosts)
        total = hosts[0].numel()
        inplace = outs is None
        if inplace:
            if hosts[0].dtype != torch.float32:
                raise Fatal(INTERNAL_INVARIANT, "in-place host all-reduce needs float32 (pass outs=)")
            if self.staging is None or self.staging[0].numel() < total or len(self.staging) != n:
                self.staging = [torch.empty(total, dtype=torch.float32).pin_memory() for _ in range(n)]
            dsts = [t[:total] for t in self.staging]
        else:
            dsts = outs
        comp = torch.cuda.current_stream(self.device)
        nchunks = max(1, -(-total // self.chunk))
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_comp = [torch.cuda.Event() for _ in range(2)]
        ev_out = [None, None]

        def stage_in(c):
            slot, off = c % 2, c * self.chunk
            ln = min(self.chunk, total - off)
            with torch.cuda.stream(self.h2d):
                for i in range(n):
                    self.din[slot][i][:ln].copy_(hosts[i][off:off + ln], non_blocking=True)
                ev_in[slot].record(self.h2d)

        stage_in(0)
        for c in range(nchunks):
            slot, off = c % 2, c * self.chunk
            ln = min(self.chunk, total - off)
            comp.wait_event(ev_in[slot])
            if ev_out[slot] is not None:
                comp.wait_event(ev_out[slot])
            tok = launch([t[:ln] for t in self.din[slot]], [t[:ln] for t in self.dout[slot]], off, total)
            ev_comp[slot].record(comp)
            if c + 1 < nchunks:
                stage_in(c + 1)  # overlaps the reduction of chunk c
            wait(tok)            # one collective in flight per ring group
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(ev_comp[slot])
                for i in range(n):
                    dsts[i][off:off + ln].copy_(self.dout[slot][i][:ln], non_blocking=True)
                ev_out[slot] = torch.cuda.Event()
                ev_out[slot].record(self.d2h)
        self.d2h.synchronize()
        if inplace:
            for h, st in zip(hosts, dsts):
                h.copy_(st)
            return hosts
        return outs


def _local_protocol() -> bool:
    """In-process rings run the one-shot kernel unless FTAR_LOCAL_MODE=protocol
    asks for the two-shot flag protocol (what one GPU per member runs)."""
    return os.environ.get("FTAR_LOCAL_MODE", "oneshot") == "protocol"


class LocalRing:
    """n single-rank members of one ring in this process, on one device —
    the B200 counterpart of ``bench._LoopbackRing`` (bench.py:53-96).
    ``all_reduce`` issues the members' calls without threads (one cooperative
    launch), which is what the benchmark times.  ``protocol=True`` runs the
    two-shot flag-protocol kernel (the multi-GPU kernel, members as CTA
    groups); the default one-shot kernel needs no inter-member waits."""

    def __init__(self, n: int, device=None, max_bucket_bytes: int = 64 * MIB, rank: int = 0,
                 protocol: bool | None = None):
        self.n = n
        self.protocol = _local_protocol() if protocol is None else protocol
        self.fabric = LocalFabric()
        self.groups = [RingGroup(rid, rank, self.fabric, device=device, max_bucket_bytes=max_bucket_bytes)
                       for rid in range(n)]
        self.gen = 0
        self.reconfig()

    def reconfig(self, members=None, contributors=None):
        members = sorted(members if members is not None else range(self.n))
        self.gen += 1
        addrs = {m: PeerAddress(m) for m in members}
        errs = []
        threads = [threading.Thread(target=self._rc, args=(self.groups[m], addrs, contributors, errs))
                   for m in members]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errs:
            raise errs[0]
        return members

    def _rc(self, g, addrs, contributors, errs):
        try:
            g.reconfig(addrs, self.gen, deadline_s=10.0, contributors=contributors)
        except Exception as exc:  # noqa: BLE001
            errs.append(exc)

    def launch(self, bufs, cfg: PipelineConfig | None = None, outs=None, scale=None, members=None,
               fault=None, base: int = 0, total: int | None = None):
        """Launch one all-reduce over `members` (default all) without waiting.
        With base/total the buffers hold elements [base, base+len) of a bucket
        of `total` elements and fold with that bucket's geometry."""
        cfg = cfg or PipelineConfig()
        members = sorted(members if members is not None else range(self.n))
        groups = [self.groups[m] for m in members]
        n = len(groups)
        code = _dtype_code(bufs[0])
        outs = outs if outs is not None else bufs
        flags = _lib.F_SCALE if scale is not None else 0
        f_scale = _f32(scale) if scale is not None else 1.0
        for g in groups:
            g._seq += 1
        ctxs = (C.c_void_p * n)(*[g.ctx for g in groups])
        ins = (C.c_void_p * n)(*[bufs[i].data_ptr() for i in range(n)])
        ous = (C.c_void_p * n)(*[outs[i].data_ptr() for i in range(n)])
        fm, fa = (-1, 0) if fault is None else fault
        if self.protocol or fault is not None:
            flags |= _lib.F_PROTOCOL
        ln = bufs[0].numel()
        rc = _lib.lib.ftar_local_allreduce_launch_range(ctxs, n, ins, code, ous, ln, base,
                                                        ln + base if total is None else total, cfg.chunk_bytes,
                                                        cfg.max_in_flight, f_scale, flags, groups[0]._contrib_mask,
                                                        fm, fa, _stream_ptr(groups[0].device))
        _lib.check(rc, "ftar_local_allreduce_launch")
        return ctxs

    def wait(self, ctxs, cfg: PipelineConfig | None = None) -> list[int]:
        cfg = cfg or PipelineConfig()
        n = len(ctxs)
        sts = (C.c_int * n)()
        dets = (C.c_int * n)()
        _lib.check(_lib.lib.ftar_wait_local(ctxs, n, cfg.per_chunk_timeout_s, sts, dets), "ftar_wait_local")
        return list(sts)

    def all_reduce(self, bufs, cfg: PipelineConfig | None = None, outs=None, scale=None, members=None):
        sts = self.wait(self.launch(bufs, cfg, outs, scale, members), cfg)
        for st in sts:
            if st:
                raise from_status(st)
        return outs if outs is not None else bufs

    def all_reduce_host(self, host_bufs, cfg: PipelineConfig | None = None, outs=None, scale=None,
                        chunk_elems: int = 8 << 20):
        """The reference call shape with HOST buffers (bench._LoopbackRing
        .timed_all_reduce on numpy arrays): chunked H2D -> range all-reduce ->
        D2H, pipelined on three streams so both PCIe directions and the
        kernel overlap.  outs (fp32 host) default to the inputs (in place:
        results are committed only once every chunk succeeded)."""
        cfg = cfg or PipelineConfig()
        hosts = [_as_host_tensor(b) for b in host_bufs]
        n = len(hosts)
        pipe = self.__dict__.get("_pipe")
        if pipe is None or pipe.key != (n, hosts[0].dtype, chunk_elems):
            pipe = self._pipe = _HostPipeline(self.groups[0].device, n, hosts[0].dtype, chunk_elems)

        def launch(dins, douts, base, total):
            return self.launch(dins, cfg, outs=douts, scale=scale, base=base, total=total)

        def wait(tok):
            for st in self.wait(tok, cfg):
                if st:
                    raise from_status(st)

        return pipe.run(hosts, [_as_host_tensor(o) for o in outs] if outs is not None else None, launch, wait)

    def all_reduce_sgd(self, bufs, cfg: PipelineConfig | None = None, *, params, momenta, lr: float, beta: float,
                       scale=None, params_out=None, momenta_out=None, grad_outs=None):
        """In-process form of ftar_all_reduce_sgd (protocol kernel): every
        member's (params, momentum) updated out of place with its reduced,
        scaled gradient."""
        cfg = cfg or PipelineConfig()
        n = len(bufs)
        groups = self.groups[:n]
        code = _dtype_code(bufs[0])
        params_out = params_out if params_out is not None else [torch.empty_like(t) for t in params]
        momenta_out = momenta_out if momenta_out is not None else [torch.empty_like(t) for t in momenta]
        flags = _lib.F_SCALE if scale is not None else 0
        f_scale = _f32(scale) if scale is not None else 1.0
        for g in groups:
            g._seq += 1
        arr = lambda ts: (C.c_void_p * n)(*[t.data_ptr() if t is not None else None for t in ts])  # noqa: E731
        ctxs = (C.c_void_p * n)(*[g.ctx for g in groups])
        rc = _lib.lib.ftar_local_allreduce_sgd_launch(
            ctxs, n, arr(bufs), code, arr(grad_outs if grad_outs is not None else [None] * n), bufs[0].numel(),
            cfg.chunk_bytes, cfg.max_in_flight, f_scale, flags, groups[0]._contrib_mask, arr(params), arr(momenta),
            arr(params_out), arr(momenta_out), _f32(lr), _f32(beta), _stream_ptr(groups[0].device))
        _lib.check(rc, "ftar_local_allreduce_sgd_launch")
        for st in self.wait(ctxs, cfg):
            if st:
                raise from_status(st)
        return params_out, momenta_out

    def close(self):
        for g in self.groups:
            g.close()


class DeviceRing:
    """n members of one ring on n GPUs driven by ONE process (peer access
    instead of CUDA IPC): member i lives on devices[i].  Same kernel and flag
    protocol as one process per GPU; the members' kernels run concurrently
    on their own GPUs.  Used for single-process multi-GPU jobs and tuning."""

    def __init__(self, devices, max_bucket_bytes: int = 64 * MIB, generation: int = 1):
        self.devices = [torch.device("cuda", d) if isinstance(d, int) else torch.device(d) for d in devices]
        self.n = len(self.devices)
        self.ctxs = []
        for d in self.devices:
            ctx = C.c_void_p()
            _lib.check(_lib.lib.ftar_ctx_create(d.index, max_bucket_bytes, 0, 0, C.byref(ctx)), "ftar_ctx_create")
            self.ctxs.append(ctx)
        for i, c in enumerate(self.ctxs):
            for j, o in enumerate(self.ctxs):
                if i != j:
                    _lib.check(_lib.lib.ftar_ctx_link_local(c, j, o), "ftar_ctx_link_local")
        self.generation = 0
        self.reconfig(generation)

    def reconfig(self, generation: int, contributors=None):
        if generation <= self.generation:
            raise Fatal(INTERNAL_INVARIANT, "generation must increase")
        self.generation = generation
        contrib = sum(1 << i for i in range(self.n) if contributors is None or i in contributors)
        for i, c in enumerate(self.ctxs):
            slots = (C.c_int * self.n)(*[-1 if j == i else j for j in range(self.n)])
            _lib.check(_lib.lib.ftar_set_membership(c, slots, self.n, i, contrib, generation),
                       "ftar_set_membership")

    def launch(self, bufs, cfg: PipelineConfig | None = None, outs=None, scale=None):
        cfg = cfg or PipelineConfig()
        outs = outs if outs is not None else bufs
        flags = _lib.F_SCALE if scale is not None else 0
        f_scale = _f32(scale) if scale is not None else 1.0
        for i, c in enumerate(self.ctxs):
            rc = _lib.lib.ftar_allreduce_launch(c, bufs[i].data_ptr(), _dtype_code(bufs[i]), outs[i].data_ptr(),
                                                bufs[i].numel(), cfg.chunk_bytes, cfg.max_in_flight, f_scale, flags,
                                                _stream_ptr(self.devices[i]))
            _lib.check(rc, "ftar_allreduce_launch")

    def wait(self, cfg: PipelineConfig | None = None) -> list[int]:
        cfg = cfg or PipelineConfig()
        out = []
        for c in self.ctxs:
            det = C.c_int(-1)
            out.append(_lib.lib.ftar_wait(c, cfg.per_chunk_timeout_s, C.byref(det)))
        return out

    def all_reduce(self, bufs, cfg: PipelineConfig | None = None, outs=None, scale=None):
        self.launch(bufs, cfg, outs, scale)
        for st in self.wait(cfg):
            if st:
                raise from_status(st)
        return outs if outs is not None else bufs

    def phase_us(self, i: int = 0):
        t = (C.c_uint64 * 6)()
        _lib.lib.ftar_phase_times(self.ctxs[i], t, 6)
        t = list(t)
        names = ["entry_wait", "reduce_scatter", "rs_to_ag_barrier", "all_gather"]
        return {k: round((t[j + 1] - t[j]) / 1e3, 1) for j, k in enumerate(names) if t[j + 1] >= t[j] > 0}

    def close(self):
        for c in self.ctxs:
            _lib.lib.ftar_ctx_destroy(c)
        self.ctxs = []
