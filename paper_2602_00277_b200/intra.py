"""Intra-replica collectives on B200 — drop-in for ``replica.IntraGroup``
(pkg/src/ftdp/replica.py:203-262), SURVEY §8f rank 2.

An HSDP replica spans R ranks (one GPU each).  Before FTAR, the ranks
reduce-scatter their full gradients so that rank r holds the sum of shard r
(the FTAR input, replica.py:573); after the optimizer step they all-gather
params and momentum (replica.py:640-644).  The reference runs the ranks as
threads over one slot array; here the data moves GPU to GPU over NVLink in
``intra_kernel`` (csrc/ftar_b200.cu) behind ``ftar_intra_launch``:

* ``reduce_scatter(rank, vec, bounds)`` -> rank r's fp32 shard
  ``vec_0[b_r] + vec_1[b_r] + ... + vec_{R-1}[b_r]``, folded rank 0 upward on
  every rank (replica.py:247-249, tests/test_replica.py:71-86), bit-exact;
  bf16 vectors are upcast exactly.
* ``all_gather(rank, shard, bounds, total)`` -> the full fp32 vector.
* ``broadcast`` / ``exchange`` / ``abort``: the control-plane helpers of the
  same class (Python objects; not data plane).

Two shapes:

* ``IntraGroup(n_ranks)`` — the reference's: one object shared by the R rank
  threads of a process.  The ranks' buffers live on one device (the ranks are
  emulated as CTA groups of one cooperative launch); this is what the
  reference-shaped tests drive.
* ``IntraRank(rank, n_ranks, fabric)`` — production: one process per GPU,
  arenas mapped over CUDA IPC through a Store rendezvous (use a Store
  namespace per replica, e.g. ``StoreFabric(PrefixStore(f"intra/{rid}", s))``).

Both return numpy arrays for numpy inputs (the reference's types) and CUDA
tensors for CUDA tensors.  A completed call guarantees every rank finished
reading this rank's input (the reference's second barrier wait).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _lib
from .errors import INTERNAL_INVARIANT, PEER_DOWN, Fatal, Recoverable, from_status
from .fabric import LocalFabric
from .ftar import MIB, PeerAddress, PendingAllReduce, PipelineConfig, RingGroup, _stream_ptr, segment_bounds

__all__ = ["IntraGroup", "IntraRank", "segment_bounds"]


def _bounds_arrays(bounds, n: int, total: int):
    if len(bounds) != n:
        raise Fatal(INTERNAL_INVARIANT, f"need {n} shard bounds, got {len(bounds)}")
    offs = (C.c_uint64 * n)(*[int(o) for o, _ in bounds])
    lens = (C.c_uint64 * n)(*[int(ln) for _, ln in bounds])
    for o, ln in bounds:
        if o < 0 or ln < 0 or o + ln > total:
            raise Fatal(INTERNAL_INVARIANT, "shard bounds exceed the vector")
    return offs, lens


def _as_device(x, device, dtypes=(torch.float32, torch.bfloat16)):
    """(device tensor, was_numpy)."""
    if isinstance(x, np.ndarray):
        if x.dtype != np.float32:
            raise Fatal(INTERNAL_INVARIANT, "intra-replica vectors must be float32")
        return torch.from_numpy(np.ascontiguousarray(x)).to(device), True
    if not isinstance(x, torch.Tensor):
        raise Fatal(INTERNAL_INVARIANT, "expected a numpy array or a torch tensor")
    if x.dtype not in dtypes:
        raise Fatal(INTERNAL_INVARIANT, f"unsupported dtype {x.dtype}")
    return x.to(device).contiguous(), False


def _raise(st: int, detail: int, members) -> None:
    if st:
        blame = members[detail] if 0 <= detail < len(members) else None
        msg = _lib.last_error() if st == 10 else ""
        raise from_status(st, (msg + f" (rank {blame})") if blame is not None else msg)


class IntraGroup:
    """The R ranks of one replica in this process (replica.py:203-262)."""

    def __init__(self, n_ranks: int, device=None, max_bytes: int = 64 * MIB):
        if not 1 <= n_ranks <= 8:
            raise Fatal(INTERNAL_INVARIANT, "1..8 ranks per replica")
        self.n = n_ranks
        self._barrier = threading.Barrier(n_ranks)
        self._slots: list = [None] * n_ranks
        self._res: list = [None] * n_ranks
        self._err = None
        self.fabric = LocalFabric()
        self.groups = [RingGroup(r, 0, self.fabric, device=device, max_bucket_bytes=max_bytes)
                       for r in range(n_ranks)]
        self.device = self.groups[0].device
        errs: list = []

        def rc(g):
            try:
                g.reconfig({r: PeerAddress(r) for r in range(n_ranks)}, 1, deadline_s=10.0)
            except Exception as exc:  # noqa: BLE001
                errs.append(exc)

        ts = [threading.Thread(target=rc, args=(g,)) for g in self.groups]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]

    # --- control-plane helpers (replica.py:217-239) -----------------------------
    def _sync(self) -> None:
        try:
            self._barrier.wait()
        except threading.BrokenBarrierError as exc:
            raise Recoverable(PEER_DOWN, "intra-replica group aborted") from exc

    def abort(self) -> None:
        self._barrier.abort()

    def broadcast(self, rank: int, value=None):
        if rank == 0:
            self._slots[0] = value
        self._sync()
        out = self._slots[0]
        self._sync()
        return out

    def exchange(self, rank: int, value) -> list:
        self._slots[rank] = value
        self._sync()
        out = list(self._slots)
        self._sync()
        return out

    # --- data plane ---------------------------------------------------------------
    def _collective(self, rank: int, op: int, x, bounds, total: int, out_len):
        self._slots[rank] = x
        self._sync()
        if rank == 0:
            self._err = None
            try:
                self._res = self._launch(op, list(self._slots), bounds, total)
            except Exception as exc:  # noqa: BLE001 - every rank raises it
                self._err = exc
        self._sync()
        if self._err is not None:
            raise self._err
        return self._res[rank]

    def _launch(self, op: int, xs, bounds, total: int):
        n, dev = self.n, self.device
        ins, was_np = zip(*[_as_device(x, dev, (torch.float32, torch.bfloat16) if op == _lib.OP_RS
                                       else (torch.float32,)) for x in xs])
        dtypes = {t.dtype for t in ins}
        if len(dtypes) != 1:
            raise Fatal(INTERNAL_INVARIANT, "ranks disagree on the vector dtype")
        code = _lib.DT_BF16 if ins[0].dtype == torch.bfloat16 else _lib.DT_F32
        offs, lens = _bounds_arrays(bounds, n, total)
        if op == _lib.OP_RS:
            for t in ins:
                if t.numel() != total:
                    raise Fatal(INTERNAL_INVARIANT, "every rank passes the full vector")
            outs = [torch.empty(int(bounds[r][1]), device=dev) for r in range(n)]
        else:
            for r, t in enumerate(ins):
                if t.numel() != int(bounds[r][1]):
                    raise Fatal(INTERNAL_INVARIANT, f"rank {r}'s shard does not match its bounds")
            outs = [torch.empty(total, device=dev) for _ in range(n)]
        ctxs = (C.c_void_p * n)(*[g.ctx for g in self.groups])
        pin = (C.c_void_p * n)(*[t.data_ptr() for t in ins])
        pout = (C.c_void_p * n)(*[t.data_ptr() for t in outs])
        rc = _lib.lib.ftar_local_intra_launch(ctxs, n, op, pin, code, pout, total, offs, lens, _stream_ptr(dev))
        _lib.check(rc, "ftar_local_intra_launch")
        sts, dets = (C.c_int * n)(), (C.c_int * n)()
        _lib.check(_lib.lib.ftar_wait_local(ctxs, n, 30.0, sts, dets), "ftar_wait_local")
        for r in range(n):
            _raise(sts[r], dets[r], list(range(n)))
        return [o.cpu().numpy() if was_np[r] else o for r, o in enumerate(outs)]

    def reduce_scatter(self, rank: int, vec, bounds) -> np.ndarray | torch.Tensor:
        """Sum over ranks, each rank keeping its own shard; the fold runs rank
        0 upward on every rank (replica.py:241-252)."""
        total = int(vec.numel() if isinstance(vec, torch.Tensor) else vec.size)
        return self._collective(rank, _lib.OP_RS, vec, bounds, total, None)

    def all_gather(self, rank: int, shard, bounds, total: int) -> np.ndarray | torch.Tensor:
        """Every rank's shard placed at its bounds (replica.py:254-262)."""
        return self._collective(rank, _lib.OP_AG, shard, bounds, int(total), None)

    def close(self) -> None:
        for g in self.groups:
            g.close()


class IntraRank:
    """One rank of a replica's intra group, one process per GPU.

    ``fabric`` must be private to this replica's ranks (a Store namespace per
    replica).  ``reconfig(generation)`` re-forms the group after a failure;
    a rank that died surfaces as ``Recoverable`` on the others."""

    def __init__(self, rank: int, n_ranks: int, fabric, device=None, max_bytes: int = 64 * MIB,
                 pool_bytes: int = 0, incarnation: int = 0, deadline_s: float = 30.0):
        if isinstance(fabric, LocalFabric):
            raise Fatal(INTERNAL_INVARIANT, "IntraRank needs a Store fabric; use IntraGroup in-process")
        self.rank, self.n = rank, n_ranks
        self.group = RingGroup(rank, 0, fabric, incarnation=incarnation, device=device,
                               max_bucket_bytes=max_bytes, pool_bytes=pool_bytes)
        self._cfg = PipelineConfig(per_chunk_timeout_s=30.0)
        self.device = self.group.device
        self.reconfig(1, deadline_s)

    def reconfig(self, generation: int, deadline_s: float = 30.0) -> None:
        self.group.reconfig({r: PeerAddress(r) for r in range(self.n)}, generation, deadline_s=deadline_s)

    def alloc(self, numel: int, dtype: torch.dtype = torch.float32) -> torch.Tensor:
        """A buffer in the registered pool: read by the peers in place."""
        return self.group.alloc_bucket(numel, dtype)

    def _run(self, op: int, x, bounds, total: int, out, wait: bool = True):
        if not self.group.links_ready():
            raise Recoverable(PEER_DOWN, "intra-replica links not established")
        t, was_np = _as_device(x, self.device, (torch.float32, torch.bfloat16) if op == _lib.OP_RS
                               else (torch.float32,))
        code = _lib.DT_BF16 if t.dtype == torch.bfloat16 else _lib.DT_F32
        offs, lens = _bounds_arrays(bounds, self.n, total)
        want = int(bounds[self.rank][1]) if op == _lib.OP_RS else total
        if op == _lib.OP_RS and t.numel() != total:
            raise Fatal(INTERNAL_INVARIANT, "reduce_scatter takes the full vector")
        if op == _lib.OP_AG and t.numel() != int(bounds[self.rank][1]):
            raise Fatal(INTERNAL_INVARIANT, "all_gather takes this rank's shard")
        if out is None:
            out = torch.empty(want, device=self.device)
        elif not (out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and out.numel() == want):
            raise Fatal(INTERNAL_INVARIANT, f"out must be a contiguous fp32 CUDA tensor of {want} elements")
        # shares the group's FIFO of queued collectives (up to 4 in flight)
        q = self.group._pending
        while len(q) >= 4:
            q[0].wait()
        rc = _lib.lib.ftar_intra_launch(self.group.ctx, op, t.data_ptr(), code, out.data_ptr(), total, offs, lens,
                                        _stream_ptr(self.device))
        _lib.check(rc, "ftar_intra_launch")
        pend = PendingAllReduce(self.group, out, self._cfg)
        pend._keep = t  # the input must outlive the call (staged copy or peers' reads)
        q.append(pend)
        if not wait:
            return pend
        res = pend.wait()
        return res.cpu().numpy() if was_np else res

    def reduce_scatter(self, rank: int, vec, bounds, *, out=None):
        if rank != self.rank:
            raise Fatal(INTERNAL_INVARIANT, "IntraRank serves its own rank only")
        total = int(vec.numel() if isinstance(vec, torch.Tensor) else vec.size)
        return self._run(_lib.OP_RS, vec, bounds, total, out)

    def all_gather(self, rank: int, shard, bounds, total: int, *, out=None):
        if rank != self.rank:
            raise Fatal(INTERNAL_INVARIANT, "IntraRank serves its own rank only")
        return self._run(_lib.OP_AG, shard, bounds, int(total), out)

    def reduce_scatter_async(self, vec: torch.Tensor, bounds, *, out=None) -> PendingAllReduce:
        """Queue a reduce-scatter (CUDA tensors); .wait() returns the shard.
        Queued calls run back to back on the stream (programmatic dependent
        launch overlaps each one's entry with the previous one's tail)."""
        return self._run(_lib.OP_RS, vec, bounds, int(vec.numel()), out, wait=False)

    def all_gather_async(self, shard: torch.Tensor, bounds, total: int, *, out=None) -> PendingAllReduce:
        return self._run(_lib.OP_AG, shard, bounds, int(total), out, wait=False)

    def close(self) -> None:
        self.group.close()
