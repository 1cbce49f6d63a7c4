"""Member rendezvous for the FTAR data plane.

In the reference each rank's ring is a pair of TCP connections: dial the right
neighbour with HELLO_RING(generation), accept the left one through the
ConnectionRouter, discarding hellos of older generations
(pkg/src/ftdp/ftar.py:206-224, transport.py:330-409).  On the B200 box the
data moves by NVLink loads from the members' arenas, so what a member needs at
reconfig time is (a) every member's arena mapping and (b) proof that every
member joined the same generation.  Two fabrics provide that:

* ``StoreFabric`` — one process per GPU.  Arena IPC handles and per-generation
  join marks live in a key/value store (``torch.distributed.TCPStore`` or any
  object with ``set/get/wait``); ``join`` times out into Recoverable(PEER_DOWN)
  exactly where the reference's accept would.
* ``LocalFabric`` — all members of a ring in one process on one device (the
  reference's ``bench._LoopbackRing`` / test ``Ring``, bench.py:53-88 and
  tests/test_ftar.py:112-170).  Members rendezvous per call and the last one
  to arrive issues a single cooperative launch over all of them (kernels that
  wait on one another must be co-resident on one GPU).

Neither fabric carries payload; they are the control plane's side channel.
"""

from __future__ import annotations

import pickle
import threading
import time
from dataclasses import dataclass, field
from datetime import timedelta

from .errors import PEER_DOWN, PEER_RESET, TIMEOUT, Recoverable


@dataclass(frozen=True)
class ArenaInfo:
    """What a member publishes about itself (the HELLO_RING payload analogue)."""

    replica_id: int
    rank: int
    incarnation: int
    device: int
    handle: bytes
    arena_bytes: int
    host: str = ""
    pid: int = 0


class StoreFabric:
    """Rendezvous through a key/value store shared by the member processes."""

    kind = "store"

    def __init__(self, store, prefix: str = "ftar"):
        self.store = store
        self.prefix = prefix

    def _k(self, *parts) -> str:
        return "/".join([self.prefix, *map(str, parts)])

    # -- publication ------------------------------------------------------
    def publish(self, info: ArenaInfo, what: str = "arena") -> None:
        self.store.set(self._k(what, info.rank, info.replica_id), pickle.dumps(info))

    def lookup(self, rank: int, replica_id: int, deadline_s: float, what: str = "arena") -> ArenaInfo:
        key = self._k(what, rank, replica_id)
        self._wait([key], deadline_s, f"{what} of replica {replica_id}")
        return pickle.loads(self.store.get(key))

    def _wait(self, keys: list[str], deadline_s: float, what: str) -> None:
        try:
            self.store.wait(keys, timedelta(seconds=max(0.01, deadline_s)))
        except Exception as exc:  # c10d raises DistStoreError / RuntimeError on timeout
            raise Recoverable(PEER_DOWN, f"{what} not published within {deadline_s:.2f}s: {exc}")

    # -- per-generation join (dial right / accept left) -------------------
    def join(self, rank: int, replica_id: int, members: list[int], generation: int,
             deadline_s: float) -> dict[int, ArenaInfo]:
        t_end = time.monotonic() + deadline_s
        self.store.set(self._k("join", rank, generation, replica_id), b"1")
        keys = [self._k("join", rank, generation, m) for m in members]
        self._wait(keys, deadline_s, f"generation {generation} join")
        out = {}
        for m in members:
            if m == replica_id:
                continue
            down = self._down_gen(rank, m)
            if down is not None and down >= generation:
                raise Recoverable(PEER_RESET, f"replica {m} closed its links at generation {down}")
            out[m] = self.lookup(rank, m, max(0.01, t_end - time.monotonic()))
        return out

    def _down_gen(self, rank: int, replica_id: int):
        key = self._k("down", rank, replica_id)
        if self.store.check([key]):
            return int(self.store.get(key))
        return None

    def mark_down(self, rank: int, replica_id: int, generation: int) -> None:
        self.store.set(self._k("down", rank, replica_id), str(generation).encode())

    # -- registered buffers (RingGroup.register) ------------------------------
    def publish_regions(self, rank: int, replica_id: int, incarnation: int, regions: list) -> None:
        """This member's registered buffers: [(rid, handle, offset, bytes)]."""
        self.store.set(self._k("regions", rank, replica_id, incarnation), pickle.dumps(regions))

    def lookup_regions(self, rank: int, replica_id: int, incarnation: int) -> list:
        key = self._k("regions", rank, replica_id, incarnation)
        return pickle.loads(self.store.get(key)) if self.store.check([key]) else []

    def region_round(self, rank: int, replica_id: int, members: list[int], generation: int, k: int,
                     deadline_s: float) -> None:
        """The k-th register() of this generation: every member has published."""
        self.store.set(self._k("regrnd", rank, generation, k, replica_id), b"1")
        self._wait([self._k("regrnd", rank, generation, k, m) for m in members], deadline_s,
                   f"register round {k} of generation {generation}")


@dataclass
class _Call:
    """One in-process all-reduce rendezvous (every member deposits its buffer)."""

    members: tuple
    deposits: dict = field(default_factory=dict)
    params: tuple | None = None
    launched: bool = False
    failed: Exception | None = None
    results: dict | None = None
    done: threading.Event = field(default_factory=threading.Event)


class LocalFabric:
    """All members of a ring in one process, on one device."""

    kind = "local"
    _default = None
    _default_lock = threading.Lock()

    def __init__(self):
        self.cond = threading.Condition()
        self.groups: dict[tuple[int, int], object] = {}
        self.joins: dict[tuple[int, int], set] = {}
        self.down: dict[tuple[int, int], int] = {}
        self.calls: dict[tuple, _Call] = {}
        self.faults: dict[tuple[int, int], int] = {}

    @classmethod
    def default(cls) -> "LocalFabric":
        with cls._default_lock:
            if cls._default is None:
                cls._default = cls()
            return cls._default

    def register(self, group) -> None:
        with self.cond:
            self.groups[(group.rank, group.self_replica)] = group

    def unregister(self, group) -> None:
        with self.cond:
            self.groups.pop((group.rank, group.self_replica), None)

    def group_of(self, rank: int, replica_id: int):
        return self.groups.get((rank, replica_id))

    # -- per-generation join ----------------------------------------------
    def join(self, rank: int, replica_id: int, members: list[int], generation: int,
             deadline_s: float) -> dict[int, object]:
        t_end = time.monotonic() + deadline_s
        with self.cond:
            self.down.pop((rank, replica_id), None)
            self.joins.setdefault((rank, generation), set()).add(replica_id)
            self.cond.notify_all()
            while True:
                joined = self.joins.get((rank, generation), set())
                missing = [m for m in members if m not in joined]
                if not missing:
                    break
                left = t_end - time.monotonic()
                if left <= 0:
                    self.joins[(rank, generation)].discard(replica_id)
                    raise Recoverable(PEER_DOWN, f"members {missing} never joined generation {generation}")
                self.cond.wait(timeout=min(left, 0.05))
            return {m: self.groups[(rank, m)] for m in members if m != replica_id}

    def mark_down(self, rank: int, replica_id: int, generation: int) -> None:
        with self.cond:
            self.down[(rank, replica_id)] = generation
            self.cond.notify_all()

    def inject_fault(self, rank: int, replica_id: int, after_tiles: int) -> None:
        """Test hook: replica stops after `after_tiles` reduce tiles of its next call."""
        with self.cond:
            self.faults[(rank, replica_id)] = after_tiles

    # -- per-call rendezvous ------------------------------------------------
    def rendezvous(self, group, key: tuple, deposit: dict, params: tuple, timeout_s: float,
                   launch) -> dict:
        """Deposit this member's buffers for call `key`; the last member to
        arrive runs ``launch(call)`` (one cooperative kernel for all) and
        everyone receives its own status.  A member that never arrives turns
        into Recoverable(TIMEOUT) after `timeout_s` (ftar.py:382-386); a member
        that closes its links turns into Recoverable(PEER_RESET)."""
        rank, gen = key[0], key[1]
        with self.cond:
            call = self.calls.get(key)
            if call is None:
                call = self.calls[key] = _Call(members=tuple(group.members))
            if call.failed is not None:
                raise call.failed
            if call.params is None:
                call.params = params
            elif call.params != params:
                from .errors import PROTOCOL_VIOLATION, Fatal
                err = Fatal(PROTOCOL_VIOLATION, f"members disagree on the call: {call.params} vs {params}")
                call.failed = err
                self.cond.notify_all()
                raise err
            call.deposits[group.index] = deposit
            launcher = len(call.deposits) == len(call.members)
            if launcher:
                call.launched = True
            else:
                t_end = time.monotonic() + timeout_s
                while not call.launched and call.failed is None:
                    dead = [m for m in call.members
                            if self.down.get((rank, m), -1) >= gen and m != group.self_replica]
                    if dead:
                        call.failed = Recoverable(PEER_RESET, f"replica {dead[0]} closed its links")
                        break
                    left = t_end - time.monotonic()
                    if left <= 0:
                        missing = [m for i, m in enumerate(call.members) if i not in call.deposits]
                        call.failed = Recoverable(TIMEOUT, f"chunk never arrived: members {missing} absent")
                        break
                    self.cond.wait(timeout=min(left, 0.02))
                if call.failed is not None and not call.launched:
                    self.calls.pop(key, None)
                    self.cond.notify_all()
                    raise call.failed
        if launcher:
            try:
                call.results = launch(call)
            except Exception as exc:  # noqa: BLE001 - delivered to every member
                call.failed = exc
            finally:
                with self.cond:
                    self.calls.pop(key, None)
                    call.done.set()
                    self.cond.notify_all()
        else:
            call.done.wait()
        if call.failed is not None:
            raise call.failed
        return call.results[group.index]
