"""Step agreement and group membership — drop-in for ``ftdp.quorum``'s
decision engine (pkg/src/ftdp/quorum.py:49-210).

This is the CPU control plane that feeds the data plane: every decision
becomes the ring's membership (``members`` = healthy + behind, ascending id),
its contributor set (``healthy``; behind replicas fold +0.0,
replica.py:574-577), its normalisation factor f32(1/(|healthy|*R))
(replica.py:622-626) and its epoch word (``generation``), which
``RingGroup.reconfig`` writes into the pinned control block the kernels check.

Semantics are the reference's, restated:
* target = max reported next_step over admissible reports, never below the
  previously issued target (a lost frontier parks everyone as behind);
* healthy = reporters at the target, behind = live reporters below it;
* generation += 1 whenever the (healthy, behind) roles change or the target
  fails to advance (a retry), so stale traffic is fenced;
* stale incarnations are ignored; scheduled rejoiners stay parked until the
  ungated group reaches their admission step.
The TCP coordinator/client (quorum.py:213-441) is transport, not data plane,
and is out of scope; ``StoreQuorum`` below runs the same engine over the
rendezvous store for multi-process runs.
"""

from __future__ import annotations

import json
import logging
import time
from dataclasses import dataclass
from datetime import timedelta

import numpy as np

from .errors import PEER_DOWN, Recoverable

log = logging.getLogger(__name__)


@dataclass(frozen=True)
class Decision:
    epoch: int
    target_step: int
    generation: int
    healthy: tuple[int, ...]
    behind: dict[int, int]

    @property
    def members(self) -> tuple[int, ...]:
        return tuple(sorted(set(self.healthy) | set(self.behind)))

    def role_of(self, replica_id: int) -> str:
        if replica_id in self.healthy:
            return "healthy"
        if replica_id in self.behind:
            return "behind"
        return "unassigned"

    # --- data-plane words ---------------------------------------------------
    def live_mask(self) -> int:
        """Bit i set for ring index i (all members)."""
        return (1 << len(self.members)) - 1

    def contrib_mask(self) -> int:
        """Bit i set when ring index i is healthy (contributes data)."""
        return sum(1 << i for i, m in enumerate(self.members) if m in self.healthy)

    def scale(self, ranks_per_replica: int = 1, normalize_by: str = "healthy",
              num_replicas: int | None = None) -> float:
        """f32(1/denom) with denom = |healthy|*R (or num_replicas*R)."""
        h = len(self.healthy) if normalize_by == "healthy" else num_replicas
        return float(np.float32(1.0 / (h * ranks_per_replica)))

    def to_json(self) -> dict:
        return {"epoch": self.epoch, "target_step": self.target_step, "generation": self.generation,
                "healthy": list(self.healthy), "behind": {str(k): v for k, v in self.behind.items()}}

    @classmethod
    def from_json(cls, d: dict) -> "Decision":
        return cls(d["epoch"], d["target_step"], d["generation"], tuple(sorted(d["healthy"])),
                   {int(k): v for k, v in d["behind"].items()})


@dataclass
class Report:
    next_step: int
    incarnation: int


class QuorumEngine:
    """Pure decision logic (quorum.py:84-210)."""

    def __init__(self):
        self.epoch = 0
        self.target_step = 0
        self.generation = 0
        self._incarnations: dict[int, int] = {}
        self._gates: dict[int, list[tuple[int, int]]] = {}  # rid -> sorted [(step, min_inc)]
        self._prev_roles = None

    # --- incarnations and admission gates ------------------------------------
    def register(self, replica_id: int, incarnation: int) -> bool:
        if incarnation < self._incarnations.get(replica_id, -1):
            return False
        self._incarnations[replica_id] = incarnation
        return True

    def admit_after(self, replica_id: int, not_before_step: int, min_incarnation: int = 0) -> None:
        gates = self._gates.setdefault(replica_id, [])
        gates.append((not_before_step, min_incarnation))
        gates.sort()

    def admission_gate(self, replica_id: int):
        gates = self._gates.get(replica_id)
        return gates[0][0] if gates else None

    def drop_admission(self, replica_id: int) -> None:
        gates = self._gates.get(replica_id)
        if gates:
            gates.pop(0)
            if not gates:
                del self._gates[replica_id]

    def _binding_gate(self, replica_id: int, incarnation: int):
        steps = [s for s, floor in self._gates.get(replica_id, ()) if incarnation >= floor]
        return max(steps) if steps else None

    def effective_reports(self, reports: dict[int, Report]) -> dict[int, Report]:
        fresh = {}
        for rid, rep in reports.items():
            if rep.incarnation < self._incarnations.get(rid, -1):
                continue  # fenced: an older incarnation of a re-registered replica
            self.register(rid, rep.incarnation)
            fresh[rid] = rep
        gate = {rid: self._binding_gate(rid, rep.incarnation) for rid, rep in fresh.items()}
        frontier = max((rep.next_step for rid, rep in fresh.items() if gate[rid] is None), default=0)
        return {rid: rep for rid, rep in fresh.items() if gate[rid] is None or gate[rid] <= frontier}

    def prospective_target(self, reports: dict[int, Report]) -> int:
        eff = self.effective_reports(reports)
        return max((r.next_step for r in eff.values()), default=self.target_step)

    def pending_joiners(self, reports: dict[int, Report]) -> set[int]:
        target = self.prospective_target(reports)
        eff = self.effective_reports(reports)
        return {rid for rid, gates in self._gates.items() if gates[0][0] <= target and rid not in eff}

    # --- state hand-over (StoreQuorum coordinator failover) ----------------------
    def state(self) -> dict:
        """Everything decide() depends on, JSON-serialisable."""
        return {"epoch": self.epoch, "target": self.target_step, "gen": self.generation,
                "inc": {str(k): v for k, v in self._incarnations.items()},
                "gates": {str(k): [list(g) for g in v] for k, v in self._gates.items()},
                "prev": None if self._prev_roles is None else [list(self._prev_roles[0]), list(self._prev_roles[1])]}

    def load_state(self, st: dict) -> None:
        self.epoch, self.target_step, self.generation = st["epoch"], st["target"], st["gen"]
        self._incarnations = {int(k): v for k, v in st["inc"].items()}
        self._gates = {int(k): [tuple(g) for g in v] for k, v in st["gates"].items()}
        self._prev_roles = None if st["prev"] is None else (tuple(st["prev"][0]), tuple(st["prev"][1]))

    # --- the decision ----------------------------------------------------------
    def decide(self, reports: dict[int, Report]) -> Decision:
        self.epoch += 1
        eff = self.effective_reports(reports)
        if not eff:
            return Decision(self.epoch, self.target_step, self.generation, (), {})
        target = max(self.target_step, max(r.next_step for r in eff.values()))
        if target > max(r.next_step for r in eff.values()):
            log.warning("quorum: frontier %d is ahead of every live report; holding", target)
        healthy = tuple(sorted(rid for rid, r in eff.items() if r.next_step == target))
        behind = {rid: eff[rid].next_step for rid in sorted(eff) if eff[rid].next_step < target}
        roles = (healthy, tuple(sorted(behind)))
        if roles != self._prev_roles or target <= self.target_step:
            self.generation += 1
        self._prev_roles = roles
        self.target_step = target
        for rid in (*healthy, *behind):
            gates = self._gates.get(rid)
            if gates:
                inc = self._incarnations.get(rid, 0)
                keep = [(s, floor) for s, floor in gates if floor > inc]
                if keep:
                    self._gates[rid] = keep
                else:
                    del self._gates[rid]
        return Decision(self.epoch, target, self.generation, healthy, behind)


class StoreQuorum:
    """One membership round over the rendezvous store (multi-process runs).

    Every live replica posts ``Report(next_step, incarnation)`` for round
    ``round_id``; ONE replica, the round's coordinator, plays the reference's
    coordinator process (quorum.py:213-441): it collects reports until all of
    the world posted, every replica that has not posted is dead, or
    ``round_deadline_s`` passed; runs ``QuorumEngine.decide``; and publishes
    the Decision together with the engine's state; everyone else reads it and
    adopts that state.  Replicas that miss the deadline are absent from that
    round, exactly like the reference's round deadline (quorum.py:354-396).
    A single decider matters: a replica that posts early and decides from its
    own partial view would publish a competing decision for the same round.

    Liveness (``start_heartbeat``): each replica refreshes a heartbeat key
    every ``hb_period_s``.  A replica whose heartbeat is older than
    ``liveness_s`` is dead: the coordinator stops waiting for its report (an
    outage round ends as soon as the live replicas have posted), and when the
    coordinator itself — or a vote's decider — is dead, the lowest live
    replica takes over the round.  Decisions and vote outcomes are published
    first-writer-wins (``compare_set``), so a take-over can never publish a
    second, different answer.  Without heartbeats the coordinator is the
    lowest id (default) and rounds last until everyone posted or the deadline."""

    def __init__(self, store, world: list[int], prefix: str = "ftar/quorum", coordinator: int | None = None,
                 liveness_s: float = 1.0):
        self.store = store
        self.world = sorted(world)
        self.prefix = prefix
        self.coordinator = self.world[0] if coordinator is None else coordinator
        if self.coordinator not in self.world:
            raise ValueError("coordinator must be a member of the world")
        self.engine = QuorumEngine()
        self.liveness_s = liveness_s
        self._hb_stop = None

    def _k(self, *p) -> str:
        return "/".join([self.prefix, *map(str, p)])

    # --- liveness ----------------------------------------------------------------
    def start_heartbeat(self, replica_id: int, period_s: float = 0.1) -> None:
        """Refresh this replica's heartbeat key from a daemon thread."""
        import threading
        self.stop_heartbeat()
        stop = threading.Event()
        key = self._k("hb", replica_id)

        def beat():
            while not stop.is_set():
                try:
                    self.store.set(key, repr(time.time()).encode())
                except Exception:  # noqa: BLE001 - store gone: the process is shutting down
                    return
                stop.wait(period_s)

        self.store.set(key, repr(time.time()).encode())
        t = threading.Thread(target=beat, name=f"quorum-hb-{replica_id}", daemon=True)
        t.start()
        self._hb_stop = stop

    def stop_heartbeat(self) -> None:
        if self._hb_stop is not None:
            self._hb_stop.set()
            self._hb_stop = None

    def alive(self, replica_id: int):
        """True / False from the heartbeat; None when the replica never beat."""
        key = self._k("hb", replica_id)
        if not self.store.check([key]):
            return None
        return time.time() - float(self.store.get(key)) < self.liveness_s

    def _dead(self, replica_id: int) -> bool:
        return self.alive(replica_id) is False

    def _acting(self, preferred: int, candidates) -> int:
        """`preferred` unless it is dead; then the lowest live candidate."""
        if not self._dead(preferred):
            return preferred
        for rid in sorted(candidates):
            if not self._dead(rid):
                return rid
        return preferred

    def _publish_once(self, key: str, value: bytes) -> bytes:
        """First writer wins; returns what the key holds afterwards."""
        try:
            return self.store.compare_set(key, b"", value)
        except Exception:  # noqa: BLE001 - a store without compare_set
            if not self.store.check([key]):
                self.store.set(key, value)
            return self.store.get(key)

    # --- the round -----------------------------------------------------------------
    def _coordinate(self, round_id: int, t_end: float) -> Decision:
        reports: dict[int, Report] = {}
        while True:
            for rid in self.world:
                if rid not in reports and self.store.check([self._k(round_id, "report", rid)]):
                    ns, inc = json.loads(self.store.get(self._k(round_id, "report", rid)))
                    reports[rid] = Report(ns, inc)
            missing = [rid for rid in self.world if rid not in reports]
            if not missing or time.monotonic() >= t_end or all(self._dead(rid) for rid in missing):
                break
            time.sleep(0.002)
        d = self.engine.decide(reports)
        doc = json.dumps({"decision": d.to_json(), "state": self.engine.state()}).encode()
        won = self._publish_once(self._k(round_id, "decision"), doc)
        return self._adopt(won)

    def _adopt(self, raw: bytes) -> Decision:
        doc = json.loads(raw)
        if "decision" not in doc:  # a decision without state (older writer)
            d = Decision.from_json(doc)
            self._follow(d)
            return d
        d = Decision.from_json(doc["decision"])
        self.engine.load_state(doc["state"])
        return d

    def exchange(self, round_id: int, replica_id: int, report: Report, round_deadline_s: float = 2.0,
                 decide_timeout_s: float = 30.0) -> Decision:
        self.store.set(self._k(round_id, "report", replica_id),
                       json.dumps([report.next_step, report.incarnation]).encode())
        key = self._k(round_id, "decision")
        t_open = time.monotonic()
        if self._acting(self.coordinator, self.world) == replica_id:
            return self._coordinate(round_id, t_open + round_deadline_s)
        t_end = t_open + decide_timeout_s
        while True:
            if self.store.check([key]):
                return self._adopt(self.store.get(key))
            if self._acting(self.coordinator, self.world) == replica_id:
                # the coordinator is dead: this replica runs the round
                return self._coordinate(round_id, max(time.monotonic(), t_open + round_deadline_s))
            if time.monotonic() >= t_end:
                raise Recoverable(PEER_DOWN, f"no decision for round {round_id} within {decide_timeout_s}s")
            try:
                self.store.wait([key], timedelta(seconds=0.05))
            except Exception:  # noqa: BLE001 - poll again (liveness check above)
                pass

    def _follow(self, d: Decision) -> None:
        # keep the local engine in lock-step for a future coordinator role
        self.engine.epoch, self.engine.target_step, self.engine.generation = d.epoch, d.target_step, d.generation
        self.engine._prev_roles = (d.healthy, tuple(sorted(d.behind)))

    def follow(self, round_id: int, timeout_s: float = 60.0) -> Decision:
        """Read round `round_id`'s decision without reporting (a replica that
        is out of the group but keeps its round counter in step)."""
        key = self._k(round_id, "decision")
        self.store.wait([key], timedelta(seconds=timeout_s))
        return self._adopt(self.store.get(key))

    def vote(self, round_id: int, decision: Decision, replica_id: int, ok: bool,
             deadline_s: float = 2.0) -> bool:
        """The commit round (the reference's 2PC, replica.py:589-603): every
        member of the decision votes; the step commits iff all voted ok before
        the deadline.  One member — the lowest live id of the decision —
        collects the votes and publishes the outcome that everyone applies, so
        a vote arriving at the deadline cannot commit on one replica and abort
        on another."""
        self.store.set(self._k(round_id, "vote", replica_id), b"1" if ok else b"0")
        out_key = self._k(round_id, "outcome")
        members = decision.members
        if not members:
            return False
        keys = [self._k(round_id, "vote", m) for m in members]
        t_open = time.monotonic()

        def decide_outcome() -> bool:
            t_end = t_open + deadline_s
            while True:
                got = [k for k in keys if self.store.check([k])]
                if len(got) == len(keys):
                    commit = all(self.store.get(k) == b"1" for k in keys)
                    break
                missing = [m for m, k in zip(members, keys) if k not in got]
                if time.monotonic() >= t_end or any(self._dead(m) for m in missing):
                    commit = False  # a member never voted (or died): abort the step
                    break
                time.sleep(0.002)
            return self._publish_once(out_key, b"commit" if commit else b"abort") == b"commit"

        if self._acting(members[0], members) == replica_id:
            return decide_outcome()
        t_end = t_open + deadline_s + 30.0
        while True:
            if self.store.check([out_key]):
                return self.store.get(out_key) == b"commit"
            if self._acting(members[0], members) == replica_id:
                return decide_outcome()
            if time.monotonic() >= t_end:
                return False  # the decider is gone: nothing was committed
            try:
                self.store.wait([out_key], timedelta(seconds=0.05))
            except Exception:  # noqa: BLE001
                pass
