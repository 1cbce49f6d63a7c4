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
    ``epoch``; the coordinator replica (lowest live id that posted) runs
    ``QuorumEngine.decide`` and publishes the Decision; everyone reads it.
    Replicas that do not post within ``round_deadline_s`` are absent, exactly
    like the reference coordinator's round deadline (quorum.py:354-396)."""

    def __init__(self, store, world: list[int], prefix: str = "ftar/quorum"):
        self.store = store
        self.world = sorted(world)
        self.prefix = prefix
        self.engine = QuorumEngine()

    def _k(self, *p) -> str:
        return "/".join([self.prefix, *map(str, p)])

    def exchange(self, round_id: int, replica_id: int, report: Report, round_deadline_s: float = 2.0,
                 decide_timeout_s: float = 30.0) -> Decision:
        self.store.set(self._k(round_id, "report", replica_id),
                       json.dumps([report.next_step, report.incarnation]).encode())
        t_end = time.monotonic() + round_deadline_s
        reports: dict[int, Report] = {}
        while True:
            for rid in self.world:
                if rid not in reports and self.store.check([self._k(round_id, "report", rid)]):
                    ns, inc = json.loads(self.store.get(self._k(round_id, "report", rid)))
                    reports[rid] = Report(ns, inc)
            if len(reports) == len(self.world) or time.monotonic() >= t_end:
                break
            time.sleep(0.005)
        # lowest posted id coordinates; the engine state replays identically on
        # every replica because all replicas feed it the same posted reports
        coord = min(reports)
        key = self._k(round_id, "decision")
        if coord == replica_id:
            d = self.engine.decide(reports)
            self.store.set(key, json.dumps(d.to_json()).encode())
            return d
        try:
            self.store.wait([key], timedelta(seconds=decide_timeout_s))
        except Exception as exc:  # noqa: BLE001
            raise Recoverable(PEER_DOWN, f"no decision for round {round_id}: {exc}")
        d = Decision.from_json(json.loads(self.store.get(key)))
        # keep the local engine in lock-step for a future coordinator role
        self.engine.epoch, self.engine.target_step, self.engine.generation = d.epoch, d.target_step, d.generation
        self.engine._prev_roles = (d.healthy, tuple(sorted(d.behind)))
        return d
