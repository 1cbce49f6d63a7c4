"""Generate the golden fixtures by RUNNING THE REFERENCE (dev container only).

    python tests/golden/make_golden.py          # needs /root/reference

Writes, next to this script:
  ftar_cases.json      per-case (n, len, chunk_bytes, max_in_flight, seed, kind)
                       + sha256 of the output of the reference's socket ring
                       (bench._LoopbackRing, pkg/src/ftdp/bench.py:53-88) on
                       inputs regenerated from the seed (tests/golden/gen.py)
  ftar_small.npz       full input/output vectors of the hand cases
                       (tests/test_ftar.py:195-210)
  config1.json         digest of config 1 (4 x 4,194,304 fp32, default
                       PipelineConfig) through the reference ring
  quorum_traces.json   QuorumEngine (quorum.py:172-210) report->decision
                       sequences: the test KATs, a seeded churn stream, and
                       the 8-replica kill trace recorded from the reference's
                       replica engine (tests/helpers.py Cluster)
  replica_ftar.npz     every ftar_all_reduce call of that 8-replica run:
                       members, generation, input, output (replay fixture)
  normalize.npz        grad *= f32(1/(h*R)) vectors (replica.py:622-626)

The reference is imported read-only from /root/reference/pkg/src; nothing
here is used at run time on the GPU box.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path.insert(0, HERE)
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

from gen import case_inputs, criterion_cases  # noqa: E402

from ftdp import bench as rbench  # noqa: E402
from ftdp import ftar as rftar  # noqa: E402
from ftdp import quorum as rquorum  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def run_ring(rings, arrays, chunk, C, step):
    n = len(arrays)
    if n not in rings:
        rings[n] = rbench._LoopbackRing(n)
    bufs = [a.copy() for a in arrays]
    cfg = rftar.PipelineConfig(chunk_bytes=chunk, max_in_flight=C, per_chunk_timeout_s=30.0)
    rings[n].timed_all_reduce(bufs, step, cfg)
    for b in bufs[1:]:
        assert np.array_equal(b, bufs[0], equal_nan=True)
    return bufs[0]


def make_ftar_cases():
    rings = {}
    cases = []
    step = 0
    try:
        for spec in criterion_cases():
            arrays = case_inputs(spec)
            step += 1
            out = run_ring(rings, arrays, spec["chunk_bytes"], spec["max_in_flight"], step)
            cases.append({**spec, "sha256": sha(out)})
        # hand cases with full vectors
        small = {}
        hand = [
            ("four_members", [np.full(8, float(i), dtype=np.float32) for i in range(4)], 8, 2),
            ("multi_partition", [np.arange(8, dtype=np.float32) * (i + 1) for i in range(4)], 4, 1),
        ]
        for name, arrays, chunk, C in hand:
            step += 1
            out = run_ring(rings, arrays, chunk, C, step)
            small[f"{name}_in"] = np.stack(arrays)
            small[f"{name}_out"] = out
            small[f"{name}_cfg"] = np.array([chunk, C])
        np.savez_compressed(os.path.join(HERE, "ftar_small.npz"), **small)
        # config 1 (BASELINE configs[0])
        from gen import member_inputs
        arrays = member_inputs(4, 4_194_304, seed=0)
        step += 1
        out = run_ring(rings, arrays, 8 * 1024 * 1024, 4, step)
        with open(os.path.join(HERE, "config1.json"), "w") as f:
            json.dump({"n": 4, "elems": 4_194_304, "seed": 0, "chunk_bytes": 8 * 1024 * 1024,
                       "max_in_flight": 4, "sha256": sha(out),
                       "head": [float(x) for x in out[:8]]}, f, indent=1)
    finally:
        for r in rings.values():
            r.close()
    with open(os.path.join(HERE, "ftar_cases.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print(f"ftar cases: {len(cases)}")


def dec_json(d):
    return {"epoch": d.epoch, "target_step": d.target_step, "generation": d.generation,
            "healthy": list(d.healthy), "behind": {str(k): v for k, v in d.behind.items()},
            "members": list(d.members)}


class Recorder:
    """Wraps one QuorumEngine: logs every admit_after and decide call."""

    def __init__(self, eng):
        self.eng = eng
        self.ops = []
        orig_decide, orig_admit, orig_register = eng.decide, eng.admit_after, eng.register

        self._depth = 0

        def decide(reports):
            self._depth += 1
            try:
                d = orig_decide(reports)
            finally:
                self._depth -= 1
            self.ops.append({"op": "decide",
                             "reports": {str(k): [v.next_step, v.incarnation] for k, v in reports.items()},
                             "decision": dec_json(d)})
            return d

        def admit_after(rid, step, min_inc=0):
            self.ops.append({"op": "admit_after", "args": [rid, step, min_inc]})
            return orig_admit(rid, step, min_inc)

        def register(rid, inc):
            ok = orig_register(rid, inc)
            if self._depth == 0:  # top-level calls only (decide registers internally)
                self.ops.append({"op": "register", "args": [rid, inc], "result": ok})
            return ok

        eng.decide, eng.admit_after = decide, admit_after
        eng.register = register


def kat_streams():
    R = rquorum.Report
    streams = {}

    def run(name, fn):
        eng = rquorum.QuorumEngine()
        rec = Recorder(eng)
        fn(eng, R)
        streams[name] = rec.ops

    def reps(**kw):
        return {int(k[1:]): R(next_step=v, incarnation=1) for k, v in kw.items()}

    run("one_behind", lambda e, R: e.decide(reps(r0=100, r1=100, r2=100, r3=96)))
    run("stall", lambda e, R: [e.decide(reps(r0=5, r1=5)) for _ in range(3)])
    run("role_change", lambda e, R: [e.decide(reps(r0=4, r1=4, r2=4)), e.decide(reps(r0=5, r1=5)),
                                     e.decide(reps(r0=6, r1=6, r2=4)), e.decide(reps(r0=7, r1=7, r2=7)),
                                     e.decide(reps(r0=8, r1=8, r2=8))])
    run("incarnation", lambda e, R: [e.register(2, 1), e.decide({0: R(5, 1), 2: R(5, 0)}),
                                     e.register(2, 3), e.register(2, 2), e.decide({0: R(6, 1), 2: R(1, 3)})])
    run("gate", lambda e, R: [e.decide(reps(r0=50, r1=50, r2=50)), e.admit_after(2, 70),
                              e.decide(reps(r0=51, r1=51, r2=1)), e.decide(reps(r0=70, r1=70, r2=1))])
    run("lost_frontier", lambda e, R: [e.decide(reps(r0=100, r1=100)), e.decide(reps(r0=1, r1=1)),
                                       e.decide(reps(r0=100, r1=1))])

    def churn(e, R):
        rng = np.random.default_rng(0xC0FFEE)
        steps = {r: 1 for r in range(8)}
        inc = {r: 1 for r in range(8)}
        alive = set(range(8))
        for rnd in range(300):
            u = rng.random()
            if u < 0.05 and len(alive) > 2:
                victim = int(rng.choice(sorted(alive)))
                alive.discard(victim)
            elif u < 0.12:
                dead = sorted(set(range(8)) - alive)
                if dead:
                    back = int(rng.choice(dead))
                    inc[back] += 1
                    steps[back] = 1 if rng.random() < 0.5 else max(steps.values()) - int(rng.integers(0, 3))
                    if rng.random() < 0.3:
                        e.admit_after(back, max(steps.values()) + int(rng.integers(0, 4)), inc[back])
                    alive.add(back)
            rep = {r: R(max(1, steps[r]), inc[r]) for r in alive if rng.random() > 0.03}
            if rng.random() < 0.02:
                r = int(rng.integers(0, 8))
                rep[r] = R(steps[r], inc[r] - 1)  # stale incarnation straggler
            d = e.decide(rep)
            for r in d.healthy:
                if rng.random() > 0.04:
                    steps[r] = d.target_step + 1
            for r in d.behind:
                if rng.random() < 0.5:
                    steps[r] = d.target_step + 1
    run("churn", churn)
    return streams


def replica_trace():
    """8 replicas, kill replica 5 at step 3 for 3 steps."""
    from helpers import Cluster, kill_failure, quick_scenario
    from ftdp import replica as rreplica

    recs = []
    calls = []
    lock = threading.Lock()
    orig_init = rquorum.QuorumEngine.__init__

    def init(self):
        orig_init(self)
        recs.append(Recorder(self))

    orig_ftar = rreplica.ftar.ftar_all_reduce

    def traced(group, buf, step, cfg=None):
        before = buf.copy()
        try:
            out = orig_ftar(group, buf, step, cfg)
            res = out.copy()
            err = None
        except Exception as exc:  # noqa: BLE001
            res, err = None, f"{type(exc).__name__}:{getattr(exc, 'reason', '')}"
            raise
        finally:
            with lock:
                calls.append({"replica": group.self_replica, "rank": group.rank, "step": step,
                              "generation": group.generation, "members": list(group.members),
                              "input": before, "output": res, "error": err,
                              "cfg": [cfg.chunk_bytes, cfg.max_in_flight] if cfg else None})
        return out

    rquorum.QuorumEngine.__init__ = init
    rreplica.ftar.ftar_all_reduce = traced
    try:
        cfg = quick_scenario(num_replicas=8, ranks=1, total_steps=10,
                             failures=[kill_failure(3, 3, (5,))])
        with tempfile.TemporaryDirectory() as d:
            cluster = Cluster(cfg, d)
            codes = cluster.run(timeout_s=120)
            assert all(c == 0 for c in codes.values()), codes
    finally:
        rquorum.QuorumEngine.__init__ = orig_init
        rreplica.ftar.ftar_all_reduce = orig_ftar
    assert len(recs) == 1
    return recs[0].ops, calls, cfg


def make_quorum_and_replica():
    streams = kat_streams()
    ops, calls, cfg = replica_trace()
    streams["replica_kill_r5_at3_for3"] = ops
    with open(os.path.join(HERE, "quorum_traces.json"), "w") as f:
        json.dump(streams, f, indent=0)
    arrays = {}
    meta = []
    for i, c in enumerate(calls):
        arrays[f"in{i}"] = c["input"]
        if c["output"] is not None:
            arrays[f"out{i}"] = c["output"]
        meta.append({k: c[k] for k in ("replica", "rank", "step", "generation", "members", "error", "cfg")})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "replica_ftar.npz"), **arrays)
    print(f"quorum streams: {len(streams)}; replica ftar calls: {len(calls)}; "
          f"scale denominators h*R with R={cfg.topology.ranks_per_replica}")


def make_normalize():
    rng = np.random.default_rng(5)
    x = (rng.standard_normal(16_384) * 10.0 ** rng.integers(-3, 4, 16_384)).astype(np.float32)
    out = {"x": x}
    for h in range(1, 9):
        for R in (1, 2):
            out[f"h{h}_R{R}"] = x * np.float32(1.0 / (h * R))
    np.savez_compressed(os.path.join(HERE, "normalize.npz"), **out)


if __name__ == "__main__":
    make_ftar_cases()
    make_quorum_and_replica()
    make_normalize()
