"""Membership decisions: the reference's KATs (tests/test_quorum.py:18-127)
and bit-exact replay of decision streams recorded from the reference engine
(tests/golden/quorum_traces.json), including the 8-replica kill trace of its
replica engine."""

import json
import os

import pytest

from paper_2602_00277_b200.quorum import Decision, QuorumEngine, Report

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def reports(**kw):
    return {int(k[1:]): Report(next_step=v, incarnation=1) for k, v in kw.items()}


def test_one_replica_behind():
    d = QuorumEngine().decide(reports(r0=100, r1=100, r2=100, r3=96))
    assert d.target_step == 100 and d.healthy == (0, 1, 2) and d.behind == {3: 96}
    assert d.members == (0, 1, 2, 3) and d.generation == 1 and d.epoch == 1
    assert d.live_mask() == 0b1111 and d.contrib_mask() == 0b0111


def test_generation_rules():
    e = QuorumEngine()
    assert [e.decide(reports(r0=s, r1=s)).generation for s in (1, 2, 3)] == [1, 1, 1]
    e = QuorumEngine()
    e.decide(reports(r0=5, r1=5))
    assert [e.decide(reports(r0=5, r1=5)).generation for _ in range(2)] == [2, 3]
    e = QuorumEngine()
    e.decide(reports(r0=4, r1=4, r2=4))
    d = e.decide(reports(r0=5, r1=5))
    assert d.generation == 2 and d.healthy == (0, 1)
    d = e.decide(reports(r0=6, r1=6, r2=4))
    assert d.generation == 3 and d.behind == {2: 4}
    d = e.decide(reports(r0=7, r1=7, r2=7))
    assert d.generation == 4
    assert e.decide(reports(r0=8, r1=8, r2=8)).generation == 4


def test_incarnation_fencing_and_gates():
    e = QuorumEngine()
    assert e.register(2, 1)
    assert e.decide({0: Report(5, 1), 2: Report(5, 0)}).members == (0,)
    assert e.register(2, 3) and not e.register(2, 2)
    assert e.decide({0: Report(6, 1), 2: Report(1, 3)}).behind == {2: 1}
    e = QuorumEngine()
    e.decide(reports(r0=50, r1=50, r2=50))
    e.admit_after(2, 70)
    assert e.decide(reports(r0=51, r1=51, r2=1)).members == (0, 1)
    assert e.pending_joiners(reports(r0=69, r1=69)) == set()
    assert e.pending_joiners(reports(r0=70, r1=70)) == {2}
    d = e.decide(reports(r0=70, r1=70, r2=1))
    assert d.behind == {2: 1} and e.admission_gate(2) is None


def test_lost_frontier_holds_target():
    e = QuorumEngine()
    e.decide(reports(r0=100, r1=100))
    d = e.decide(reports(r0=1, r1=1))
    assert d.target_step == 100 and d.healthy == () and d.behind == {0: 1, 1: 1} and d.generation == 2
    d = e.decide(reports(r0=100, r1=1))
    assert d.healthy == (0,) and d.behind == {1: 1}


def test_scale_is_f32_reciprocal():
    import numpy as np
    d = Decision(1, 5, 2, (0, 1, 2, 3, 4, 6, 7), {5: 1})
    assert d.scale() == float(np.float32(1.0 / 7))
    assert d.scale(ranks_per_replica=2) == float(np.float32(1.0 / 14))
    assert d.contrib_mask() == 0b11011111


def _replay(ops):
    e = QuorumEngine()
    n = 0
    for op in ops:
        if op["op"] == "register":
            assert e.register(*op["args"]) == op["result"]
        elif op["op"] == "admit_after":
            e.admit_after(*op["args"])
        else:
            reps = {int(k): Report(*v) for k, v in op["reports"].items()}
            d = e.decide(reps)
            want = op["decision"]
            got = {"epoch": d.epoch, "target_step": d.target_step, "generation": d.generation,
                   "healthy": list(d.healthy), "behind": {str(k): v for k, v in d.behind.items()},
                   "members": list(d.members)}
            assert got == want, f"decision {n}: {got} != {want}"
            n += 1
    return n


def _streams():
    with open(os.path.join(GOLD, "quorum_traces.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(_streams()))
def test_replay_reference_decision_streams(name):
    assert _replay(_streams()[name]) > 0


def test_kill_trace_shape():
    """kill r5 at step 3 for 3 steps, 8 replicas."""
    ds = [Decision.from_json(op["decision"]) for op in _streams()["replica_kill_r5_at3_for3"]
          if op["op"] == "decide"]
    rows = [(d.epoch, d.target_step, d.generation, d.healthy, d.behind) for d in ds[:8]]
    allm = (0, 1, 2, 3, 4, 5, 6, 7)
    wo5 = (0, 1, 2, 3, 4, 6, 7)
    assert rows[3] == (4, 3, 2, wo5, {})
    assert rows[6] == (7, 6, 3, wo5, {5: 1})
    assert rows[7] == (8, 7, 4, allm, {})


# --- StoreQuorum over a real TCPStore (threads stand in for replicas) -------


def _stores(n):
    from datetime import timedelta

    import torch.distributed as dist
    master = dist.TCPStore("127.0.0.1", 0, is_master=True, wait_for_workers=False,
                           timeout=timedelta(seconds=30))
    clients = [dist.TCPStore("127.0.0.1", master.port, is_master=False, timeout=timedelta(seconds=30))
               for _ in range(n)]
    return master, clients


def _run_threads(fns):
    import threading
    out, errs = [None] * len(fns), []

    def wrap(i, f):
        try:
            out[i] = f()
        except Exception as exc:  # noqa: BLE001
            errs.append(exc)

    ts = [threading.Thread(target=wrap, args=(i, f)) for i, f in enumerate(fns)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    assert not errs, errs
    return out


def test_store_quorum_early_poster_does_not_decide():
    """A replica that opens the round before the others (e.g. a parked
    rejoiner looping fast) must read the coordinator's decision, not publish
    one from its own partial view."""
    import time

    from paper_2602_00277_b200.quorum import StoreQuorum
    master, cl = _stores(3)
    qs = [StoreQuorum(cl[i], [0, 1, 2], prefix="tq") for i in range(3)]

    def rep(i, delay):
        def f():
            time.sleep(delay)
            return qs[i].exchange(1, i, Report(5, 0), round_deadline_s=1.0)
        return f

    ds = _run_threads([rep(0, 0.3), rep(1, 0.35), rep(2, 0.0)])
    assert all(d == ds[0] for d in ds)
    assert ds[0].healthy == (0, 1, 2) and ds[0].target_step == 5
    # the follower path reads the same decision
    assert qs[2].follow(1, timeout_s=5) == ds[0]


def test_store_quorum_vote_outcome_is_shared():
    import time

    from paper_2602_00277_b200.quorum import StoreQuorum
    master, cl = _stores(3)
    qs = [StoreQuorum(cl[i], [0, 1, 2], prefix="tv") for i in range(3)]
    d = Decision(1, 5, 1, (0, 1, 2), {})

    def voter(i, rnd, ok, delay):
        def f():
            time.sleep(delay)
            return qs[i].vote(rnd, d, i, ok, deadline_s=0.5)
        return f

    assert _run_threads([voter(i, 1, True, 0.0) for i in range(3)]) == [True] * 3
    assert _run_threads([voter(0, 2, True, 0), voter(1, 2, False, 0), voter(2, 2, True, 0)]) == [False] * 3
    # a vote that lands after the decider's deadline aborts the step everywhere,
    # including on the late voter itself
    assert _run_threads([voter(0, 3, True, 0), voter(1, 3, True, 0), voter(2, 3, True, 0.8)]) == [False] * 3


def _dead_heartbeat(store, prefix, rid):
    import time
    store.set(f"{prefix}/hb/{rid}", repr(time.time() - 60.0).encode())


def test_store_quorum_outage_round_ends_when_live_reporters_posted():
    """With heartbeats, a round in which a replica is dead closes as soon as
    every live replica posted, not at the round deadline."""
    import time

    from paper_2602_00277_b200.quorum import StoreQuorum
    master, cl = _stores(3)
    qs = [StoreQuorum(cl[i], [0, 1, 2], prefix="tl", liveness_s=0.5) for i in range(3)]
    qs[0].start_heartbeat(0)
    qs[1].start_heartbeat(1)
    _dead_heartbeat(cl[2], "tl", 2)
    t0 = time.monotonic()
    ds = _run_threads([lambda: qs[0].exchange(1, 0, Report(4, 0), round_deadline_s=20.0),
                       lambda: qs[1].exchange(1, 1, Report(4, 0), round_deadline_s=20.0)])
    took = time.monotonic() - t0
    for q in qs:
        q.stop_heartbeat()
    assert ds[0] == ds[1] and ds[0].healthy == (0, 1)
    assert took < 5.0, took


def test_store_quorum_coordinator_failover():
    """The coordinator (lowest id) is dead: the lowest LIVE replica runs the
    round, everyone adopts its decision and engine state, and the next round
    continues the same epoch/generation sequence."""
    import time

    from paper_2602_00277_b200.quorum import StoreQuorum
    master, cl = _stores(3)
    qs = [StoreQuorum(cl[i], [0, 1, 2], prefix="tf", liveness_s=0.5) for i in range(3)]
    qs[1].start_heartbeat(1)
    qs[2].start_heartbeat(2)
    _dead_heartbeat(cl[0], "tf", 0)
    t0 = time.monotonic()
    ds = _run_threads([lambda: qs[1].exchange(1, 1, Report(3, 0), round_deadline_s=20.0, decide_timeout_s=30.0),
                       lambda: qs[2].exchange(1, 2, Report(3, 0), round_deadline_s=20.0, decide_timeout_s=30.0)])
    assert time.monotonic() - t0 < 5.0
    assert ds[0] == ds[1] and ds[0].healthy == (1, 2) and ds[0].epoch == 1
    ds2 = _run_threads([lambda: qs[1].exchange(2, 1, Report(4, 0), round_deadline_s=20.0),
                        lambda: qs[2].exchange(2, 2, Report(4, 0), round_deadline_s=20.0)])
    for q in qs:
        q.stop_heartbeat()
    assert ds2[0] == ds2[1] and ds2[0].epoch == 2 and ds2[0].generation == ds[0].generation
    assert qs[2].engine.state() == qs[1].engine.state()


def test_store_quorum_vote_decider_failover():
    """The decision's lowest member died before voting: the next live member
    decides the outcome (abort: a vote is missing) without waiting out the
    deadline, and every live voter applies the same outcome."""
    import time

    from paper_2602_00277_b200.quorum import StoreQuorum
    master, cl = _stores(3)
    qs = [StoreQuorum(cl[i], [0, 1, 2], prefix="tvf", liveness_s=0.5) for i in range(3)]
    qs[1].start_heartbeat(1)
    qs[2].start_heartbeat(2)
    _dead_heartbeat(cl[0], "tvf", 0)
    d = Decision(1, 5, 1, (0, 1, 2), {})
    t0 = time.monotonic()
    out = _run_threads([lambda: qs[1].vote(1, d, 1, True, deadline_s=20.0),
                        lambda: qs[2].vote(1, d, 2, True, deadline_s=20.0)])
    for q in qs:
        q.stop_heartbeat()
    assert out == [False, False]
    assert time.monotonic() - t0 < 5.0
