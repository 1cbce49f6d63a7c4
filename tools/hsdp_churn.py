"""Config 5: end-to-end HSDP steps with a failure/rejoin schedule.

    python -m torch.distributed.run --nproc-per-node N tools/hsdp_churn.py \\
        [--params 1e9] [--steps 12] [--kill-at 4] [--dead 3]

Each GPU is a replica (R = 1 rank) holding a full copy of a 1B-parameter
model's fp32 params + SGD momentum (the reference's HSDP layout,
replica.py:725-760).  The step loop mirrors the reference's
_RankWorker.iterate (replica.py:518-668) over this repo's drop-in API:

  1. StoreQuorum round -> Decision (QuorumEngine, quorum.py:172-210)
  2. RingGroup.reconfig when the generation moved (replica.py:551-561),
     contributors = healthy (behind replicas fold +0.0, replica.py:574-577)
  3. healthy: synthetic bf16 gradients of the step (a random-init
     "transformer" gradient stream), bucketed 256 MiB; behind: start the
     striped NVLink catch-up pull of step target-1 (replica.py:452-493)
  4. FTAR of every bucket: bf16 in, fp32 out, x f32(1/h) fused, queued
  5. commit vote (the 2PC, replica.py:589-603); on commit: behind installs
     the fetched state, everyone applies m = m*beta + g; p -= lr*m in fp32
     (model.py:146-155), snapshot capture (replica.py:645-648)

Failure schedule (scenario.py kill_replica): the victim dies mid-collective
at step --kill-at (it never joins that step's FTAR, like a killed process),
restarts as a new incarnation from the initial state, is parked by the
engine for --dead steps and admitted at the gate step kill_at + dead
(quorum.admit_after), catches up over NVLink and must end bit-identical to
the survivors.  Rank 0 prints a JSON report:
per-step healthy counts / generations / retries (the reference's KAT shape,
tests/test_replica.py:368-385), step times, stall, effective throughput and
the cross-replica params/momentum digests.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--params", type=float, default=1e9)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--bucket-mib", type=int, default=256, help="bf16 bucket MiB")
    ap.add_argument("--kill-at", type=int, default=4)
    ap.add_argument("--dead", type=int, default=3)
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--beta", type=float, default=0.9)
    ap.add_argument("--chunk-timeout", type=float, default=0.5)
    ap.add_argument("--unfused", action="store_true", help="separate torch optimizer instead of the fused SGD")
    ap.add_argument("--pull-ctas", type=int, default=8, help="CTA budget of the catch-up pull")
    ap.add_argument("--boost-ctas", type=int, default=0,
                    help="widen the pull to this many more CTAs once the step's FTAR is done (0: never)")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2602_00277_b200 import checkpoint as ck
    from paper_2602_00277_b200 import errors, ftar
    from paper_2602_00277_b200.fabric import StoreFabric
    from paper_2602_00277_b200.quorum import Report, StoreQuorum

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    rid, world = dist.get_rank(), dist.get_world_size()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", rid)))
    torch.cuda.set_device(dev)
    store = dist.PrefixStore("hsdp", dist.distributed_c10d._get_default_store())
    fabric = StoreFabric(store)
    victim = world - 1 if world >= 2 else -1
    quorum = StoreQuorum(store, list(range(world)), prefix="hsdp/quorum")
    gate = args.kill_at + args.dead
    quorum.engine.admit_after(victim, gate, 1)  # the harness schedules the rejoin (harness.py:367-391)

    P = int(args.params)
    be = args.bucket_mib * (1 << 20) // 2  # bf16 elements per bucket
    buckets = [(o, min(be, P - o)) for o in range(0, P, be)]
    group = ftar.RingGroup(rid, 0, fabric, device=dev, max_bucket_bytes=be * 2,
                           pool_bytes=P * 2 + P * 4 + 8192)
    grads = group.alloc_bucket(P, torch.bfloat16)
    red = group.alloc_bucket(P, torch.float32)  # reduced fp32 gradient (push-mode target)
    f32 = lambda x: float(np.float32(x))  # noqa: E731

    def init_state():
        g = torch.Generator(device=dev).manual_seed(1234)
        p = (torch.randn(P, device=dev, generator=g) * 0.02).float()
        return p, torch.zeros(P, device=dev)

    params, mom = init_state()
    base = torch.Generator(device=dev).manual_seed(77 + rid)
    grad_base = torch.randn(P, device=dev, generator=base).to(torch.bfloat16)
    snap = ck.SnapshotStore(capacity_bytes=P * 8, device=dev, fabric=fabric, rank=0, replica_id=rid)
    snap.capture(0, params, mom)
    fetched = (torch.empty(P, device=dev), torch.empty(P, device=dev))
    nxt = (torch.empty(P, device=dev), torch.empty(P, device=dev))  # fused optimizer writes here (out of place)
    cfg = ftar.PipelineConfig(per_chunk_timeout_s=args.chunk_timeout)

    torch.cuda.synchronize()
    dist.barrier()  # replicas enter round 1 together (no start-up skew vs the round deadline)
    step, inc, rnd = 0, 0, 0
    killed = False
    log, t_steps = [], []
    t_run = time.monotonic()
    while True:
        rnd += 1
        t0 = time.monotonic()
        if killed:
            # The respawned process starts at once and reports from the next
            # round on; the engine parks it until the gate step (admit_after),
            # so its start-up cost (init + mapping the donors' snapshot arenas,
            # ~0.3 s per 8 GB donor) never races the round deadline and it is
            # admitted at exactly the gate, as the reference harness arranges.
            d = quorum.follow(rnd)
            t_r = time.monotonic()
            params, mom = init_state()  # a fresh incarnation from the initial state
            step, inc, killed = 0, inc + 1, False
            torch.cuda.synchronize()
            t_i = time.monotonic()
            snap.connect(d.healthy, 0, timeout_s=10)  # not ready (no report) until mapped
            log.append({"round": rnd, "target": d.target_step, "event": "restarted",
                        "init_ms": round((t_i - t_r) * 1e3, 3),
                        "connect_ms": round((time.monotonic() - t_i) * 1e3, 3),
                        "map_ms": [(m[0], round(m[1] * 1e3, 1), round(m[2] * 1e3, 1)) for m in snap.map_log]})
            continue
        d = quorum.exchange(rnd, rid, Report(step + 1, inc), round_deadline_s=0.25)
        t_x = time.monotonic()
        if d.target_step > args.steps:
            break
        role = d.role_of(rid)
        if role == "unassigned":
            log.append({"round": rnd, "target": d.target_step, "role": role,
                        "t_ms": round((time.monotonic() - t_run) * 1e3, 1)})
            continue
        t_rc = time.monotonic()
        if d.generation > group.generation:
            group.reconfig({m: ftar.PeerAddress(m) for m in d.members}, d.generation, deadline_s=30,
                           contributors=d.healthy)
        t_rc = time.monotonic() - t_rc
        target = d.target_step
        pull = None

        def fetch(refresh=False):
            # donors were mapped at restart (connect): no Store lookups here
            return ck.start_fetch(snap, list(d.healthy), target - 1, 0, fetched[0], fetched[1],
                                  timeout_s=10, ctas=args.pull_ctas, refresh=refresh)

        if role == "healthy":
            grads.copy_(grad_base)
            grads.mul_(1.0 / (1.0 + 0.1 * target))  # the step's synthetic gradient
        if rid == victim and target == args.kill_at and inc == 0:
            # killed mid-collective: never joins this step's FTAR
            killed = True
            log.append({"round": rnd, "target": target, "event": "killed"})
            continue
        ok = True
        fused = role == "healthy" and not args.unfused
        bucket_ms = []
        t_ar = time.monotonic()
        try:
            bucket_ms = []
            if fused:
                # §8f: all-reduce + x f32(1/h) + SGD-momentum in one kernel per
                # bucket, out of place (applied by the swap at commit)
                pend = [ftar.ftar_all_reduce_sgd_async(group, grads[o:o + n], target, cfg, params=params[o:o + n],
                                                       momentum=mom[o:o + n], lr=args.lr, beta=args.beta,
                                                       scale=d.scale(), params_out=nxt[0][o:o + n],
                                                       momentum_out=nxt[1][o:o + n]) for o, n in buckets]
                for p_ in pend:
                    p_.wait()
                    bucket_ms.append(round((time.monotonic() - t_ar) * 1e3, 2))
            else:
                pend = [ftar.ftar_all_reduce_async(group, grads[o:o + n], target, cfg, out=red[o:o + n],
                                                   scale=d.scale()) for o, n in buckets[:3]]
                if role == "behind" and not snap.connecting():
                    # the ring's first buckets are queued: now start the pull on its
                    # low-priority side stream (its host-side donor lookups must not
                    # delay this replica's entry into the collective)
                    t_f = time.monotonic()
                    pull = fetch()
                    bucket_ms.append(("fetch_call_ms", round((time.monotonic() - t_f) * 1e3, 3),
                                      "streams_ms/launch_ms", getattr(snap, "launch_log", None)))
                for o, n in buckets[3:]:
                    t_l = time.monotonic()
                    pend.append(ftar.ftar_all_reduce_async(group, grads[o:o + n], target, cfg, out=red[o:o + n],
                                                           scale=d.scale()))
                    if role == "behind":
                        bucket_ms.append(("launch_ms", round((time.monotonic() - t_l) * 1e3, 3)))
                for p_ in pend:
                    p_.wait()
                    bucket_ms.append(round((time.monotonic() - t_ar) * 1e3, 2))
        except errors.Recoverable:
            ok = False
        torch.cuda.current_stream(dev).synchronize()  # the FTAR only (a catch-up pull runs on a side stream)
        t_ar = time.monotonic() - t_ar
        fetch_ok = True
        t_pw = time.monotonic()
        if role == "behind":
            try:
                if pull is None:  # donors still being mapped when the step began
                    pull = fetch()
                if args.boost_ctas:
                    pull.boost(args.boost_ctas)  # the collectives are done: full width
                try:
                    pull.wait()
                except ck.SnapshotUnavailable:
                    pull = fetch(refresh=True)  # a donor restarted since it was mapped
                    pull.wait()
            except (errors.FtdpError, ck.SnapshotUnavailable):
                fetch_ok = False
        t_pw = time.monotonic() - t_pw
        t_v = time.monotonic()
        committed = quorum.vote(rnd, d, rid, ok and fetch_ok, deadline_s=1.0)
        t_v = time.monotonic() - t_v
        if committed:
            if fused:
                params, nxt = nxt[0], (params, nxt[1])
                mom, nxt = nxt[1], (nxt[0], mom)
            else:
                if role == "behind":
                    params.copy_(fetched[0])
                    mom.copy_(fetched[1])
                mom.mul_(f32(args.beta)).add_(red)          # m = f32(m*beta) + g
                params.sub_(mom * f32(args.lr))             # p -= f32(lr*m)
            step = target
            snap.capture(step, params, mom)
        torch.cuda.synchronize()
        dt = time.monotonic() - t0
        t_steps.append(dt)
        log.append({"round": rnd, "target": target, "generation": d.generation, "role": role,
                    "healthy": len(d.healthy), "behind": sorted(d.behind), "committed": committed,
                    "ftar_ms": round(t_ar * 1e3, 3), "step_ms": round(dt * 1e3, 3),
                    "quorum_ms": round((t_x - t0) * 1e3, 3), "reconfig_ms": round(t_rc * 1e3, 3),
                    "bucket_done_ms": bucket_ms,
                    "pull_wait_ms": round(t_pw * 1e3, 3),
                    "vote_ms": round(t_v * 1e3, 3)})
    elapsed = time.monotonic() - t_run
    # cross-replica agreement on the final state
    dig = hashlib.sha256(params.cpu().numpy().tobytes() + mom.cpu().numpy().tobytes()).hexdigest()
    digs = [None] * world
    dist.all_gather_object(digs, dig)
    logs = [None] * world
    dist.all_gather_object(logs, log)
    if rid == 0:
        commits = [e for e in logs[0] if e.get("committed")]
        hist = {e["target"]: e["healthy"] for e in commits}
        ok_steps = [e for e in commits if e["healthy"] == world]
        steady = sorted(e["step_ms"] for e in ok_steps)[len(ok_steps) // 2] if ok_steps else None
        ftar_ms = sorted(e["ftar_ms"] for e in ok_steps)[len(ok_steps) // 2] if ok_steps else None
        grad_bytes = P * 2
        rep = {"config": "config5: HSDP steps, 1 replica per GPU, failure/rejoin churn",
               "replicas": world, "params": P, "buckets": len(buckets), "bucket_mib_bf16": args.bucket_mib,
               "steps": args.steps, "victim": victim, "killed_at": args.kill_at, "rejoin_gate": gate,
               "healthy_count_per_step": hist,
               "retried_steps": sorted({e["target"] for e in logs[0] if e.get("committed") is False}),
               "victim_catch_up_steps": [e["target"] for e in (logs[victim] if victim >= 0 else [])
                                         if e.get("role") == "behind" and e.get("committed")],
               "generations": sorted({e["generation"] for e in logs[0] if "generation" in e}),
               "final_digests_equal": len(set(digs)) == 1, "digest": digs[0][:16],
               "steady_step_ms_median": steady, "steady_ftar_ms_median": ftar_ms,
               "ftar_busbw_steady_GBps": round(grad_bytes / (ftar_ms / 1e3) * 2 * (world - 1) / world / 1e9, 1)
               if ftar_ms else None,
               "run_seconds": round(elapsed, 3), "log_rank0": logs[0],
               "log_victim": logs[victim] if victim >= 0 else []}
        print(json.dumps(rep), flush=True)
    group.close()
    snap.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
