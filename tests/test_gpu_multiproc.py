"""One process per GPU over NVLink (the production topology): CUDA-IPC arena
mapping through a TCPStore rendezvous, the two-shot pull kernel, failure of a
member mid-collective, quorum re-agreement and retry.  Needs >= 2 GPUs (run
with `gpurun --gpus 2` / `--gpus 4`); skipped otherwise."""

import json
import os
import socket
import sys
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, scenario, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import hashlib

    import numpy as np
    import torch.distributed as dist
    from datetime import timedelta

    from gen import behind_set, case_inputs, member_inputs
    from oracle import ftar_oracle as orc
    from paper_2602_00277_b200 import errors, ftar
    from paper_2602_00277_b200.fabric import StoreFabric
    from paper_2602_00277_b200.quorum import Report, StoreQuorum

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    store = dist.TCPStore("127.0.0.1", port, world, rank == 0, timeout=timedelta(seconds=60))
    fabric = StoreFabric(dist.PrefixStore(scenario, store))
    res = {"rank": rank, "ok": [], "errors": []}

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()

    group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=64 << 20, pool_bytes=16 << 20)
    try:
        if scenario == "golden":
            with open(os.path.join(ROOT, "tests", "golden", "ftar_cases.json")) as f:
                cases = [c for c in json.load(f) if c["n"] == world]
            gen = 0
            for case in cases:
                gen += 1
                behind = behind_set(case)
                group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, gen, deadline_s=30,
                               contributors=[r for r in range(world) if r not in behind])
                arrays = case_inputs(case, garbage_behind=bool(behind))
                cfg = ftar.PipelineConfig(chunk_bytes=case["chunk_bytes"], max_in_flight=case["max_in_flight"],
                                          per_chunk_timeout_s=10)
                if case["kind"] == "bf16":
                    buf = torch.from_numpy(arrays[rank]).to(dev).to(torch.bfloat16)
                    out = torch.empty(case["elems"], device=dev)
                    ftar.ftar_all_reduce(group, buf, 1, cfg, out=out)
                else:
                    out = torch.from_numpy(arrays[rank]).to(dev)
                    assert ftar.ftar_all_reduce(group, out, 1, cfg) is out
                got = sha(out.cpu().numpy())
                (res["ok"] if got == case["sha256"] else res["errors"]).append(case["idx"])
            # big bucket: registered (zero-copy) bf16 with fused scale, default geometry
            gen += 1
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, gen, deadline_s=30)
            arrays = member_inputs(world, 1_500_001, seed=4, dtype="bf16")
            b = group.alloc_bucket(arrays[0].size, torch.bfloat16)
            b.copy_(torch.from_numpy(arrays[rank]).to(dev).to(torch.bfloat16))
            o = group.alloc_bucket(arrays[0].size, torch.float32)
            for _ in range(3):
                ftar.ftar_all_reduce(group, b, 2, ftar.PipelineConfig(), out=o, scale=1.0 / world)
            want = orc.normalize(orc.oracle_reduce(arrays, 8 << 20, 4), world)
            (res["ok"] if np.array_equal(o.cpu().numpy(), want) else res["errors"]).append("big_bf16")
        elif scenario == "failure":
            # config 2 in miniature: the highest rank stalls mid-collective
            # (it never calls); survivors must get Recoverable within 2x the
            # timeout, regroup through the quorum (generation+1) and retry.
            victim = world - 1
            q = StoreQuorum(fabric.store, list(range(world)))
            d = q.exchange(1, rank, Report(1, 0))
            group.reconfig({r: ftar.PeerAddress(r) for r in d.members}, d.generation, deadline_s=30)
            arrays = member_inputs(world, 2_000_003, seed=8)
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=1.0)
            buf = torch.from_numpy(arrays[rank]).to(dev)
            if rank == victim:
                import time
                time.sleep(6.0)  # a hung replica: misses this round and the next quorum round
                res["ok"].append("victim")
            else:
                import time
                t0 = time.monotonic()
                try:
                    ftar.ftar_all_reduce(group, buf, 1, cfg)
                    res["errors"].append("no error")
                except errors.Recoverable as exc:
                    took = time.monotonic() - t0
                    res["ok"].append(f"recoverable:{exc.reason}:{took:.2f}")
                    if took > 2 * cfg.per_chunk_timeout_s + 0.5:
                        res["errors"].append(f"slow abort {took:.2f}")
                if not np.array_equal(buf.cpu().numpy(), arrays[rank]):
                    res["errors"].append("buffer modified")
                d2 = q.exchange(2, rank, Report(1, 0), round_deadline_s=2.0)
                res["decision"] = d2.to_json()
                if victim in d2.members or d2.generation != d.generation + 1:
                    res["errors"].append(f"bad decision {d2}")
                group.reconfig({r: ftar.PeerAddress(r) for r in d2.members}, d2.generation, deadline_s=30)
                out = torch.empty_like(buf)
                ftar.ftar_all_reduce(group, buf, 1, cfg, out=out, scale=d2.scale())
                want = orc.normalize(orc.oracle_reduce([arrays[r] for r in d2.members], cfg.chunk_bytes,
                                                       cfg.max_in_flight), len(d2.healthy))
                (res["ok"] if np.array_equal(out.cpu().numpy(), want) else res["errors"]).append("retry")
        elif scenario == "host":
            # the reference's call shape: numpy buffers in, reduced in place;
            # chunked H2D / range all-reduce / D2H pipeline (bit-exact)
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
            e = 20_000_003
            arrays = member_inputs(world, e, seed=31)
            cfg = ftar.PipelineConfig(chunk_bytes=1 << 20, max_in_flight=3)
            want = orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight)
            buf = arrays[rank].copy()
            assert ftar.ftar_all_reduce(group, buf, 1, cfg) is buf
            (res["ok"] if np.array_equal(buf, want) else res["errors"]).append("host_inplace")
            hb = torch.from_numpy(arrays[rank]).to(torch.bfloat16).pin_memory()
            ho = torch.empty(e).pin_memory()
            arrays16 = [torch.from_numpy(a).to(torch.bfloat16).float().numpy() for a in arrays]
            ftar.ftar_all_reduce(group, hb, 2, cfg, out=ho, scale=1.0 / world)
            want16 = orc.normalize(orc.oracle_reduce(arrays16, cfg.chunk_bytes, cfg.max_in_flight), world)
            (res["ok"] if np.array_equal(ho.numpy(), want16) else res["errors"]).append("host_bf16")
        elif scenario == "sgd":
            # §8f: all-reduce + normalisation + SGD-momentum fused, bit-exact
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
            e = 3_000_001
            arrays = member_inputs(world, e, seed=51, dtype="bf16")
            rng = np.random.default_rng(52)
            p0 = rng.standard_normal(e).astype(np.float32)
            m0 = (rng.standard_normal(e) * 0.1).astype(np.float32)
            g = torch.from_numpy(arrays[rank]).to(dev).to(torch.bfloat16)
            pt, mt = torch.from_numpy(p0).to(dev), torch.from_numpy(m0).to(dev)
            po, mo = ftar.ftar_all_reduce_sgd(group, g, 1, params=pt, momentum=mt, lr=0.01, beta=0.9,
                                              scale=1.0 / world)
            gw = orc.normalize(orc.oracle_reduce(arrays, 8 << 20, 4), world)
            pw, mw = orc.sgd_momentum(p0.copy(), m0.copy(), gw, 0.9, 0.01)
            good = np.array_equal(po.cpu().numpy(), pw) and np.array_equal(mo.cpu().numpy(), mw)
            (res["ok"] if good else res["errors"]).append("sgd")
            # queued: three buckets (bucket k = the same data x (k+1)) in flight at once, each with its
            # own optimizer state, collected in launch order
            pend, wants = [], []
            for k in range(3):
                gk = (g.float() * (k + 1)).to(torch.bfloat16)
                pend.append(ftar.ftar_all_reduce_sgd_async(group, gk, 2, params=pt, momentum=mt, lr=0.01,
                                                           beta=0.9, scale=1.0 / world))
                ak = [(torch.from_numpy(a).to(torch.bfloat16).float() * (k + 1)).to(torch.bfloat16).float().numpy()
                      for a in arrays]
                gwk = orc.normalize(orc.oracle_reduce(ak, 8 << 20, 4), world)
                wants.append(orc.sgd_momentum(p0.copy(), m0.copy(), gwk, 0.9, 0.01))
            good = True
            for pk, (pwk, mwk) in zip(pend, wants):
                pok, mok = pk.wait()
                good &= np.array_equal(pok.cpu().numpy(), pwk) and np.array_equal(mok.cpu().numpy(), mwk)
            (res["ok"] if good else res["errors"]).append("sgd_async")
        elif scenario == "death":
            # a member PROCESS dies with its kernel in flight and its arena
            # still mapped by the others: survivors get Recoverable (no CUDA
            # fault), their contexts stay usable, and they regroup without it
            import time
            victim = world - 1
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
            e = 2 << 20  # 8 MiB: fits the test pool
            b = group.alloc_bucket(e)
            b.fill_(1.0)
            o = torch.empty(e, device=dev)
            ftar.ftar_all_reduce(group, b, 0, out=o)
            torch.cuda.synchronize()
            store.set(f"armed{rank}", b"1")
            store.wait([f"armed{r}" for r in range(world)])
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=1.0)
            if rank == victim:
                res["ok"].append("victim")
                with open(os.path.join(outdir, f"r{rank}.json"), "w") as f:
                    json.dump(res, f)
                ftar.ftar_all_reduce_async(group, b, 1, cfg, out=o)
                time.sleep(0.0002)
                os._exit(0)
            t0 = time.monotonic()
            try:
                for i in range(3):
                    ftar.ftar_all_reduce(group, b, 1 + i, cfg, out=o)
                res["errors"].append("no error")
            except errors.Recoverable:
                if time.monotonic() - t0 > 2 * cfg.per_chunk_timeout_s + 1.0:
                    res["errors"].append("slow")
                res["ok"].append("recoverable")
            survivors = [r for r in range(world) if r != victim]
            group.reconfig({r: ftar.PeerAddress(r) for r in survivors}, 2, deadline_s=30)
            b.fill_(1.0)
            ftar.ftar_all_reduce(group, b, 9, cfg, out=o)
            (res["ok"] if torch.all(o == float(len(survivors))).item() else res["errors"]).append("regrouped")
            store.set(f"fin{victim}", b"1")  # the victim cannot
        elif scenario == "async_failure":
            # a member skips a step while the others have 4 buckets queued:
            # every handle resolves Recoverable, the host and device queues end
            # empty, and after the regroup a fresh queue of buckets is bit-exact
            # (a stale handle left behind would collect a later op's status).
            # Two-shot buckets first, then small-path ones (push one-shot, PDL).
            import time

            from paper_2602_00277_b200 import _lib
            victim = world - 1
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=1.0)
            for rnd, e in enumerate((300_007, 50_021)):
                g0 = 1 + 2 * rnd
                group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, g0, deadline_s=30)
                bks = [member_inputs(world, e, seed=200 + 10 * rnd + b) for b in range(6)]
                bufs = [torch.from_numpy(bk[rank]).to(dev) for bk in bks]
                outs = [torch.empty_like(b) for b in bufs]
                if rank != victim:
                    pend = [ftar.ftar_all_reduce_async(group, bufs[i], 1, cfg, out=outs[i]) for i in range(4)]
                    failed = 0
                    for p in pend:
                        try:
                            p.wait()
                        except errors.Recoverable:
                            failed += 1
                    (res["ok"] if failed == 4 else res["errors"]).append(f"all_failed:{failed}")
                    left = _lib.lib.ftar_inflight(group.ctx)
                    (res["ok"] if not group._pending and left == 0 else res["errors"]).append("queues_empty")
                    store.set(f"af_failed{rnd}_{rank}", b"1")
                else:
                    store.wait([f"af_failed{rnd}_{r}" for r in range(world - 1)])
                    time.sleep(0.1)
                group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, g0 + 1, deadline_s=30)
                pend = [ftar.ftar_all_reduce_async(group, b, 2, cfg, out=o, scale=0.5) for b, o in zip(bufs, outs)]
                for p in pend:
                    p.wait()
                good = all(np.array_equal(o.cpu().numpy(), orc.oracle_reduce(bk, 8 << 20, 4) * np.float32(0.5))
                           for bk, o in zip(bks, outs))
                (res["ok"] if good else res["errors"]).append(f"regrouped_queue{rnd}")
        elif scenario == "fuzz":
            os.environ["FTAR_TMA_MIN_SLICE_MIB"] = "0"  # the bulk-copy path at every size it can take
            # randomized mixes of every mode, the same seeded sequence on every
            # rank: sizes across the small-bucket and two-shot paths, fp32 and
            # bf16, registered and staged inputs, in place / out of place, with
            # and without scale, contributor subsets, 1-4 calls queued
            rng = np.random.default_rng(4321)
            gen = 0
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=10)
            pool_left = [group.alloc_bucket(900_000), group.alloc_bucket(900_000, torch.bfloat16)]
            for it in range(25):
                gen += 1
                contrib = [r for r in range(world) if rng.random() < 0.8] or [0]
                group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, gen, deadline_s=30,
                               contributors=contrib)
                depth = int(rng.integers(1, 5))
                jobs = []
                for k in range(depth):
                    elems = int(np.exp(rng.uniform(0, np.log(2_500_000))))
                    bf16 = bool(rng.random() < 0.4)
                    reg = bool(rng.random() < 0.5) and elems <= 900_000
                    inplace = (not bf16) and bool(rng.random() < 0.4)
                    scale = float(rng.choice([0.5, 1.0 / 3.0])) if rng.random() < 0.6 else None
                    seed = int(rng.integers(1 << 30))
                    arrays = member_inputs(world, elems, seed=seed, dtype="bf16" if bf16 else "f32")
                    if reg:
                        x = pool_left[1 if bf16 else 0][:elems]
                        x.copy_(torch.from_numpy(arrays[rank]).to(dev).to(torch.bfloat16 if bf16 else torch.float32))
                    else:
                        x = torch.from_numpy(arrays[rank]).to(dev)
                        if bf16:
                            x = x.to(torch.bfloat16)
                    out = None if inplace else torch.empty(elems, device=dev)
                    pend = ftar.ftar_all_reduce_async(group, x, it, cfg, out=out, scale=scale)
                    result = x if inplace else out
                    if reg:
                        pend.wait()  # the registered scratch is reused by the next job,
                        if inplace:  # which would overwrite an in-place result living in it
                            result = x.clone()
                    jobs.append((pend, arrays, scale, result, (elems, bf16, reg, inplace, scale)))
                for pend, arrays, sc, res_t, desc in jobs:
                    pend.wait()
                    want = orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight,
                                             contrib=[r in contrib for r in range(world)])
                    if sc is not None:
                        want = want * np.float32(ftar._f32(sc))
                    good = np.array_equal(res_t.float().cpu().numpy(), want)
                    (res["ok"] if good else res["errors"]).append(f"fuzz{it}:{desc}")
        elif scenario == "chain":
            # queued IN-PLACE calls on the same buffers: call k+1 reads what
            # call k wrote, so programmatic dependent launch must never let
            # k+1 publish or push its input before k has finished writing it
            # (small push one-shot and two-shot kernels, alternating)
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=10)
            # not 1/world: identical inputs must still change every call, or a
            # read of the previous call's output before it is final would go unseen
            scale = 1.0 / 3.0
            for elems in (65_537, 1_048_579, 200_003):  # small path, two-shot, small path
                arrays = member_inputs(world, elems, seed=700 + elems % 97)
                x = group.alloc_bucket(elems) if elems * 4 <= (8 << 20) else torch.empty(elems, device=dev)
                x.copy_(torch.from_numpy(arrays[rank]).to(dev))
                pend = [ftar.ftar_all_reduce_async(group, x, k, cfg, out=None, scale=scale) for k in range(3)]
                pend += [ftar.ftar_all_reduce_async(group, x, 3 + k, cfg, scale=scale) for k in range(3)]
                for p_ in pend:
                    p_.wait()
                want = [a.copy() for a in arrays]
                for _ in range(6):
                    r = orc.normalize(orc.oracle_reduce(want, 8 << 20, 4), 3)
                    want = [r] * world
                (res["ok"] if np.array_equal(x.cpu().numpy(), want[0]) else res["errors"]).append(f"chain{elems}")
            # alternate sizes inside one queue (small -> two-shot -> small), in place
            a_small = group.alloc_bucket(70_001)
            b_big = torch.empty(1_500_007, device=dev)
            sa = member_inputs(world, 70_001, seed=801)
            sb = member_inputs(world, 1_500_007, seed=802)
            a_small.copy_(torch.from_numpy(sa[rank]).to(dev))
            b_big.copy_(torch.from_numpy(sb[rank]).to(dev))
            pend = []
            for k in range(4):
                pend.append(ftar.ftar_all_reduce_async(group, a_small, k, cfg, scale=scale))
                pend.append(ftar.ftar_all_reduce_async(group, b_big, k, cfg, scale=scale))
            for p_ in pend:
                p_.wait()
            for arrays, t, tag in ((sa, a_small, "mix_small"), (sb, b_big, "mix_big")):
                want = [a.copy() for a in arrays]
                for _ in range(4):
                    r = orc.normalize(orc.oracle_reduce(want, 8 << 20, 4), 3)
                    want = [r] * world
                (res["ok"] if np.array_equal(t.cpu().numpy(), want[0]) else res["errors"]).append(tag)
        elif scenario == "intra":
            # §8f rank 2: the replica's ranks reduce-scatter / all-gather over
            # NVLink (one process per GPU), bit-exact vs the reference goldens
            from paper_2602_00277_b200.intra import IntraRank, segment_bounds
            ir = IntraRank(rank, world, StoreFabric(dist.PrefixStore("intra/0", store)), device=dev,
                           max_bytes=16 << 20, pool_bytes=48 << 20)
            with open(os.path.join(ROOT, "tests", "golden", "intra_cases.json")) as f:
                cases = [c for c in json.load(f) if c["n"] == world]
            for c in cases:
                vecs = member_inputs(world, c["total"], c["seed"], c["kind"])
                bounds = [tuple(b) for b in c["bounds"]]
                v = torch.from_numpy(vecs[rank]).to(dev)
                if c["kind"] == "bf16":
                    v = v.to(torch.bfloat16)
                shard = ir.reduce_scatter(rank, v, bounds)
                full = ir.all_gather(rank, shard, bounds, c["total"])
                good = sha(shard.cpu().numpy()) == c["rs_sha"][rank] and sha(full.cpu().numpy()) == c["ag_sha"]
                (res["ok"] if good else res["errors"]).append(f"intra{c['seed']}")
            # registered (zero-copy) bf16 vector, 4M elements, segment_bounds
            total = 4_000_037
            vecs = member_inputs(world, total, 9, "bf16")
            bounds = segment_bounds(total, world)
            v = ir.alloc(total, torch.bfloat16)
            v.copy_(torch.from_numpy(vecs[rank]).to(dev).to(torch.bfloat16))
            shard = ir.reduce_scatter(rank, v, bounds)
            want = orc.intra_reduce_scatter(vecs, bounds)
            full = ir.all_gather(rank, shard, bounds, total)
            good = np.array_equal(shard.cpu().numpy(), want[rank]) and \
                np.array_equal(full.cpu().numpy(), orc.intra_all_gather(want, bounds, total))
            (res["ok"] if good else res["errors"]).append("intra_big")
            # queued: RS -> AG -> RS back to back (the AG reads the RS output)
            sh = torch.empty(bounds[rank][1], device=dev)
            p1 = ir.reduce_scatter_async(v, bounds, out=sh)
            p2 = ir.all_gather_async(sh, bounds, total)
            p3 = ir.reduce_scatter_async(v, bounds)
            s1, f2, s3 = p1.wait(), p2.wait(), p3.wait()
            good = np.array_equal(s1.cpu().numpy(), want[rank]) and np.array_equal(s3.cpu().numpy(), want[rank]) \
                and np.array_equal(f2.cpu().numpy(), orc.intra_all_gather(want, bounds, total))
            (res["ok"] if good else res["errors"]).append("intra_queued")
            ir.close()
        elif scenario == "churn":
            # 300 kill/rejoin reconfigs of one member (verdict r1 item 6): the
            # victim drops its ring group (arena freed) and rejoins as a new
            # incarnation; survivors map the new arena and unmap the dead
            # one, so the victim GPU's memory stays flat and every call is exact
            victim = world - 1
            e = 70_001
            arrays = member_inputs(world, e, seed=77)
            want = orc.oracle_reduce(arrays, 8 << 20, 4)
            group.close()
            group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=1 << 20, incarnation=0)
            free_at, bad, maxmapped = {}, 0, 0
            for it in range(300):
                if rank == victim and it > 0:
                    group.close()
                    group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=1 << 20, incarnation=it)
                group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, it + 1, deadline_s=60)
                buf = torch.from_numpy(arrays[rank]).to(dev)
                ftar.ftar_all_reduce(group, buf, it)
                bad += int(not np.array_equal(buf.cpu().numpy(), want))
                maxmapped = max(maxmapped, len(group.mapped_peers))
                if it in (20, 299):
                    torch.cuda.synchronize()
                    free_at[it] = torch.cuda.mem_get_info(dev)[0]
            (res["ok"] if bad == 0 else res["errors"]).append(f"churn_exact:{bad}")
            (res["ok"] if maxmapped <= world - 1 else res["errors"]).append(f"mapped:{maxmapped}")
            drift = free_at[20] - free_at[299]
            res["free_drift_mib"] = drift / 2**20
            (res["ok"] if drift < (64 << 20) else res["errors"]).append(f"memory_flat:{drift >> 20}MiB")
        elif scenario == "bench":
            # bench.py's bucket over NVLink: 64 Mi fp32 per replica, default
            # geometry, x f32(1/n); registered out-of-place (push all-gather),
            # registered in place, and ordinary torch tensors (the reference
            # call shape), three calls queued before the first wait
            e = 64 << 20
            group.close()
            group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=e * 4, pool_bytes=2 * e * 4 + 4096)
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=60)
            hosts = [np.random.default_rng((0, r)).standard_normal(e).astype(np.float32) for r in range(world)]
            want = orc.normalize(orc.oracle_reduce(hosts, 8 << 20, 4), world)
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=10)
            x = group.alloc_bucket(e)
            o = group.alloc_bucket(e)
            x.copy_(torch.from_numpy(hosts[rank]))
            pend = [ftar.ftar_all_reduce_async(group, x, k, cfg, out=o, scale=1.0 / world) for k in range(3)]
            for p_ in pend:
                p_.wait()
            (res["ok"] if np.array_equal(o.cpu().numpy(), want) else res["errors"]).append("bench_push")
            ftar.ftar_all_reduce(group, x, 3, cfg, scale=1.0 / world)
            (res["ok"] if np.array_equal(x.cpu().numpy(), want) else res["errors"]).append("bench_inplace")
            u = torch.from_numpy(hosts[rank]).to(dev)
            uo = torch.empty(e, device=dev)
            pend = [ftar.ftar_all_reduce_async(group, u, 4 + k, cfg, out=uo, scale=1.0 / world) for k in range(3)]
            for p_ in pend:
                p_.wait()
            (res["ok"] if np.array_equal(uo.cpu().numpy(), want) else res["errors"]).append("bench_unregistered")
            ftar.ftar_all_reduce(group, u, 7, cfg, scale=1.0 / world)
            (res["ok"] if np.array_equal(u.cpu().numpy(), want) else res["errors"]).append("bench_unreg_inplace")
        elif scenario == "queued":
            # back-to-back queued calls with DIFFERENT data per call: the early
            # PDL trigger lets a peer start call t+1 while this member is still
            # in call t, so every queued result must still be call t's own --
            # push mode with per-call outs and with one reused out (the last
            # call's result wins), pull mode (no early trigger), and the early
            # trigger forced everywhere, also on the bulk-copy path
            # (FTAR_PDL_EARLY=2, FTAR_TMA_MIN_SLICE_MIB=0); 2 MiB and 24 MiB buckets
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=10)
            # (64 Ki elements: the small one-shot, also forced onto 32 CTAs, where
            # its flags once raced with a peer's next call)
            for gen, e in ((9, 64 << 10), (10, 512 << 10), (11, 6 << 20)):
                group.close()
                group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=e * 4,
                                       pool_bytes=12 * e * 4 + 4096)
                group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, gen, deadline_s=60)
                K = 6
                hosts = [[np.random.default_rng((k, r, e)).standard_normal(e).astype(np.float32) for r in range(world)]
                         for k in range(K)]
                wants = [orc.oracle_reduce(h, cfg.chunk_bytes, cfg.max_in_flight) for h in hosts]
                xs = [group.alloc_bucket(e) for _ in range(K)]
                for x, h in zip(xs, hosts):
                    x.copy_(torch.from_numpy(h[rank]))
                outs = [group.alloc_bucket(e) for _ in range(K - 1)]
                modes = [("push", {}), ("pull", {"FTAR_NO_PUSH": "1"}),
                         ("early2", {"FTAR_PDL_EARLY": "2", "FTAR_TMA_MIN_SLICE_MIB": "0"})]
                if e == 64 << 10:
                    modes.append(("small32", {"FTAR_TEST_CTAS": "32"}))
                for mode, env in modes:
                    old_env = {k: os.environ.get(k) for k in env}
                    os.environ.update(env)
                    if "FTAR_TEST_CTAS" in env:
                        from paper_2602_00277_b200 import _lib as lib_
                        lib_.lib.ftar_set_tuning(int(env["FTAR_TEST_CTAS"]), 0)
                    try:
                        for _ in range(3):
                            pend = [ftar.ftar_all_reduce_async(group, xs[k], k, cfg, out=outs[k]) for k in range(K - 1)]
                            for p_ in pend:
                                p_.wait()
                            good = all(np.array_equal(outs[k].cpu().numpy(), wants[k]) for k in range(K - 1))
                            (res["ok"] if good else res["errors"]).append(f"queued_{mode}_{e}")
                            shared = outs[0]
                            pend = [ftar.ftar_all_reduce_async(group, xs[k], k, cfg, out=shared) for k in range(K)]
                            for p_ in pend:
                                p_.wait()
                            good = np.array_equal(shared.cpu().numpy(), wants[K - 1])
                            (res["ok"] if good else res["errors"]).append(f"queued_shared_{mode}_{e}")
                    finally:
                        if "FTAR_TEST_CTAS" in env:
                            lib_.lib.ftar_set_tuning(0, 0)
                        for k, v in old_env.items():
                            if v is None:
                                os.environ.pop(k, None)
                            else:
                                os.environ[k] = v
        elif scenario == "register":
            # ordinary torch tensors registered with the ring (RingGroup.register):
            # zero-copy in place and push into a registered out; a member that
            # rejoins as a new incarnation registers before its reconfig and the
            # others map its buffers at the reconfig
            e = 3_000_017
            arrays = member_inputs(world, e, seed=61)
            want = orc.oracle_reduce(arrays, 8 << 20, 4)
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=10)
            os.environ["FTAR_TMA_MIN_SLICE_MIB"] = "0"
            x = torch.from_numpy(arrays[rank]).to(dev)
            o = torch.empty(e, device=dev)
            group.register(x)
            group.register(o)
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
            ftar.ftar_all_reduce(group, x, 1, cfg, out=o, scale=0.5)
            (res["ok"] if np.array_equal(o.cpu().numpy(), want * np.float32(0.5)) else res["errors"]).append("push")
            ftar.ftar_all_reduce(group, x, 2, cfg)
            (res["ok"] if np.array_equal(x.cpu().numpy(), want) else res["errors"]).append("inplace")
            victim = world - 1
            if rank == victim:
                group.close()
                group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=64 << 20, incarnation=1)
                x = torch.from_numpy(arrays[rank]).to(dev)
                group.register(x)  # links are down: published now, mapped by the others at the reconfig
            else:
                x.copy_(torch.from_numpy(arrays[rank]))
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 2, deadline_s=30)
            ftar.ftar_all_reduce(group, x, 3, cfg)
            (res["ok"] if np.array_equal(x.cpu().numpy(), want) else res["errors"]).append("after_rejoin")
            # a late registration inside a generation is a collective round
            y = torch.from_numpy(arrays[rank]).to(dev)
            group.register(y)
            ftar.ftar_all_reduce(group, y, 4, cfg)
            (res["ok"] if np.array_equal(y.cpu().numpy(), want) else res["errors"]).append("late_register")
        elif scenario == "fetch":
            # the reference's fetch_shard(addr, step, rank, replica_id,
            # incarnation, timeout_s) shape across processes
            # (tests/test_checkpoint.py:41-95 with tensor buffers)
            from paper_2602_00277_b200 import checkpoint as ck
            snap = ck.SnapshotStore(capacity_bytes=16 << 20, device=dev, fabric=fabric, rank=0, replica_id=rank,
                                    incarnation=1)
            rec = world - 1
            donors = list(range(world - 1))
            params = torch.arange(10, dtype=torch.float32, device=dev)
            momentum = torch.ones(5, dtype=torch.float32, device=dev)
            big = torch.randn(3 << 20, device=dev, generator=torch.Generator(device=dev).manual_seed(9))
            if rank != rec:
                snap.capture(7, params, momentum)
                torch.cuda.synchronize()
            store.set(f"f_captured{rank}", b"1")
            store.wait([f"f_captured{r}" for r in donors])
            if rank == rec:
                got = []
                for attempt in range(len(donors)):
                    d = ck.pick_donor(donors + [rec], rec, 0, attempt)
                    got.append(d)
                    gp, gm = ck.fetch_shard(ftar.PeerAddress(d), 7, rank=0, replica_id=rec, incarnation=1,
                                            timeout_s=10)
                    good = torch.equal(gp.view(torch.float32), params) and torch.equal(gm.view(torch.float32), momentum)
                    (res["ok"] if good else res["errors"]).append(f"roundtrip_from_{d}")
                (res["ok"] if sorted(got) == donors else res["errors"]).append("rotation")
                try:
                    ck.fetch_shard(ftar.PeerAddress(0), 6, rank=0, replica_id=rec, incarnation=1, timeout_s=10)
                    res["errors"].append("stale step served")
                except ck.SnapshotUnavailable as exc:
                    (res["ok"] if exc.available == 7 else res["errors"]).append("unavailable")
                try:
                    ck.fetch_shard(ftar.PeerAddress(99), 1, rank=0, replica_id=rec, incarnation=1, timeout_s=0.4)
                    res["errors"].append("dead donor served")
                except errors.Recoverable:
                    res["ok"].append("dead_donor_recoverable")
                store.set("f_fetched", b"1")
                store.wait(["f_recaptured"])
                try:
                    ck.fetch_shard(ftar.PeerAddress(0), 7, rank=0, replica_id=rec, incarnation=1, timeout_s=10)
                    res["errors"].append("overwritten step served")
                except ck.SnapshotUnavailable as exc:
                    (res["ok"] if exc.available == 8 else res["errors"]).append("moved_on")
                gp, gm = ck.fetch_shard(ftar.PeerAddress(0), 8, rank=0, replica_id=rec, incarnation=1, timeout_s=10)
                (res["ok"] if torch.equal(gp.view(torch.float32), big) else res["errors"]).append("big_shard")
            elif rank == 0:
                store.wait(["f_fetched"])
                snap.capture(8, big, momentum)
                torch.cuda.synchronize()
                store.set("f_recaptured", b"1")
            store.set(f"f_done{rank}", b"1")
            store.wait([f"f_done{r}" for r in range(world)])
            snap.close()
        elif scenario == "zombie":
            # a member dropped on timeout that resumes and
            # pushes its old generation's small-bucket call late, with its old
            # ring index, must never corrupt the regrouped ring's results
            # (replica 1 leaves {0,1,2,..}: replica 2 takes ring index 1)
            import time
            victim = 1
            cfg = ftar.PipelineConfig(per_chunk_timeout_s=1.0)
            e = 65_537  # the small-bucket (push one-shot) path
            group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
            arrays = member_inputs(world, e, seed=91)
            buf = torch.from_numpy(arrays[rank]).to(dev)
            ftar.ftar_all_reduce(group, buf, 1, cfg)
            (res["ok"] if np.array_equal(buf.cpu().numpy(), orc.oracle_reduce(arrays, 8 << 20, 4))
             else res["errors"]).append("gen1")
            store.set(f"z1_{rank}", b"1")
            store.wait([f"z1_{r}" for r in range(world)])
            survivors = [r for r in range(world) if r != victim]
            if rank == victim:
                store.wait(["z_regrouped"])
                junk = torch.full((e,), 1.0e6, device=dev)
                for k in range(20):  # the zombie: stale generation, stale mappings, late
                    try:
                        ftar.ftar_all_reduce(group, junk.clone(), 10 + k, cfg)
                    except errors.FtdpError:
                        pass
                    group._links_up = True  # keep pushing as a confused replica would
                store.set("z_zombie_done", b"1")
                res["ok"].append("victim")
            else:
                try:
                    ftar.ftar_all_reduce(group, torch.from_numpy(arrays[rank]).to(dev), 2, cfg)
                    res["errors"].append("no error without the victim")
                except errors.Recoverable:
                    pass
                gen, it, wrong, okc, retried = 2, 0, 0, 0, 0
                sub = [arrays[r] for r in survivors]
                want = orc.oracle_reduce(sub, 8 << 20, 4)
                group.reconfig({r: ftar.PeerAddress(r) for r in survivors}, gen, deadline_s=30)
                if rank == survivors[0]:
                    store.set("z_regrouped", b"1")
                t_end = None
                while True:
                    it += 1
                    b = torch.from_numpy(arrays[rank]).to(dev)
                    st = b"ok"
                    try:
                        ftar.ftar_all_reduce(group, b, it, cfg)
                        if np.array_equal(b.cpu().numpy(), want):
                            okc += 1
                        else:
                            wrong += 1
                    except errors.Recoverable:
                        st = b"retry"
                    store.set(f"z_it{it}_{rank}", st)
                    store.wait([f"z_it{it}_{r}" for r in survivors])
                    if any(store.get(f"z_it{it}_{r}") != b"ok" for r in survivors):
                        retried += 1
                        gen += 1
                        group.reconfig({r: ftar.PeerAddress(r) for r in survivors}, gen, deadline_s=30)
                    if t_end is None and store.check(["z_zombie_done"]):
                        t_end = it + 20
                    if (t_end is not None and it >= t_end) or it > 2000:
                        break
                res["zombie"] = {"calls": it, "ok": okc, "wrong": wrong, "regroups": retried}
                (res["ok"] if wrong == 0 else res["errors"]).append(f"never_wrong:{wrong}")
                (res["ok"] if okc > 0 else res["errors"]).append("progress")
        elif scenario == "catchup":
            from paper_2602_00277_b200 import checkpoint as ck
            snap = ck.SnapshotStore(capacity_bytes=64 << 20, device=dev, fabric=fabric, rank=0, replica_id=rank)
            rec = world - 1
            donors = list(range(world - 1))
            g = torch.Generator(device=dev).manual_seed(3)
            p = torch.randn(8 << 20 >> 2, device=dev, generator=g)
            m = torch.randn(8 << 20 >> 2, device=dev, generator=g)
            if rank != rec:  # every healthy replica holds the same retention-1 snapshot
                snap.capture(5, p, m)
                torch.cuda.synchronize()
            store.set(f"captured{rank}", b"1")
            store.wait([f"captured{r}" for r in donors])
            if rank == rec:
                g0 = torch.Generator(device=dev).manual_seed(3)
                wp = torch.randn(8 << 20 >> 2, device=dev, generator=g0)
                wm = torch.randn(8 << 20 >> 2, device=dev, generator=g0)
                po, mo = torch.empty_like(p), torch.empty_like(m)
                snap.connect(donors, 0, timeout_s=10, background=True)  # the fetch joins it
                ck.fetch_shard(0, 5, 0, local=snap, out=(po, mo), timeout_s=10)
                (res["ok"] if not snap.connecting() else res["errors"]).append("connected")
                (res["ok"] if torch.equal(po, wp) and torch.equal(mo, wm) else res["errors"]).append("pull")
                po.zero_()
                mo.zero_()
                ck.start_fetch(snap, donors, 5, 0, po, mo, timeout_s=10).wait()  # striped over all donors
                (res["ok"] if torch.equal(po, wp) and torch.equal(mo, wm) else res["errors"]).append("striped")
                try:
                    ck.fetch_shard(0, 4, 0, local=snap, out=(po, mo), timeout_s=10)
                    res["errors"].append("stale step served")
                except ck.SnapshotUnavailable as exc:
                    (res["ok"] if exc.available == 5 else res["errors"]).append("unavailable")
            store.set(f"done{rank}", b"1")
            store.wait([f"done{r}" for r in range(world)])
    except Exception as exc:  # noqa: BLE001
        import traceback
        res["errors"].append(f"exception: {exc!r}\n{traceback.format_exc()}")
    finally:
        store.set(f"fin{rank}", b"1")
        try:
            store.wait([f"fin{r}" for r in range(world)], timedelta(seconds=60))
        except Exception:  # noqa: BLE001
            pass
        group.close()
        with open(os.path.join(outdir, f"r{rank}.json"), "w") as f:
            json.dump(res, f)


def run(scenario, world):
    with tempfile.TemporaryDirectory() as d:
        for attempt in range(4):
            # free_port() cannot reserve the port: another process may take it
            # before rank 0's TCPStore binds (EADDRINUSE) -- then retry on a new one
            port = free_port()
            try:
                mp.start_processes(_worker, args=(world, port, scenario, d), nprocs=world, join=True,
                                   start_method="spawn")
                break
            except mp.ProcessRaisedException as exc:
                if "EADDRINUSE" not in str(exc) or attempt == 3:
                    raise
        out = []
        for r in range(world):
            with open(os.path.join(d, f"r{r}.json")) as f:
                out.append(json.load(f))
    return out


def world_size():
    return min(torch.cuda.device_count(), 8)


def test_golden_cases_over_nvlink():
    res = run("golden", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert "big_bf16" in r["ok"]


def test_member_failure_requorum_and_retry():
    res = run("failure", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
    survivors = [r for r in res if "victim" not in r["ok"]]
    assert all(any(x.startswith("recoverable") for x in r["ok"]) for r in survivors)
    assert all("retry" in r["ok"] for r in survivors)


def test_host_buffers_over_nvlink():
    res = run("host", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert "host_inplace" in r["ok"] and "host_bf16" in r["ok"]


def test_queued_calls_keep_their_own_results():
    res = run("queued", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert any(x.startswith("queued_push") for x in r["ok"]) and any(x.startswith("queued_pull") for x in r["ok"])


def test_fused_sgd_over_nvlink():
    res = run("sgd", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert "sgd" in r["ok"] and "sgd_async" in r["ok"]


def test_member_process_death_is_recoverable():
    world = world_size()
    res = run("death", world)
    for r in res[:-1]:
        assert not r["errors"], r["errors"]
        assert "recoverable" in r["ok"] and "regrouped" in r["ok"]


def test_failed_async_queue_is_drained():
    world = world_size()
    res = run("async_failure", world)
    for r in res:
        assert not r["errors"], r["errors"]
        assert "regrouped_queue0" in r["ok"] and "regrouped_queue1" in r["ok"]
    for r in res[:-1]:
        assert r["ok"].count("all_failed:4") == 2 and r["ok"].count("queues_empty") == 2


def test_randomized_mode_mix_is_exact():
    res = run("fuzz", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert len(r["ok"]) >= 25


def test_queued_in_place_chains_are_exact():
    res = run("chain", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert {"mix_small", "mix_big"} <= set(r["ok"]) and sum(x.startswith("chain") for x in r["ok"]) == 3


def test_intra_replica_collectives_over_nvlink():
    res = run("intra", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert "intra_big" in r["ok"] and "intra_queued" in r["ok"] and len(r["ok"]) >= 3


def test_catchup_pull_over_nvlink():
    world = world_size()
    res = run("catchup", world)
    rec = res[world - 1]
    assert not rec["errors"], rec["errors"]
    assert {"connected", "pull", "striped", "unavailable"} <= set(rec["ok"])


def test_zombie_member_never_corrupts_regrouped_ring():
    world = world_size()
    if world < 3:
        pytest.skip("needs >= 3 GPUs (a survivor must take the zombie's ring index)")
    res = run("zombie", world)
    for r in res:
        assert not r["errors"], (r["errors"], r.get("zombie"))


def test_kill_rejoin_churn_keeps_memory_flat():
    """300 kill/rejoin reconfigs of one member: bit-exact every time, at most
    world-1 peer arenas mapped, and the victim GPU's free memory flat (dead
    incarnations' arenas are unmapped, so their memory is released)."""
    res = run("churn", world_size())
    for r in res:
        assert not r["errors"], (r["errors"], r.get("free_drift_mib"))
        assert "churn_exact:0" in r["ok"]


def test_bench_workload_over_nvlink():
    res = run("bench", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert {"bench_push", "bench_inplace", "bench_unregistered", "bench_unreg_inplace"} <= set(r["ok"])


def test_registered_user_tensors():
    res = run("register", world_size())
    for r in res:
        assert not r["errors"], r["errors"]
        assert {"push", "inplace", "after_rejoin", "late_register"} <= set(r["ok"])


def test_reference_shaped_fetch_shard():
    world = world_size()
    res = run("fetch", world)
    rec = res[world - 1]
    assert not rec["errors"], rec["errors"]
    assert {"rotation", "unavailable", "dead_donor_recoverable", "moved_on", "big_shard"} <= set(rec["ok"])


def _async_worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import numpy as np
    import torch.distributed as dist
    from datetime import timedelta

    from gen import member_inputs
    from oracle import ftar_oracle as orc
    from paper_2602_00277_b200 import ftar
    from paper_2602_00277_b200.fabric import StoreFabric

    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    store = dist.TCPStore("127.0.0.1", port, world, rank == 0, timeout=timedelta(seconds=60))
    fabric = StoreFabric(dist.PrefixStore("async", store))
    res = {"rank": rank, "ok": [], "errors": []}
    group = ftar.RingGroup(rank, 0, fabric, device=dev, max_bucket_bytes=16 << 20)
    try:
        group.reconfig({r: ftar.PeerAddress(r) for r in range(world)}, 1, deadline_s=30)
        buckets = [member_inputs(world, 1_000_003 + 7 * b, seed=100 + b) for b in range(7)]
        bufs = [torch.from_numpy(bk[rank]).to(dev) for bk in buckets]
        outs = [torch.empty_like(b) for b in bufs]
        pend = [ftar.ftar_all_reduce_async(group, b, 1, out=o, scale=0.5) for b, o in zip(bufs, outs)]
        for p in reversed(pend):  # waiting a later one collects the earlier ones first
            p.wait()
        for bk, o in zip(buckets, outs):
            want = orc.normalize(orc.oracle_reduce(bk, 8 << 20, 4), 2) if world == 2 else None
            if want is None:
                want = orc.oracle_reduce(bk, 8 << 20, 4) * np.float32(0.5)
            (res["ok"] if np.array_equal(o.cpu().numpy(), want) else res["errors"]).append("bucket")
    except Exception as exc:  # noqa: BLE001
        import traceback
        res["errors"].append(f"exception: {exc!r}\n{traceback.format_exc()}")
    finally:
        store.set(f"fin{rank}", b"1")
        store.wait([f"fin{r}" for r in range(world)], timedelta(seconds=60))
        group.close()
        with open(os.path.join(outdir, f"r{rank}.json"), "w") as f:
            json.dump(res, f)


def test_async_queue_of_buckets():
    world = world_size()
    port = free_port()
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_async_worker, args=(world, port, d), nprocs=world, join=True, start_method="spawn")
        for r in range(world):
            with open(os.path.join(d, f"r{r}.json")) as f:
                res = json.load(f)
            assert not res["errors"], res["errors"]
            assert res["ok"].count("bucket") == 7


def test_hsdp_step_with_ranks_is_bit_exact():
    """tools/hsdp_r.py --check: R=2 ranks per replica on every visible GPU,
    intra RS -> FTAR+SGD -> intra AG for 4 steps, final params bit-exact
    against the oracle on every rank."""
    import subprocess
    world = world_size()
    if world % 2:
        pytest.skip("needs an even number of GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.join(ROOT, "tools", "hsdp_r.py"),
           "--ranks", "2", "--params", "3000017", "--steps", "4", "--check"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["all_ranks_identical_params"] and line["bit_exact_vs_oracle"], line


def test_buffer_on_another_gpu_is_rejected():
    """The kernel runs on the group's GPU; a tensor living on another GPU is an
    invariant violation, not a silent peer read."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    sys.path.insert(0, ROOT)
    from paper_2602_00277_b200 import errors, ftar
    g = ftar.RingGroup(0, 0, device=torch.device("cuda", 0))
    try:
        with pytest.raises(errors.Fatal):
            ftar.ftar_all_reduce(g, torch.ones(16, device="cuda:1"), 0)
        with pytest.raises(errors.Fatal):
            ftar.ftar_all_reduce(g, torch.ones(16, device="cuda:0"), 0, out=torch.empty(16, device="cuda:1"))
        assert torch.equal(ftar.ftar_all_reduce(g, torch.ones(16, device="cuda:0"), 0), torch.ones(16, device="cuda:0"))
    finally:
        g.close()
