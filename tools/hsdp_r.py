"""HSDP steps with R ranks per replica (SURVEY §8f rank 2 in situ): the
reference's _RankWorker.iterate data path (replica.py:565-644) on B200.

    python -m torch.distributed.run --nproc-per-node 4 tools/hsdp_r.py --ranks 2 [--params 8e6] [--check]

Process p is rank p % R of replica p // R, one GPU each.  Per step:
  1. every rank holds a full bf16 gradient (its micro-batch; synthetic)
  2. intra-replica reduce-scatter -> fp32 shard r = sum over ranks, rank 0
     upward (replica.py:573, IntraRank over NVLink)
  3. FTAR of shard r across the replicas' rank-r ring, normalisation
     x f32(1/(h*R)) and SGD-momentum fused (replica.py:584, 622-633)
  4. intra-replica all-gather of the updated params (replica.py:640-642)
With --check (small --params), rank 0 recomputes every step with the numpy
oracle (intra fold, FTAR fold, normalisation, SGD) and asserts bit-equality
of the final params on every rank.  Rank 0 prints one JSON line.
"""

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
    ap.add_argument("--ranks", type=int, default=2)
    ap.add_argument("--params", type=float, default=1e9)
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--beta", type=float, default=0.9)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2602_00277_b200 import ftar
    from paper_2602_00277_b200.fabric import StoreFabric
    from paper_2602_00277_b200.intra import IntraRank, segment_bounds

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    dist.init_process_group("gloo")
    p, world = dist.get_rank(), dist.get_world_size()
    R = args.ranks
    assert world % R == 0, "world must be a multiple of --ranks"
    reps = world // R
    rid, rank = p // R, p % R
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", p)))
    torch.cuda.set_device(dev)
    store = dist.distributed_c10d._get_default_store()
    P = int(args.params)
    bounds = segment_bounds(P, R)
    off, ln = bounds[rank]

    intra = IntraRank(rank, R, StoreFabric(dist.PrefixStore(f"intra/{rid}", store)), device=dev,
                      max_bytes=P * 4, pool_bytes=P * 2 + 64 * 4096)
    ring = ftar.RingGroup(rid, rank, StoreFabric(dist.PrefixStore("ftar", store)), device=dev,
                          max_bucket_bytes=ln * 4 + 4096)
    ring.reconfig({m: ftar.PeerAddress(m, rank) for m in range(reps)}, 1, deadline_s=60)

    def grad_of(step, r_id, r_rank, device):  # synthetic micro-batch gradient (bf16)
        g = torch.Generator(device=device).manual_seed(1000 * step + 17 * r_id + r_rank)
        return torch.randn(P, device=device, generator=g).to(torch.bfloat16)

    g0 = torch.Generator(device=dev).manual_seed(7)
    params = (torch.randn(P, device=dev, generator=g0) * 0.02)
    mom = torch.zeros(ln, device=dev)
    gfull = intra.alloc(P, torch.bfloat16)
    shard = torch.empty(ln, device=dev)
    scale = 1.0 / (reps * R)  # healthy = every replica (no failures in this driver)
    cfg = ftar.PipelineConfig()
    times = []
    for step in range(1, args.steps + 1):
        gfull.copy_(grad_of(step, rid, rank, dev))
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.monotonic()
        intra.reduce_scatter(rank, gfull, bounds, out=shard)
        p_new, m_new = ftar.ftar_all_reduce_sgd(ring, shard, step, cfg, params=params[off:off + ln], momentum=mom,
                                                lr=args.lr, beta=args.beta, scale=scale)
        mom = m_new
        params = intra.all_gather(rank, p_new, bounds, P)
        torch.cuda.synchronize()
        times.append(time.monotonic() - t0)
    dig = hashlib.sha256(params.cpu().numpy().tobytes()).hexdigest()
    digs = [None] * world
    dist.all_gather_object(digs, dig)
    ok = None
    if args.check and p == 0:
        sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
        from oracle import ftar_oracle as orc
        # same initial params as the GPUs (same CUDA generator), then every
        # step restated on the CPU: intra fold rank 0 upward, FTAR fold across
        # replicas, x f32(1/(h*R)), SGD-momentum
        pw = (torch.randn(P, device=dev, generator=torch.Generator(device=dev).manual_seed(7)) * 0.02).cpu().numpy()
        mw = [np.zeros(b[1], dtype=np.float32) for b in bounds]
        for step in range(1, args.steps + 1):
            rs = [orc.intra_reduce_scatter([grad_of(step, q, k, dev).float().cpu().numpy() for k in range(R)], bounds)
                  for q in range(reps)]  # rs[replica][rank shard]
            newp = pw.copy()
            for r, (o, n) in enumerate(bounds):
                g = orc.normalize(orc.oracle_reduce([rs[q][r] for q in range(reps)], cfg.chunk_bytes,
                                                    cfg.max_in_flight), reps * R)
                pp, mm = orc.sgd_momentum(pw[o:o + n].copy(), mw[r], g, args.beta, args.lr)
                newp[o:o + n] = pp
                mw[r] = mm
            pw = newp
        ok = hashlib.sha256(pw.astype(np.float32).tobytes()).hexdigest() == digs[0]
    if p == 0:
        steady = sorted(times[1:])[len(times[1:]) // 2] if len(times) > 1 else times[0]
        print(json.dumps({"config": "HSDP steps, R ranks per replica: intra RS -> FTAR+SGD -> intra AG",
                          "replicas": reps, "ranks_per_replica": R, "params": P, "steps": args.steps,
                          "all_ranks_identical_params": len(set(digs)) == 1,
                          "bit_exact_vs_oracle": ok, "step_ms_median": round(steady * 1e3, 3),
                          "step_ms": [round(t * 1e3, 3) for t in times]}), flush=True)
    intra.close()
    ring.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
