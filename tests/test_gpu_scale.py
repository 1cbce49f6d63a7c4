"""Parity at the sizes the benchmark reports, the reference's criterion 02 in
full, and the bulk-copy (TMA) data path's geometry edge cases.

* criterion 02 (tests/test_acceptance.py:86-137): 1,000 randomized cases,
  seed 0xF7A2, N 2..8, up to 1e6 elements, the reference's own case, chunk,
  window and input RNG stream, every member bit-equal to the oracle;
* the bench workload: 4 replicas x 64 Mi fp32 (256 MiB), default geometry,
  fused x f32(1/4), out of place (push all-gather) and in place (pull), three
  calls queued before the first wait;
* 1 GiB bf16 buckets (512 Mi elements) through the protocol kernel;
* TMA tiles cut by segment boundaries at every offset mod 4, many
  partitions, ragged slice tails, behind replicas whose buffers are garbage.

All members run on cuda:0 as CTA groups of one cooperative launch of the
multi-GPU kernel (tests/test_gpu_multiproc.py runs the NVLink form).
"""

import hashlib

import numpy as np
import pytest
import torch

from oracle import ftar_oracle as orc

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)
MIB = 1 << 20


@pytest.fixture(scope="module")
def ftar():
    from paper_2602_00277_b200 import ftar as f
    return f


def _dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV).to(dtype)


def test_criterion_02_full(ftar):
    """The reference's criterion 02 case stream, bit-exact on every member."""
    rng = np.random.default_rng(0xF7A2)
    cases = [(2, 1), (8, 1), (2, 1_000_000), (4, 1_000_000), (8, 9)]
    while len(cases) < 1000:
        n = 2 + len(cases) % 7
        cases.append((n, int(10 ** rng.uniform(0, 6))))
    rings = {}
    bad = []
    tma_cases = 0
    try:
        for n, elems in cases:
            if n not in rings:
                rings[n] = ftar.LocalRing(n, device=DEV, max_bucket_bytes=4 * MIB, protocol=True)
            nbytes = elems * 4
            if nbytes <= 4096:
                chunk = int(rng.integers(1, 65)) * 4
            else:
                chunk = max(4, (nbytes >> int(rng.integers(0, 9))) & ~3)
            cfg = ftar.PipelineConfig(chunk_bytes=chunk, max_in_flight=int(rng.integers(1, 6)),
                                      per_chunk_timeout_s=30.0)
            bufs = [rng.standard_normal(elems).astype(np.float32) for _ in range(n)]
            expected = orc.oracle_reduce(bufs, cfg.chunk_bytes, cfg.max_in_flight)
            plan = orc.partition_plan(elems, cfg.chunk_bytes, cfg.max_in_flight, n)
            tma_cases += int(min(p for _, p in plan) // n >= 2048)
            dbufs = [_dev(b) for b in bufs]
            rings[n].all_reduce(dbufs, cfg)
            for rid, d in enumerate(dbufs):
                if not np.array_equal(d.cpu().numpy(), expected):
                    bad.append((n, elems, chunk, cfg.max_in_flight, rid))
            if bad:
                break
    finally:
        for r in rings.values():
            r.close()
    assert not bad, f"not bit-equal to the oracle: {bad[:5]}"
    assert tma_cases > 100  # the bulk-copy path is exercised, not only the register one


def _chunked_oracle_check(arrays_fn, n, elems, chunk_bytes, C, outs, scale=None, span=16 * MIB):
    """Compare device outputs with the oracle fold segment by segment without
    materialising whole fp32 copies of every member (1 GiB buckets)."""
    for p_off, p_len in orc.partition_plan(elems, chunk_bytes, C, n):
        s_off = p_off
        for owner, (_, s_len) in enumerate(orc.segments(p_len, n)):
            for lo in range(s_off, s_off + s_len, span):
                hi = min(lo + span, s_off + s_len)
                xs = arrays_fn(lo, hi)
                acc = xs[owner].copy()
                for k in range(1, n):
                    acc = acc + xs[(owner + k) % n]
                if scale is not None:
                    acc = acc * np.float32(scale)
                for o in outs:
                    got = o[lo:hi].cpu().numpy()
                    if not np.array_equal(got, acc):
                        return (lo, hi, int(np.sum(got != acc)))
            s_off += s_len
    return None


@pytest.mark.parametrize("inplace", [False, True], ids=["push", "inplace"])
def test_bench_workload_queued(ftar, inplace):
    """bench.py's N=1 bucket (4 x 64 Mi fp32, default geometry, x f32(1/4)),
    three launches queued before the first wait, each checked."""
    n, elems = 4, 64 * MIB
    hosts = [torch.from_numpy(np.random.default_rng((0, r)).standard_normal(elems).astype(np.float32))
             for r in range(n)]
    ring = ftar.LocalRing(n, device=DEV, max_bucket_bytes=elems * 4, protocol=True)
    try:
        cfg = ftar.PipelineConfig()
        want = orc.normalize(orc.oracle_reduce([h.numpy() for h in hosts], cfg.chunk_bytes, cfg.max_in_flight), n)
        wsha = hashlib.sha256(want.tobytes()).hexdigest()
        bufs = [h.to(DEV) for h in hosts]
        outs = bufs if inplace else [torch.full((elems,), float("nan"), device=DEV) for _ in range(n)]
        calls = 1 if inplace else 3  # in place, the second call would reduce the first's result
        toks = [ring.launch(bufs, cfg, outs=outs, scale=1.0 / n) for _ in range(calls)]
        for t in toks:
            assert ring.wait(t, cfg) == [0] * n
        for o in outs:
            assert hashlib.sha256(o.cpu().numpy().tobytes()).hexdigest() == wsha
    finally:
        ring.close()


def test_1gib_bf16_bucket(ftar):
    """1 GiB bf16 buckets (512 Mi elements) per member, fused cast + scale,
    through the protocol kernel; checked span by span against the oracle."""
    n, elems = 4, 512 * MIB
    g = torch.Generator(device=DEV).manual_seed(11)
    bufs = [torch.randn(elems, device=DEV, generator=g).to(torch.bfloat16) for _ in range(n)]
    hosts = [b.cpu() for b in bufs]
    ring = ftar.LocalRing(n, device=DEV, max_bucket_bytes=elems * 2, protocol=True)
    try:
        outs = [torch.empty(elems, device=DEV) for _ in range(n)]
        cfg = ftar.PipelineConfig()
        ring.all_reduce(bufs, cfg, outs=outs, scale=1.0 / n)
        torch.cuda.synchronize()
        del bufs

        def arrays(lo, hi):
            return [h[lo:hi].float().numpy() for h in hosts]

        bad = _chunked_oracle_check(arrays, n, elems, cfg.chunk_bytes, cfg.max_in_flight, outs,
                                    scale=np.float32(1.0 / n))
        assert bad is None, f"mismatch in [{bad[0]}, {bad[1]}): {bad[2]} elements"
    finally:
        ring.close()


def _tma_cases():
    rng = np.random.default_rng(0x7A3A)
    out = []
    for i in range(28):
        n = 2 + i % 7
        dtype = "bf16" if i % 3 == 0 else "f32"
        elems = int(rng.integers(3 * 2048 * n, 40 * 2048 * n)) + int(rng.integers(0, 8))
        # partitions of at least one tile per segment: cap = S*C*n/4 >= 2048*n
        C = int(rng.integers(1, 5))
        chunk = int(rng.integers(4 * 4096 // C + 4, 8 * 2048 * 4)) & ~3
        behind = [] if i % 4 else [int(rng.integers(0, n))]
        out.append(dict(n=n, dtype=dtype, elems=elems, chunk=chunk, C=C, behind=behind, inplace=(i % 5 == 1),
                        scale=(i % 2 == 0)))
    return out


@pytest.mark.parametrize("protocol", [True, False], ids=["protocol", "oneshot"])
@pytest.mark.parametrize("c", _tma_cases(), ids=lambda c: f"n{c['n']}-{c['dtype']}-e{c['elems']}-S{c['chunk']}-C{c['C']}"
                                                        f"-b{len(c['behind'])}{'-inplace' if c['inplace'] else ''}")
def test_tma_geometry_edges(ftar, c, protocol):
    """Multi-partition buckets whose segment boundaries fall at every offset
    within a tile, ragged slice tails, garbage in behind replicas' buffers;
    the bulk-copy path and the register path both bit-exact -- in the
    multi-GPU protocol kernel and in the in-process one-shot (local_bulk_kernel
    vs local_oneshot_kernel)."""
    n = c["n"]
    arrays = orc.member_inputs(n, c["elems"], seed=c["elems"], dtype=c["dtype"])
    contrib = [m not in c["behind"] for m in range(n)]
    garbage = [a if ok else np.full_like(a, np.nan) for a, ok in zip(arrays, contrib)]
    want = orc.oracle_reduce(arrays, c["chunk"], c["C"], contrib=contrib)
    if c["scale"]:
        want = orc.normalize(want, n)
    plan = orc.partition_plan(c["elems"], c["chunk"], c["C"], n)
    assert min(p for _, p in plan) // n >= 2048
    cfg = ftar.PipelineConfig(chunk_bytes=c["chunk"], max_in_flight=c["C"], per_chunk_timeout_s=10.0)
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    ring = ftar.LocalRing(n, device=DEV, max_bucket_bytes=c["elems"] * 4, protocol=protocol)
    try:
        ring.reconfig(contributors=[m for m in range(n) if contrib[m]])
        for tma in ("1", "0"):
            import os
            os.environ["FTAR_TMA"] = tma
            try:
                bufs = [_dev(a, tdt) for a in garbage]
                if c["inplace"] and tdt == torch.float32:
                    outs = bufs
                else:
                    outs = [torch.full((c["elems"],), float("nan"), device=DEV) for _ in range(n)]
                ring.all_reduce(bufs, cfg, outs=outs, scale=(1.0 / n) if c["scale"] else None)
                for m, o in enumerate(outs):
                    got = o.cpu().numpy()
                    assert np.array_equal(got, want), (f"FTAR_TMA={tma} member {m}: "
                                                       f"{int(np.sum(got != want))} elements differ")
            finally:
                os.environ.pop("FTAR_TMA", None)
    finally:
        ring.close()
