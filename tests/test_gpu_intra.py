"""Intra-replica collectives on the GPU, in the
reference's own test shape: one IntraGroup, R rank threads
(tests/test_replica.py:34-97), every golden case recorded from the
reference's IntraGroup (tests/golden/intra_cases.json), bit-exact."""

import hashlib
import json
import os
import sys
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, GOLD)

from gen import member_inputs  # noqa: E402


def sha(a):
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def run_ranks(n, fn):
    out, errs = [None] * n, [None] * n

    def main(r):
        try:
            out[r] = fn(r)
        except BaseException as exc:  # noqa: BLE001
            errs[r] = exc

    ts = [threading.Thread(target=main, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    assert not any(t.is_alive() for t in ts), "rank thread hung"
    for e in errs:
        if e is not None:
            raise e
    return out


@pytest.fixture(scope="module")
def intra():
    from paper_2602_00277_b200 import intra as m
    return m


_groups = {}


def group(intra, n):
    if n not in _groups:
        _groups[n] = intra.IntraGroup(n, device=torch.device("cuda", 0), max_bytes=8 << 20)
    return _groups[n]


def test_reduce_scatter_hand_values(intra):
    g = group(intra, 2)
    vecs = [np.array([1, 2, 3, 4], dtype=np.float32), np.array([10, 20, 30, 40], dtype=np.float32)]
    shards = run_ranks(2, lambda r: g.reduce_scatter(r, vecs[r], [(0, 2), (2, 2)]))
    assert shards[0].tolist() == [11.0, 22.0]
    assert shards[1].tolist() == [33.0, 44.0]


def test_all_gather_restores_full_vector(intra):
    g = group(intra, 3)
    full = np.arange(10, dtype=np.float32)
    b = [(0, 4), (4, 3), (7, 3)]
    outs = run_ranks(3, lambda r: g.all_gather(r, full[b[r][0]:b[r][0] + b[r][1]].copy(), b, 10))
    for got in outs:
        assert np.array_equal(got, full)


def test_broadcast_and_exchange(intra):
    g = group(intra, 4)
    assert run_ranks(4, lambda r: g.broadcast(r, "payload" if r == 0 else None)) == ["payload"] * 4
    assert all(o == [0, 1, 4, 9] for o in run_ranks(4, lambda r: g.exchange(r, r * r)))


def _cases():
    with open(os.path.join(GOLD, "intra_cases.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"n{c['n']}-e{c['total']}-{c['kind']}-s{c['seed']}")
def test_golden_case(intra, case):
    n, total, bounds = case["n"], case["total"], [tuple(b) for b in case["bounds"]]
    vecs = member_inputs(n, total, case["seed"], case["kind"])
    g = group(intra, n)
    if case["kind"] == "bf16":  # the bf16 bucket itself, upcast exactly in the fold
        ins = [torch.from_numpy(v).cuda().to(torch.bfloat16) for v in vecs]
    else:
        ins = vecs
    shards = run_ranks(n, lambda r: g.reduce_scatter(r, ins[r], bounds))
    assert [sha(s) for s in shards] == case["rs_sha"]
    full = run_ranks(n, lambda r: g.all_gather(r, shards[r], bounds, total))
    assert all(sha(f) == case["ag_sha"] for f in full)


def test_large_bf16_shards_cuda_tensors(intra):
    """bf16 gradients (CUDA tensors in, CUDA tensors out) at a size where the
    kernel runs many CTAs per rank; fold order checked against the oracle."""
    from oracle import ftar_oracle as orc
    from paper_2602_00277_b200.intra import segment_bounds
    n, total = 4, 3_000_017
    g = intra.IntraGroup(n, device=torch.device("cuda", 0), max_bytes=16 << 20)
    try:
        vecs = member_inputs(n, total, 77, "bf16")
        ins = [torch.from_numpy(v).cuda().to(torch.bfloat16) for v in vecs]
        bounds = segment_bounds(total, n)
        shards = run_ranks(n, lambda r: g.reduce_scatter(r, ins[r], bounds))
        want = orc.intra_reduce_scatter(vecs, bounds)
        for s, w in zip(shards, want):
            assert s.is_cuda and np.array_equal(s.cpu().numpy(), w)
        full = run_ranks(n, lambda r: g.all_gather(r, shards[r], bounds, total))
        wf = orc.intra_all_gather(want, bounds, total)
        assert all(np.array_equal(f.cpu().numpy(), wf) for f in full)
    finally:
        g.close()


def test_wrong_shard_length_is_invariant(intra):
    from paper_2602_00277_b200 import errors
    g = group(intra, 2)
    with pytest.raises(errors.Fatal):
        run_ranks(2, lambda r: g.all_gather(r, np.zeros(3, dtype=np.float32), [(0, 2), (2, 2)], 4))
