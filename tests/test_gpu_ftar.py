"""FTAR on the GPU vs the oracle / the reference's golden outputs.

In-process rings (all members on cuda:0, one cooperative launch per call)
exercise the same kernel, flag protocol and fold as the one-process-per-GPU
path; tests/test_gpu_multiproc.py covers the NVLink/IPC path.  Parity bar:
bit-exact (the fold order is the reference's; every fp32 op is separately
rounded), which is stricter than north_star's 1e-6 relative tolerance.
"""

import hashlib
import json
import os
import threading
import time

import numpy as np
import pytest
import torch

from gen import behind_set, case_inputs, member_inputs
from oracle import ftar_oracle as orc

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")
DEV = torch.device("cuda", 0)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def cases():
    with open(os.path.join(GOLD, "ftar_cases.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def ftar():
    from paper_2602_00277_b200 import ftar as f
    return f


@pytest.fixture(scope="module")
def rings(ftar):
    made = {}

    def get(n, protocol=True):
        if (n, protocol) not in made:
            made[(n, protocol)] = ftar.LocalRing(n, device=DEV, max_bucket_bytes=32 * 1024 * 1024,
                                                 protocol=protocol)
        return made[(n, protocol)]

    yield get
    for r in made.values():
        r.close()


def to_dev(a, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV).to(dtype)


@pytest.mark.parametrize("mode", ["protocol", "twoshot", "oneshot"])
@pytest.mark.parametrize("case", cases(), ids=lambda c: f"{c['idx']}-{c['kind']}-n{c['n']}-e{c['elems']}")
def test_golden_cases_bit_exact(ftar, rings, case, mode, monkeypatch):
    """protocol: the multi-GPU kernels (small buckets take the push one-shot);
    twoshot: the same with the small-bucket path disabled; oneshot: the
    in-process one-shot kernel."""
    if mode == "twoshot":
        monkeypatch.setenv("FTAR_SMALL_BYTES", "0")
    ring = rings(case["n"], protocol=(mode != "oneshot"))
    cfg = ftar.PipelineConfig(chunk_bytes=case["chunk_bytes"], max_in_flight=case["max_in_flight"],
                              per_chunk_timeout_s=10.0)
    behind = behind_set(case)
    arrays = case_inputs(case, garbage_behind=bool(behind))
    contributors = [m for m in range(case["n"]) if m not in behind]
    ring.reconfig(contributors=contributors)
    if case["kind"] == "bf16":
        bufs = [to_dev(a, torch.bfloat16) for a in arrays]
        outs = [torch.full((case["elems"],), float("nan"), device=DEV) for _ in arrays]
        ring.all_reduce(bufs, cfg, outs=outs)
    else:
        bufs = [to_dev(a) for a in arrays]
        outs = ring.all_reduce(bufs, cfg)
    torch.cuda.synchronize()
    for o in outs:
        assert sha(o.cpu().numpy()) == case["sha256"]


@pytest.mark.parametrize("mode", ["protocol", "oneshot"])
def test_config1_digest_and_scale(ftar, rings, mode):
    with open(os.path.join(GOLD, "config1.json")) as f:
        g = json.load(f)
    arrays = member_inputs(g["n"], g["elems"], seed=g["seed"])
    ring = rings(4, protocol=(mode == "protocol"))
    ring.reconfig()
    bufs = [to_dev(a) for a in arrays]
    ring.all_reduce(bufs)
    for b in bufs:
        assert sha(b.cpu().numpy()) == g["sha256"]
    # fused normalisation == reference's separate multiply (replica.py:626)
    bufs = [to_dev(a) for a in arrays]
    outs = [torch.empty_like(b) for b in bufs]
    ring.all_reduce(bufs, outs=outs, scale=1.0 / 3)
    want = orc.normalize(orc.oracle_reduce(arrays, g["chunk_bytes"], g["max_in_flight"]), 3)
    for o in outs:
        np.testing.assert_array_equal(o.cpu().numpy(), want)
    for b, a in zip(bufs, arrays):  # out-of-place leaves inputs alone
        np.testing.assert_array_equal(b.cpu().numpy(), a)


@pytest.mark.parametrize("mode", ["protocol", "oneshot"])
@pytest.mark.parametrize("n", [1, 2, 3, 5, 8])
def test_bf16_bucket_default_geometry(ftar, rings, n, mode):
    arrays = member_inputs(n, 1_000_003, seed=5, dtype="bf16")
    ring = rings(n, protocol=(mode == "protocol"))
    ring.reconfig()
    bufs = [to_dev(a, torch.bfloat16) for a in arrays]
    outs = [torch.empty(a.size, device=DEV) for a in arrays]
    ring.all_reduce(bufs, outs=outs)
    want = orc.oracle_reduce(arrays, 8 << 20, 4)
    for o in outs:
        np.testing.assert_array_equal(o.cpu().numpy(), want)


@pytest.mark.parametrize("mode", ["protocol", "oneshot"])
def test_nonfinite_is_fatal_everywhere_and_nothing_committed(ftar, rings, mode):
    for poison in (np.nan, np.inf):
        arrays = [np.ones(4099, dtype=np.float32) for _ in range(3)]
        arrays[1][3000] = poison
        ring = rings(3, protocol=(mode == "protocol"))
        ring.reconfig()
        bufs = [to_dev(a) for a in arrays]
        with pytest.raises(Exception) as ei:
            ring.all_reduce(bufs, ftar.PipelineConfig(chunk_bytes=64, max_in_flight=2))
        from paper_2602_00277_b200 import errors
        assert isinstance(ei.value, errors.Fatal) and ei.value.reason == errors.NUMERICAL
        for b, a in zip(bufs, arrays):
            np.testing.assert_array_equal(b.cpu().numpy(), a)


def test_fault_injection_mid_reduce_scatter_then_requorum(ftar, rings):
    """Config 2 on one GPU: 8 replicas, replica 5 stops after 1 reduce tile;
    survivors abort Recoverable within 2x per_chunk_timeout_s with buffers
    untouched, regroup without it (generation+1) and the retry matches the
    oracle over 7 members with scale f32(1/7)."""
    from paper_2602_00277_b200 import errors
    n, e = 8, 3_000_000
    arrays = member_inputs(n, e, seed=11)
    ring = rings(n)
    ring.reconfig()
    cfg = ftar.PipelineConfig(per_chunk_timeout_s=0.5)
    bufs = [to_dev(a) for a in arrays]
    t0 = time.monotonic()
    ctxs = ring.launch(bufs, cfg, fault=(5, 1))
    sts = ring.wait(ctxs, cfg)
    took = time.monotonic() - t0
    assert sts[5] == errors.ST_INJECTED
    for i, st in enumerate(sts):
        if i != 5:
            assert isinstance(errors.from_status(st), errors.Recoverable), (i, st)
    assert took < 2 * cfg.per_chunk_timeout_s + 1.0
    for b, a in zip(bufs, arrays):
        np.testing.assert_array_equal(b.cpu().numpy(), a)
    survivors = [m for m in range(n) if m != 5]
    gen_before = ring.groups[0].generation
    ring.reconfig(members=survivors)
    assert ring.groups[0].generation == gen_before + 1
    sb = [bufs[m] for m in survivors]
    outs = [torch.empty_like(b) for b in sb]
    ring.all_reduce(sb, cfg, outs=outs, scale=1.0 / 7, members=survivors)
    want = orc.normalize(orc.oracle_reduce([arrays[m] for m in survivors], cfg.chunk_bytes, cfg.max_in_flight), 7)
    for o in outs:
        np.testing.assert_array_equal(o.cpu().numpy(), want)
    ring.reconfig()  # restore full membership for other tests


@pytest.mark.parametrize("mode", ["protocol", "oneshot"])
def test_replay_reference_replica_run(ftar, rings, mode):
    """Every successful ftar_all_reduce of the reference's 8-replica
    kill/rejoin run (tests/golden/replica_ftar.npz): same members, same
    inputs (behind replicas' zeros), same outputs bit for bit."""
    z = np.load(os.path.join(GOLD, "replica_ftar.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    groups = {}
    for i, m in enumerate(meta):
        if m["error"] is None:
            groups.setdefault((m["step"], m["generation"], tuple(m["members"])), []).append(i)
    assert groups
    for (step, gen, members), idxs in sorted(groups.items()):
        by_rep = {meta[i]["replica"]: i for i in idxs}
        assert sorted(by_rep) == list(members)
        n = len(members)
        ring = rings(8, protocol=(mode == "protocol"))
        ring.reconfig(members=list(range(n)))
        chunk, C = meta[idxs[0]]["cfg"]
        cfg = ftar.PipelineConfig(chunk_bytes=chunk, max_in_flight=C)
        bufs = [to_dev(z[f"in{by_rep[r]}"]) for r in members]
        ring.all_reduce(bufs, cfg, members=list(range(n)))
        for r, b in zip(members, bufs):
            np.testing.assert_array_equal(b.cpu().numpy(), z[f"out{by_rep[r]}"])
    ring.reconfig()


# ---------------------------------------------------------------------------
# Drop-in tests in the shape of the reference's tests/test_ftar.py: one
# RingGroup per member, members calling ftar_all_reduce from threads.


class Ring:
    def __init__(self, ftar, n):
        from paper_2602_00277_b200.fabric import LocalFabric
        self.ftar = ftar
        self.n = n
        self.fabric = LocalFabric()
        self.groups = [ftar.RingGroup(rid, 0, self.fabric, device=DEV, max_bucket_bytes=4 << 20) for rid in range(n)]
        self.addrs = {rid: ftar.PeerAddress(rid, 0) for rid in range(n)}
        self.gen = 0

    def reconfig(self, members=None, skip=()):
        members = sorted(members if members is not None else range(self.n))
        self.gen += 1
        addrs = {rid: self.addrs[rid] for rid in members}
        errs = {}

        def go(rid):
            try:
                self.groups[rid].reconfig(addrs, self.gen, deadline_s=5.0)
            except Exception as exc:  # noqa: BLE001
                errs[rid] = exc

        ts = [threading.Thread(target=go, args=(r,)) for r in members if r not in skip]
        [t.start() for t in ts]
        [t.join(10) for t in ts]
        if errs:
            raise next(iter(errs.values()))
        return members

    def all_reduce(self, bufs, step, cfg, participants):
        results = {}

        def go(rid):
            try:
                results[rid] = self.ftar.ftar_all_reduce(self.groups[rid], bufs[rid], step, cfg)
            except Exception as exc:  # noqa: BLE001
                results[rid] = exc

        ts = [threading.Thread(target=go, args=(r,)) for r in participants]
        [t.start() for t in ts]
        [t.join(30) for t in ts]
        assert not any(t.is_alive() for t in ts), "all-reduce hung"
        return results

    def close(self):
        for g in self.groups:
            g.close()


def run_case(ring, members, arrays, step, cfg):
    bufs = {rid: to_dev(a) for rid, a in zip(members, arrays)}
    res = ring.all_reduce(bufs, step, cfg, members)
    for r in res.values():
        if isinstance(r, Exception):
            raise r
    want = orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight)
    for rid in members:
        assert res[rid] is bufs[rid]
        np.testing.assert_array_equal(bufs[rid].cpu().numpy(), want)


def test_dropin_hand_cases_and_membership_churn(ftar):
    ring = Ring(ftar, 4)
    try:
        ring.reconfig()
        cfg = ftar.PipelineConfig(chunk_bytes=8, max_in_flight=2)
        run_case(ring, [0, 1, 2, 3], [np.full(8, float(i), dtype=np.float32) for i in range(4)], 1, cfg)
        cfg = ftar.PipelineConfig(chunk_bytes=4, max_in_flight=1)
        run_case(ring, [0, 1, 2, 3], [np.arange(8, dtype=np.float32) * (i + 1) for i in range(4)], 2, cfg)
        run_case(ring, [0, 1, 2, 3], [np.zeros(0, dtype=np.float32)] * 4, 3, ftar.PipelineConfig())
        rng = np.random.default_rng(3)
        cfg = ftar.PipelineConfig(chunk_bytes=64, max_in_flight=2)
        ring.reconfig(members=[0, 1, 2])
        run_case(ring, [0, 1, 2], [rng.standard_normal(37).astype(np.float32) for _ in range(3)], 4, cfg)
        ring.reconfig(members=[0, 2])
        run_case(ring, [0, 2], [rng.standard_normal(37).astype(np.float32) for _ in range(2)], 5, cfg)
        ring.reconfig(members=[0, 1, 2, 3])
        run_case(ring, [0, 1, 2, 3], [rng.standard_normal(37).astype(np.float32) for _ in range(4)], 6, cfg)
        assert all(ring.groups[r].generation == ring.gen for r in range(4))
    finally:
        ring.close()


def test_dropin_single_member_and_stale_reconfig(ftar):
    from paper_2602_00277_b200 import errors
    ring = Ring(ftar, 4)
    try:
        ring.reconfig()
        with pytest.raises(errors.Fatal):
            ring.groups[0].reconfig(ring.addrs, ring.gen, deadline_s=0.5)
        with pytest.raises(errors.Fatal):
            ring.groups[0].reconfig({1: ring.addrs[1], 2: ring.addrs[2]}, ring.gen + 5, deadline_s=0.5)
        g = ring.groups[0]
        g.reconfig({0: ring.addrs[0]}, ring.gen + 1)
        assert g.n == 1 and g.links_ready()
        buf = to_dev(np.arange(5, dtype=np.float32))
        out = ftar.ftar_all_reduce(g, buf, 1, ftar.PipelineConfig())
        assert out is buf
        np.testing.assert_array_equal(out.cpu().numpy(), np.arange(5, dtype=np.float32))
        bad = to_dev(np.array([1.0, np.nan], dtype=np.float32))
        with pytest.raises(errors.Fatal):
            ftar.ftar_all_reduce(g, bad, 2, ftar.PipelineConfig())
        with pytest.raises(errors.Fatal):
            ftar.ftar_all_reduce(g, torch.ones(4, dtype=torch.float64, device=DEV), 3)
    finally:
        ring.close()


def test_dropin_absent_peer_times_out_untouched(ftar):
    from paper_2602_00277_b200 import errors
    ring = Ring(ftar, 2)
    try:
        ring.reconfig()
        cfg = ftar.PipelineConfig(chunk_bytes=64, max_in_flight=1, per_chunk_timeout_s=0.4)
        original = np.arange(64, dtype=np.float32)
        buf = to_dev(original)
        res = ring.all_reduce({0: buf}, 1, cfg, [0])
        assert isinstance(res[0], errors.Recoverable)
        np.testing.assert_array_equal(buf.cpu().numpy(), original)
        assert not ring.groups[0].links_ready()
        with pytest.raises(errors.Recoverable):
            ftar.ftar_all_reduce(ring.groups[0], buf, 2, cfg)
    finally:
        ring.close()


def test_dropin_peer_death_and_retry(ftar):
    from paper_2602_00277_b200 import errors
    ring = Ring(ftar, 3)
    try:
        ring.reconfig()
        cfg = ftar.PipelineConfig(chunk_bytes=32, max_in_flight=2, per_chunk_timeout_s=2.0)
        rng = np.random.default_rng(11)
        arrays = [rng.standard_normal(50).astype(np.float32) for _ in range(3)]
        bufs = {r: to_dev(arrays[r]) for r in range(3)}

        def die_soon():
            time.sleep(0.05)
            ring.groups[2].close_links()

        killer = threading.Thread(target=die_soon)
        killer.start()
        t0 = time.monotonic()
        res = ring.all_reduce(bufs, 1, cfg, [0, 1])
        killer.join()
        assert time.monotonic() - t0 < 1.5  # released by the close, not the timeout
        for r in (0, 1):
            assert isinstance(res[r], errors.Recoverable)
            np.testing.assert_array_equal(bufs[r].cpu().numpy(), arrays[r])
        ring.reconfig()
        run_case(ring, [0, 1, 2], arrays, 1, ftar.PipelineConfig(chunk_bytes=32, max_in_flight=2))
    finally:
        ring.close()


def test_stale_generation_flags_do_not_satisfy_new_calls(ftar, rings):
    """Flags left in the arenas by generation g (including an aborted call)
    never complete a wait of generation g+1 (ftar.py:281-282, 390-393)."""
    ring = rings(3)
    ring.reconfig()
    cfg = ftar.PipelineConfig(per_chunk_timeout_s=0.3)
    arrays = member_inputs(3, 100_000, seed=9)
    bufs = [to_dev(a) for a in arrays]
    sts = ring.wait(ring.launch(bufs, cfg, fault=(2, 0)), cfg)  # aborted attempt
    assert sts[2] != 0 and all(s != 0 for s in sts)
    ring.reconfig()
    ring.all_reduce(bufs, cfg)
    want = orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight)
    for b in bufs:
        np.testing.assert_array_equal(b.cpu().numpy(), want)


def test_mismatched_call_is_protocol_violation(ftar):
    from paper_2602_00277_b200 import errors
    ring = Ring(ftar, 2)
    try:
        ring.reconfig()
        cfg = ftar.PipelineConfig(per_chunk_timeout_s=1.0)
        bufs = {0: to_dev(np.ones(8, dtype=np.float32)), 1: to_dev(np.ones(9, dtype=np.float32))}
        res = ring.all_reduce(bufs, 1, cfg, [0, 1])
        for r in (0, 1):
            assert isinstance(res[r], errors.Fatal) and res[r].reason == errors.PROTOCOL_VIOLATION
    finally:
        ring.close()


def test_registered_pool_zero_copy(ftar):
    """Buckets allocated in the group's pool are read in place by peers."""
    from paper_2602_00277_b200.fabric import LocalFabric
    fab = LocalFabric()
    gs = [ftar.RingGroup(r, 0, fab, device=DEV, max_bucket_bytes=1 << 20, pool_bytes=4 << 20) for r in range(2)]
    try:
        addrs = {r: ftar.PeerAddress(r) for r in range(2)}
        ts = [threading.Thread(target=g.reconfig, args=(addrs, 1)) for g in gs]
        [t.start() for t in ts]
        [t.join() for t in ts]
        arrays = member_inputs(2, 1000, seed=3)
        bufs = []
        for g, a in zip(gs, arrays):
            t = g.alloc_bucket(1000)
            t.copy_(to_dev(a))
            bufs.append(t)
        res = {}
        th = [threading.Thread(target=lambda i=i: res.__setitem__(i, ftar.ftar_all_reduce(gs[i], bufs[i], 1)))
              for i in range(2)]
        [t.start() for t in th]
        [t.join() for t in th]
        want = orc.oracle_reduce(arrays, 8 << 20, 4)
        for b in bufs:
            np.testing.assert_array_equal(b.cpu().numpy(), want)
    finally:
        for g in gs:
            g.close()


def test_inflight_bound_follows_the_path(ftar, monkeypatch):
    """InflightMeter (ftar.py:141-159): each call records the per-link bound of
    the path it takes -- small push one-shot (the whole input), register path
    (CTAs x 512 x U x 16 B), bulk-copy (CTAs x (stages-1) x tile)."""
    from paper_2602_00277_b200 import _lib
    from paper_2602_00277_b200.fabric import LocalFabric
    monkeypatch.delenv("FTAR_TMA", raising=False)
    fab = LocalFabric()
    gs = [ftar.RingGroup(r, 0, fab, device=DEV, max_bucket_bytes=1 << 20, pool_bytes=4 << 20) for r in range(2)]
    try:
        addrs = {r: ftar.PeerAddress(r) for r in range(2)}
        ts = [threading.Thread(target=g.reconfig, args=(addrs, 1)) for g in gs]
        [t.start() for t in ts]
        [t.join() for t in ts]
        cfg = ftar.PipelineConfig()
        paths = {}
        for elems in (256, 1 << 21, 1 << 24):
            b, g, path = _lib.C.c_uint64(), _lib.C.c_int(), _lib.C.c_int()
            _lib.check(_lib.lib.ftar_inflight_bound(2, elems, _lib.DT_F32, cfg.chunk_bytes,
                                                    cfg.max_in_flight, 1, _lib.C.byref(b), _lib.C.byref(g),
                                                    _lib.C.byref(path)), "bound")
            paths[elems] = path.value
            assert (b.value, g.value) == gs[0].inflight_bound(elems, _lib.DT_F32, cfg, True)
            assert g.value >= 1
            if path.value == 1:
                assert b.value == elems * 4
            elif path.value == 3:  # n=2 f32: U = 8 vectors of 4 fp32 per thread
                assert b.value == g.value * 512 * 8 * 16
            else:
                assert path.value == 2 and b.value % g.value == 0 and b.value < elems * 4
        assert paths == {256: 1, 1 << 21: 3, 1 << 24: 2}
        # a call records its bound in the meter
        buf = gs[0].alloc_bucket(256)
        buf2 = gs[1].alloc_bucket(256)
        th = [threading.Thread(target=ftar.ftar_all_reduce, args=(g, t, 1)) for g, t in zip(gs, (buf, buf2))]
        [t.start() for t in th]
        [t.join() for t in th]
        assert gs[0].meter.max_unacked_bytes == 1024 and gs[0].meter.unacked_bytes == 0
    finally:
        for g in gs:
            g.close()


# ---------------------------------------------------------------------------
# Host buffers (the reference's numpy call shape) and range launches.


@pytest.mark.parametrize("mode", ["protocol", "oneshot"])
def test_host_pipeline_chunks_fold_with_whole_bucket_geometry(ftar, rings, mode):
    """Chunked H2D/reduce/D2H: chunk boundaries cut partitions and segments,
    yet every element folds as in one whole-bucket call."""
    n, e = 3, 1_000_003
    arrays = member_inputs(n, e, seed=21)
    ring = rings(n, protocol=(mode == "protocol"))
    ring.reconfig()
    cfg = ftar.PipelineConfig(chunk_bytes=40_000, max_in_flight=3)  # 90k-element partitions
    want = orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight)
    hosts = [torch.from_numpy(a.copy()).pin_memory() for a in arrays]
    outs = [torch.empty(e).pin_memory() for _ in range(n)]
    ring.all_reduce_host(hosts, cfg, outs=outs, chunk_elems=77_777)
    for o in outs:
        np.testing.assert_array_equal(o.numpy(), want)
    # in place, numpy arrays, fused scale
    bufs = [a.copy() for a in arrays]
    ring.all_reduce_host(bufs, cfg, scale=1.0 / n, chunk_elems=300_000)
    for b in bufs:
        np.testing.assert_array_equal(b, orc.normalize(want, n))


def test_host_pipeline_bf16_to_f32(ftar, rings):
    n, e = 4, 2_000_001
    arrays = member_inputs(n, e, seed=22, dtype="bf16")
    ring = rings(n, protocol=False)
    ring.reconfig()
    hosts = [torch.from_numpy(a).to(torch.bfloat16).pin_memory() for a in arrays]
    outs = [torch.empty(e).pin_memory() for _ in range(n)]
    ring.all_reduce_host(hosts, outs=outs, chunk_elems=1 << 19)
    want = orc.oracle_reduce(arrays, 8 << 20, 4)
    for o in outs:
        np.testing.assert_array_equal(o.numpy(), want)


def test_dropin_numpy_buffers_threaded(ftar):
    """ftar_all_reduce on numpy arrays, members on threads: the reference's
    tests/test_ftar.py run_case shape, unchanged."""
    ring = Ring(ftar, 3)
    try:
        ring.reconfig()
        cfg = ftar.PipelineConfig(chunk_bytes=28, max_in_flight=2)
        rng = np.random.default_rng(42)
        arrays = [rng.standard_normal(2049).astype(np.float32) for _ in range(3)]
        bufs = {r: arrays[r].copy() for r in range(3)}
        res = ring.all_reduce(bufs, 1, cfg, [0, 1, 2])
        want = orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight)
        for r in range(3):
            assert res[r] is bufs[r]
            np.testing.assert_array_equal(bufs[r], want)
    finally:
        ring.close()


# ---------------------------------------------------------------------------
# §8f rank 1: normalisation + SGD-momentum fused into the collective.


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_fused_sgd_momentum_bit_exact(ftar, rings, dtype):
    """model.optimizer_step(grad * f32(1/(h*R))) (model.py:146-155,
    replica.py:622-633) on every member, bit for bit, out of place."""
    n, e = 4, 1_000_003
    arrays = member_inputs(n, e, seed=41, dtype=dtype)
    ring = rings(n, protocol=True)
    ring.reconfig()
    rng = np.random.default_rng(42)
    p0 = rng.standard_normal(e).astype(np.float32)
    m0 = (rng.standard_normal(e) * 0.1).astype(np.float32)
    lr, beta, denom = 0.05, 0.9, n * 2
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    bufs = [to_dev(a, tdt) for a in arrays]
    params = [to_dev(p0) for _ in range(n)]
    moms = [to_dev(m0) for _ in range(n)]
    gouts = [torch.empty(e, device=DEV) for _ in range(n)]
    pout, mout = ring.all_reduce_sgd(bufs, params=params, momenta=moms, lr=lr, beta=beta, scale=1.0 / denom,
                                     grad_outs=gouts)
    g = orc.normalize(orc.oracle_reduce(arrays, 8 << 20, 4), denom)
    pw, mw = orc.sgd_momentum(p0.copy(), m0.copy(), g, beta, lr)
    for i in range(n):
        np.testing.assert_array_equal(gouts[i].cpu().numpy(), g)
        np.testing.assert_array_equal(pout[i].cpu().numpy(), pw)
        np.testing.assert_array_equal(mout[i].cpu().numpy(), mw)
        np.testing.assert_array_equal(params[i].cpu().numpy(), p0)  # inputs untouched (commit is the caller's)
        np.testing.assert_array_equal(moms[i].cpu().numpy(), m0)


def test_local_ring_queued_launches(ftar):
    """In-process rings queue like the multi-GPU path: three buckets in
    flight on one stream, collected oldest first, each bit-exact."""
    ring = ftar.LocalRing(4, device=DEV, max_bucket_bytes=8 << 20)
    try:
        cfg = ftar.PipelineConfig()
        jobs = []
        for b in range(3):
            arrays = member_inputs(4, 1_000_003 + b, seed=600 + b)
            bufs = [to_dev(a) for a in arrays]
            outs = [torch.empty_like(x) for x in bufs]
            jobs.append((arrays, outs, ring.launch(bufs, cfg, outs=outs, scale=0.25)))
        for arrays, outs, tok in jobs:
            assert ring.wait(tok, cfg) == [0] * 4
            want = orc.normalize(orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight), 4)
            for o in outs:
                np.testing.assert_array_equal(o.cpu().numpy(), want)
    finally:
        for g in ring.groups:
            g.close()


@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("elems", [1, 257, 4099, 65_537, 262_143])
def test_small_one_shot_unaligned_and_behind(ftar, n, elems):
    """The small one-shot's fold (fold_small) on buffers that are NOT 16-byte
    aligned (the per-element path with its cached owner run), with a behind
    member whose buffer is garbage, every bucket at most 1 MiB: bit-exact."""
    ring = ftar.LocalRing(n, device=DEV, max_bucket_bytes=4 << 20, protocol=True)
    try:
        arrays = member_inputs(n, elems, seed=900 + n + elems)
        contrib = [m != n - 1 for m in range(n)]
        ring.reconfig(contributors=[m for m in range(n) if contrib[m]])
        cfg = ftar.PipelineConfig(chunk_bytes=4096, max_in_flight=2)
        base = [torch.full((elems + 1,), float("nan"), device=DEV) for _ in range(n)]
        bufs = []
        for m, (b, a) in enumerate(zip(base, arrays)):
            if contrib[m]:
                b[1:].copy_(to_dev(a))
            bufs.append(b[1:])  # 4 bytes past an aligned allocation
        outs = [torch.full((elems + 1,), float("nan"), device=DEV)[1:] for _ in range(n)]
        ring.all_reduce(bufs, cfg, outs=outs, scale=1.0 / n)
        want = orc.normalize(orc.oracle_reduce(arrays, cfg.chunk_bytes, cfg.max_in_flight, contrib=contrib), n)
        for o in outs:
            np.testing.assert_array_equal(o.cpu().numpy(), want)
    finally:
        ring.close()
