"""Catch-up snapshot/pull and the operator plugin on the GPU."""

import numpy as np
import pytest
import torch

from paper_2602_00277_b200 import checkpoint as ck

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def test_accumulate_and_copy_into_vs_torch_fp32():
    from paper_2602_00277_b200 import kernels
    assert kernels.BACKEND == "sm_100a" and set(kernels.backends()) == {"sm_100a"}
    g = torch.Generator(device=DEV).manual_seed(0)
    for n in (0, 1, 7, 4096, 1_000_003):
        dst = torch.randn(n, device=DEV, generator=g)
        src = torch.randn(n, device=DEV, generator=g)
        want = dst + src
        kernels.accumulate(dst, src)
        assert torch.equal(dst, want)
        srcb = src.to(torch.bfloat16)
        want = dst + srcb.float()
        kernels.accumulate(dst, srcb)
        assert torch.equal(dst, want)
        kernels.copy_into(dst, srcb)
        assert torch.equal(dst, srcb.float())
    with pytest.raises(ValueError):
        kernels.accumulate(torch.zeros(4, device=DEV), torch.zeros(5, device=DEV))


def test_snapshot_retention_and_pull_bit_exact():
    from paper_2602_00277_b200 import checkpoint as ck
    donor = ck.SnapshotStore(device=DEV)
    rec = ck.SnapshotStore(device=DEV)
    g = torch.Generator(device=DEV).manual_seed(1)
    p = torch.randn(3_000_001, device=DEV, generator=g)
    m = torch.randn(1_234_567, device=DEV, generator=g)
    assert donor.step is None
    donor.capture(7, p, m)
    assert donor.step == 7 and donor.device_step() == 7
    p_out = torch.empty_like(p)
    m_out = torch.empty_like(m)
    ck.fetch_shard(donor, 7, rank=0, local=rec, out=(p_out, m_out), ctas=8)
    torch.cuda.synchronize()
    assert torch.equal(p_out, p) and torch.equal(m_out, m)
    # later writes to the live tensors do not leak into the snapshot
    p.add_(1.0)
    p2 = torch.empty_like(p)
    ck.fetch_shard(donor, 7, rank=0, local=rec, out=(p2, torch.empty_like(m)))
    assert torch.equal(p2, p_out)
    # retention is one: a new capture replaces the old step
    donor.capture(8, p, m)
    with pytest.raises(ck.SnapshotUnavailable) as ei:
        ck.fetch_shard(donor, 7, rank=0, local=rec, out=(p2, torch.empty_like(m)))
    assert ei.value.available == 8
    with pytest.raises(ck.SnapshotUnavailable):
        donor.get(7)
    assert donor.lengths == (p.numel() * 4, m.numel() * 4)
    gp, gm = donor.get(8)  # payload views of the device snapshot (checkpoint.py:76-80)
    assert torch.equal(gp.view(torch.float32), p) and torch.equal(gm.view(torch.float32), m)


def test_pull_on_side_stream_overlaps_ftar():
    """The pull runs on a low-priority side stream while an FTAR runs on the
    default stream; both finish and both are correct."""
    from paper_2602_00277_b200 import checkpoint as ck
    from paper_2602_00277_b200 import ftar
    from oracle import ftar_oracle as orc
    from gen import member_inputs
    donor = ck.SnapshotStore(device=DEV)
    rec = ck.SnapshotStore(device=DEV)
    p = torch.randn(64 << 20 >> 2, device=DEV)
    m = torch.randn(64 << 20 >> 2, device=DEV)
    donor.capture(3, p, m)
    torch.cuda.synchronize()
    ring = ftar.LocalRing(4, device=DEV, max_bucket_bytes=16 << 20)
    try:
        arrays = member_inputs(4, 1 << 20, seed=2)
        bufs = [torch.from_numpy(a).to(DEV) for a in arrays]
        po, mo = torch.empty_like(p), torch.empty_like(m)
        pull = ck.start_fetch(rec, donor, 3, 0, po, mo, ctas=8)
        ring.all_reduce(bufs)
        pull.wait()
        torch.cuda.synchronize()
        assert torch.equal(po, p) and torch.equal(mo, m)
        want = orc.oracle_reduce(arrays, 8 << 20, 4)
        for b in bufs:
            np.testing.assert_array_equal(b.cpu().numpy(), want)
    finally:
        ring.close()


def test_pick_donor():
    from paper_2602_00277_b200 import checkpoint as ck
    from paper_2602_00277_b200 import errors
    assert [ck.pick_donor([0, 1, 2], 3, r) for r in range(4)] == [0, 1, 2, 0]
    assert ck.pick_donor([0, 1, 2], 3, rank=0, attempt=1) == 1
    assert ck.pick_donor([0, 3], 3, rank=1) == 0
    with pytest.raises(errors.Recoverable):
        ck.pick_donor([3], 3, rank=0)


def test_persist_snapshot_to_reference_format(tmp_path):
    """§8f rank 4: the device snapshot streamed to the reference's shard file
    (checkpoint.py:174-198) in the background; read back bit-exact through
    both the bytes reader and the device restore."""
    from paper_2602_00277_b200 import checkpoint as ck
    store = ck.SnapshotStore(device=DEV, rank=2)
    g = torch.Generator(device=DEV).manual_seed(5)
    p = torch.randn(20_000_003, device=DEV, generator=g)  # > one 64 MiB staging chunk
    m = torch.randn(3_000_001, device=DEV, generator=g)
    store.capture(11, p, m)
    job = store.persist(str(tmp_path))
    path = job.wait()
    assert path == ck.shard_path(str(tmp_path), 11, 2) and job.done()
    rp, rm = ck.read_shard(str(tmp_path), 11, 2)
    assert rp == p.cpu().numpy().tobytes() and rm == m.cpu().numpy().tobytes()
    p2, m2 = torch.empty_like(p), torch.empty_like(m)
    ck.read_shard_into(str(tmp_path), 11, 2, p2, m2)
    assert torch.equal(p2, p) and torch.equal(m2, m)
    ck.write_manifest(str(tmp_path), 11, 3, (1,), {})
    for r in (0, 1):
        ck.write_shard(str(tmp_path), 11, r, b"", b"")
    assert ck.find_latest(str(tmp_path))[0] == 11
    store.close()


def test_persist_detects_a_capture_during_the_write(tmp_path):
    """A capture of the next step while the snapshot is being streamed out
    must not leave a torn file: SnapshotUnavailable, nothing on disk."""
    import os

    from paper_2602_00277_b200 import checkpoint as ck
    store = ck.SnapshotStore(device=DEV)
    p = torch.ones(40_000_000, device=DEV)
    m = torch.zeros(10, device=DEV)
    store.capture(3, p, m)

    def recapture(i):
        if i == 0:
            store.capture(4, p * 2, m)
            torch.cuda.synchronize()

    job = store.persist(str(tmp_path), rank=0, background=False, _hook=recapture)
    with pytest.raises(ck.SnapshotUnavailable):
        job.wait()
    assert not os.listdir(str(tmp_path))
    # the new step persists cleanly afterwards
    assert store.persist(str(tmp_path), rank=0).wait() == ck.shard_path(str(tmp_path), 4, 0)
    store.close()


# --- the reference's tests/test_checkpoint.py snapshot / fetch cases, with
# tensor buffers and the reference's fetch_shard signature (in-process donors)


def test_reference_snapshot_retention_is_one():
    """tests/test_checkpoint.py:29-39."""
    st = ck.SnapshotStore(device=DEV, replica_id=40)
    assert st.step is None
    st.capture(3, b"ppp", b"mmm")
    gp, gm = st.get(3)
    assert bytes(gp.cpu().numpy()) == b"ppp" and bytes(gm.cpu().numpy()) == b"mmm"
    st.capture(4, b"qqqq", b"nn")
    assert st.step == 4
    with pytest.raises(ck.SnapshotUnavailable) as ei:
        st.get(3)
    assert ei.value.available == 4
    st.close()


def test_reference_fetch_roundtrip():
    """tests/test_checkpoint.py:42-64: fetch_shard(addr, step, rank,
    replica_id, incarnation) -> (params, momentum); a step the donor no
    longer holds -> SnapshotUnavailable(available)."""
    from paper_2602_00277_b200.ftar import PeerAddress
    donor = ck.SnapshotStore(device=DEV, replica_id=0, rank=0)
    params = torch.arange(10, dtype=torch.float32, device=DEV)
    momentum = torch.ones(5, dtype=torch.float32, device=DEV)
    donor.capture(7, params, momentum)
    gp, gm = ck.fetch_shard(PeerAddress(0, 0, "127.0.0.1", 0), 7, rank=0, replica_id=3, incarnation=1)
    assert torch.equal(gp.view(torch.float32), params) and torch.equal(gm.view(torch.float32), momentum)
    with pytest.raises(ck.SnapshotUnavailable) as ei:
        ck.fetch_shard(PeerAddress(0), 6, rank=0, replica_id=3, incarnation=1)
    assert ei.value.available == 7  # donor moved on; catch up next step
    donor.close()


def test_reference_fetch_from_empty_store():
    """tests/test_checkpoint.py:67-80."""
    from paper_2602_00277_b200.ftar import PeerAddress
    donor = ck.SnapshotStore(device=DEV, replica_id=11, rank=2)
    with pytest.raises(ck.SnapshotUnavailable) as ei:
        ck.fetch_shard(PeerAddress(11), 1, rank=2, replica_id=1, incarnation=1)
    assert ei.value.available is None
    donor.close()


def test_reference_fetch_from_dead_donor_is_recoverable():
    """tests/test_checkpoint.py:83-89: a donor that is not there (never
    published, or its process is gone) -> Recoverable."""
    from datetime import timedelta

    import torch.distributed as dist

    from paper_2602_00277_b200 import errors
    from paper_2602_00277_b200.fabric import StoreFabric
    from paper_2602_00277_b200.ftar import PeerAddress
    store = dist.HashStore()
    store.set_timeout(timedelta(seconds=1))
    rec = ck.SnapshotStore(device=DEV, replica_id=21, rank=0, fabric=StoreFabric(store))
    with pytest.raises(errors.Recoverable):
        ck.fetch_shard(PeerAddress(99), 1, rank=0, replica_id=21, incarnation=1, timeout_s=0.4)
    rec.close()


def test_serve_fetches_is_a_thread_target():
    import threading
    stop = threading.Event()
    t = threading.Thread(target=ck.serve_fetches, args=(None, None, stop), daemon=True)
    t.start()
    stop.set()
    t.join(timeout=2.0)
    assert not t.is_alive()


def test_pull_boost_bit_exact():
    """A pull started narrow and widened by a second grid (chunks claimed from
    one counter) lands every byte exactly once; a boost after the pull ended
    is a no-op; the next pull after a boosted one is exact too."""
    donor = ck.SnapshotStore(device=DEV, replica_id=50)
    rec = ck.SnapshotStore(device=DEV, replica_id=51)
    g = torch.Generator(device=DEV).manual_seed(3)
    p = torch.randn(40 << 20, device=DEV, generator=g)   # 160 MiB
    m = torch.randn(24 << 20, device=DEV, generator=g)
    donor.capture(9, p, m)
    for boost in (True, False, True):
        po, mo = torch.full_like(p, float("nan")), torch.full_like(m, float("nan"))
        h = ck.start_fetch(rec, donor, 9, 0, po, mo, ctas=1)
        if boost:
            h.boost(16)
        h.wait()
        h.boost(8)  # finished: no-op
        torch.cuda.synchronize()
        assert torch.equal(po, p) and torch.equal(mo, m)
    donor.close()
    rec.close()
