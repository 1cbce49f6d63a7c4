"""Host-side API without a GPU: the C-ABI library loads and exports every
symbol the header declares; the geometry helpers match the reference's
(tests/test_ftar.py:48-107); error mapping follows errors.py."""

import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_2602_00277_b200 import _build, _lib, errors, ftar
from oracle import ftar_oracle as orc

MIB = 1024 * 1024


def test_library_exports_every_header_symbol():
    syms = _lib.header_symbols()
    assert len(syms) >= 25
    lib = C.CDLL(_build.LIB)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_library_is_sm100a():
    assert "sm_100a" in _lib.version()
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_geometry_abi_without_gpu():
    slice_e, ctas, threads = C.c_uint64(), C.c_int(), C.c_int()
    assert _lib.lib.ftar_geometry(1000, 4, C.byref(slice_e), C.byref(ctas), C.byref(threads)) == 0
    assert slice_e.value == 256 and threads.value == 512 and ctas.value >= 1
    assert _lib.lib.ftar_geometry(1000, 9, None, None, None) == errors.ST_INVARIANT


def test_status_mapping():
    assert errors.from_status(0) is None
    for code, cls, reason in [(1, errors.Recoverable, errors.TIMEOUT), (7, errors.Recoverable, errors.TIMEOUT),
                              (2, errors.Recoverable, errors.PEER_RESET), (3, errors.Recoverable, errors.PEER_DOWN),
                              (4, errors.Fatal, errors.PROTOCOL_VIOLATION), (5, errors.Fatal, errors.NUMERICAL),
                              (6, errors.Fatal, errors.INTERNAL_INVARIANT)]:
        e = errors.from_status(code)
        assert isinstance(e, cls) and e.reason == reason


def test_partition_plan_large_message_splits_at_cap():
    cfg = ftar.PipelineConfig(chunk_bytes=8 * MIB, max_in_flight=4)
    plan = ftar.build_partition_plan(256 * MIB, cfg, 4)
    assert plan.partition_bytes() == [(0, 128 * MIB), (128 * MIB, 128 * MIB)]
    assert ftar.build_partition_plan(100, ftar.PipelineConfig(), 4).partitions == [(0, 25)]


def test_partition_plan_properties_match_oracle():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(1, 9))
        chunk = int(rng.integers(1, 65)) * 4
        c = int(rng.integers(1, 6))
        total = int(rng.integers(0, 5000))
        plan = ftar.build_partition_plan(total * 4, ftar.PipelineConfig(chunk_bytes=chunk, max_in_flight=c), n)
        assert plan.partitions == orc.partition_plan(total, chunk, c, n)
        lengths = [ln for _, ln in plan.partitions]
        assert max(lengths) - min(lengths) <= 1
        assert all(ln * 4 <= max(chunk * c * n, 4) for ln in lengths)


def test_geometry_errors_and_helpers():
    with pytest.raises(errors.Fatal):
        ftar.build_partition_plan(102, ftar.PipelineConfig(), 2)
    for part, n in [(10, 4), (3, 5), (0, 3), (7, 1), (8, 8)]:
        segs = ftar.segment_bounds(part, n)
        assert len(segs) == n and sum(s for _, s in segs) == part
    assert ftar.iter_chunks(10, 4) == [(0, 0, 4), (1, 4, 4), (2, 8, 2)]
    assert ftar.iter_chunks(0, 4) == [] and ftar.iter_chunks(3, 8) == [(0, 0, 3)]
    for bad in (dict(chunk_bytes=2), dict(max_in_flight=0), dict(per_chunk_timeout_s=0)):
        with pytest.raises(errors.Fatal):
            ftar.PipelineConfig(**bad)


def test_classify_error():
    assert ftar.classify_error(errors.Recoverable(errors.TIMEOUT)) == "recoverable"
    assert ftar.classify_error(errors.Fatal(errors.NUMERICAL)) == "fatal"
    assert ftar.classify_error(TimeoutError()) == "recoverable"
    assert ftar.classify_error(ConnectionResetError()) == "recoverable"
    assert ftar.classify_error(ValueError("x")) == "fatal"


def _bound(n, elems, dt=_lib.DT_F32, push=1, env=None):
    b, g, path = C.c_uint64(), C.c_int(), C.c_int()
    cfg = ftar.PipelineConfig()
    rc = _lib.lib.ftar_inflight_bound(n, elems, dt, cfg.chunk_bytes, cfg.max_in_flight, push,
                                      C.byref(b), C.byref(g), C.byref(path))
    assert rc == 0
    return b.value, g.value, path.value


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_inflight_bound_per_path(n, monkeypatch):
    """The per-link in-flight bound follows the data path each bucket size takes
    (host policy only: no device work)."""
    for k in ("FTAR_TMA", "FTAR_SMALL_BYTES", "FTAR_TMA_MIN_SLICE_MIB", "FTAR_CTAS_TMA", "FTAR_CTAS_PUSH"):
        monkeypatch.delenv(k, raising=False)
    assert _bound(n, 0) == (0, 0, 0)
    b, g, path = _bound(n, 256)  # 1 KB: the push one-shot posts the whole input
    assert (b, path) == (1024, 1) and g >= 1
    b, g, path = _bound(n, (2 << 20) // 4 * n)  # 2 MiB slices: register path
    assert path == 3 and 1 <= g <= 128 and b % (g * 512 * 16) == 0
    b, g, path = _bound(n, (64 << 20) // 4 * n)  # 64 MiB slices: bulk-copy reduce-scatter
    assert path == 2 and 1 <= g <= (96 if n == 2 else 48) and b < 227 * 1024 * g
    monkeypatch.setenv("FTAR_TMA", "0")
    assert _bound(n, (64 << 20) // 4 * n)[2] == 3
    monkeypatch.setenv("FTAR_CTAS_PUSH", "7")
    assert _bound(n, (64 << 20) // 4 * n)[1] == 7
    assert _lib.lib.ftar_inflight_bound(9, 1, 0, 8 << 20, 4, 0, None, None, None) == errors.ST_INVARIANT


def test_inflight_meter():
    m = ftar.InflightMeter()
    m.sent(100, 2)
    m.sent(50)
    m.acked(150, 3)
    assert (m.unacked_bytes, m.max_unacked_bytes, m.max_unacked_chunks) == (0, 150, 3)


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    """The product path must fail loudly when the CUDA library is missing."""
    import importlib
    monkeypatch.setattr(_build, "LIB", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        importlib.reload(_lib)
    monkeypatch.undo()
    importlib.reload(_lib)


# --- persistent checkpoint format (§8f rank 4), pinned to the reference -------


def _ckpt_cases():
    with open(os.path.join(os.path.dirname(__file__), "golden", "ckpt_cases.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _ckpt_cases(), ids=lambda c: f"step{c['step']}-rank{c['rank']}")
def test_checkpoint_files_match_reference_bytes(tmp_path, case):
    import hashlib

    import numpy as np
    from paper_2602_00277_b200 import checkpoint as ck
    rng = np.random.default_rng(case["seed"])
    p = rng.standard_normal(case["n_params"]).astype(np.float32)
    m = rng.standard_normal(case["n_momentum"]).astype(np.float32)
    path = ck.write_shard(str(tmp_path), case["step"], case["rank"], p.tobytes(), m.tobytes())
    assert os.path.basename(path) == case["file_name"]
    assert hashlib.sha256(open(path, "rb").read()).hexdigest() == case["file_sha256"]
    rp, rm = ck.read_shard(str(tmp_path), case["step"], case["rank"])
    assert rp == p.tobytes() and rm == m.tobytes()
    mpath = ck.write_manifest(str(tmp_path), case["step"], case["rank"] + 1, (4, 8), {0: 5, 2: 9})
    assert open(mpath, "rb").read().decode() == case["manifest"]


def test_checkpoint_find_latest_and_validation(tmp_path):
    from paper_2602_00277_b200 import checkpoint as ck
    from paper_2602_00277_b200.errors import Fatal
    d = str(tmp_path)
    assert ck.find_latest(d) is None
    for step in (3, 5):
        for r in range(2):
            ck.write_shard(d, step, r, b"\x01" * 8, b"\x02" * 4)
        ck.write_manifest(d, step, 2, (1,), {0: step})
    ck.write_manifest(d, 9, 2, (1,), {})  # a manifest without its shards is skipped
    step, doc = ck.find_latest(d)
    assert step == 5 and doc["n_ranks"] == 2
    os.rename(ck.shard_path(d, 3, 0), ck.shard_path(d, 7, 0))  # header says (3, 0)
    with pytest.raises(Fatal):
        ck.read_shard(d, 7, 0)
    with open(ck.shard_path(d, 5, 1), "r+b") as fh:  # truncated
        fh.truncate(20)
    with pytest.raises(Fatal):
        ck.read_shard(d, 5, 1)
