"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden digests in tests/golden/ were produced by running the reference
(its socket ring, bench._LoopbackRing, and its replica engine) with
tests/golden/make_golden.py; inputs are regenerated here from their seeds.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from gen import behind_set, case_inputs, criterion_cases, member_inputs
from oracle import cref
from oracle import ftar_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def load_cases():
    with open(os.path.join(GOLD, "ftar_cases.json")) as f:
        return json.load(f)


def test_case_specs_are_reproducible():
    # the committed specs must be exactly what gen.py regenerates
    got = [{k: v for k, v in c.items() if k != "sha256"} for c in load_cases()]
    assert got == criterion_cases()


@pytest.mark.parametrize("case", load_cases(), ids=lambda c: f"{c['idx']}-{c['kind']}-n{c['n']}-e{c['elems']}")
def test_numpy_oracle_matches_reference_ring(case):
    arrays = case_inputs(case)
    out = orc.oracle_reduce(arrays, case["chunk_bytes"], case["max_in_flight"])
    assert sha(out) == case["sha256"]


@pytest.mark.parametrize("case", [c for c in load_cases() if c["kind"] == "behind"],
                         ids=lambda c: f"{c['idx']}")
def test_contributor_mask_equals_zero_buffers(case):
    """Behind replicas with garbage buffers + contrib mask == the reference's zeros."""
    arrays = case_inputs(case, garbage_behind=True)
    contrib = [i not in behind_set(case) for i in range(case["n"])]
    out = orc.oracle_reduce(arrays, case["chunk_bytes"], case["max_in_flight"], contrib=contrib)
    assert sha(out) == case["sha256"]


def test_c_port_matches_reference_ring():
    cref.build()
    for case in load_cases()[::3]:
        arrays = case_inputs(case)
        closed = cref.reduce_f32(arrays, case["chunk_bytes"], case["max_in_flight"])
        assert sha(closed) == case["sha256"], case["idx"]
        bufs = [a.copy() for a in arrays]
        st = cref.ring_allreduce(bufs, case["chunk_bytes"], case["max_in_flight"], threads_per_member=2)
        assert st == 0
        for b in bufs:
            assert sha(b) == case["sha256"], case["idx"]


def test_hand_cases_full_vectors():
    z = np.load(os.path.join(GOLD, "ftar_small.npz"))
    for name in ("four_members", "multi_partition"):
        chunk, C = (int(x) for x in z[f"{name}_cfg"])
        out = orc.oracle_reduce(list(z[f"{name}_in"]), chunk, C)
        np.testing.assert_array_equal(out, z[f"{name}_out"])
    np.testing.assert_array_equal(z["four_members_out"], np.full(8, 6.0, dtype=np.float32))


def test_config1_digest():
    with open(os.path.join(GOLD, "config1.json")) as f:
        g = json.load(f)
    arrays = member_inputs(g["n"], g["elems"], seed=g["seed"])
    out = orc.oracle_reduce(arrays, g["chunk_bytes"], g["max_in_flight"])
    assert sha(out) == g["sha256"]
    np.testing.assert_array_equal(orc.member_inputs(4, 1000)[3], member_inputs(4, 1000)[3])


def test_nonfinite_port_reports_numerical():
    arrays = [np.ones(12, dtype=np.float32) for _ in range(2)]
    arrays[1][3] = np.nan
    bufs = [a.copy() for a in arrays]
    assert cref.ring_allreduce(bufs, 16, 2) == 5
    for b, a in zip(bufs, arrays):  # single partition: nothing committed
        np.testing.assert_array_equal(b, a)


def test_normalize_vectors():
    z = np.load(os.path.join(GOLD, "normalize.npz"))
    for h in range(1, 9):
        for R in (1, 2):
            np.testing.assert_array_equal(orc.normalize(z["x"], h * R), z[f"h{h}_R{R}"])


def test_normalize_is_a_multiply_not_a_divide():
    # replica.py:626 multiplies by f32(1/denom); a true divide differs
    z = np.load(os.path.join(GOLD, "normalize.npz"))
    x = z["x"]
    assert not np.array_equal(x / np.float32(7.0), z["h7_R1"])


def test_owner_map_matches_segments():
    own = orc.owners(23, 8, 1, 3)  # cap = 6 elems -> 4 partitions of 6,6,6,5
    assert own.tolist() == [0, 0, 1, 1, 2, 2] * 3 + [0, 0, 1, 1, 2]


def test_reference_compiled_kernel_matches_port():
    """oracle/_ref holds the reference's own _ckernels (cythonized from the
    reference tree); its accumulate must equal a plain fp32 add."""
    ref_dir = cref.build_ref()
    if ref_dir is None:
        pytest.skip("reference tree not present (GPU box)")
    import importlib.util
    import glob
    so = glob.glob(os.path.join(ref_dir, "_ckernels*.so"))[0]
    spec = importlib.util.spec_from_file_location("_ckernels", so)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    rng = np.random.default_rng(1)
    dst = rng.standard_normal(1000).astype(np.float32)
    src = rng.standard_normal(1000).astype(np.float32)
    want = dst + src
    mod.accumulate(dst, memoryview(src.tobytes()).cast("B"))
    np.testing.assert_array_equal(dst, want)


# --- intra-replica collectives (replica.py:241-262), pinned to the reference ----


def _intra_cases():
    with open(os.path.join(GOLD, "intra_cases.json")) as f:
        return json.load(f)


def test_intra_oracle_matches_reference_goldens():
    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()

    cases = _intra_cases()
    assert len(cases) >= 40
    for c in cases:
        vecs = member_inputs(c["n"], c["total"], c["seed"], c["kind"])
        bounds = [tuple(b) for b in c["bounds"]]
        shards = orc.intra_reduce_scatter(vecs, bounds)
        assert [sha(s) for s in shards] == c["rs_sha"], c
        assert sha(orc.intra_all_gather(shards, bounds, c["total"])) == c["ag_sha"], c


def test_intra_oracle_hand_values():
    """tests/test_replica.py:61-68 and :89-97."""
    vecs = [np.array([1, 2, 3, 4], dtype=np.float32), np.array([10, 20, 30, 40], dtype=np.float32)]
    s = orc.intra_reduce_scatter(vecs, [(0, 2), (2, 2)])
    assert s[0].tolist() == [11.0, 22.0] and s[1].tolist() == [33.0, 44.0]
    full = np.arange(10, dtype=np.float32)
    b = [(0, 4), (4, 3), (7, 3)]
    assert np.array_equal(orc.intra_all_gather([full[o:o + n] for o, n in b], b, 10), full)
