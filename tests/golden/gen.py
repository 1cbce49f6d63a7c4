"""Deterministic inputs for the golden cases (shared by make_golden.py, which
feeds them to the reference, and by the tests, which feed them to the oracle
and the CUDA path).  numpy's default_rng (PCG64) streams are stable across
numpy versions, so only seeds and digests need to be committed."""

from __future__ import annotations

import numpy as np


def bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def member_inputs(n: int, elems: int, seed: int = 0, dtype: str = "f32") -> list[np.ndarray]:
    out = []
    for r in range(n):
        x = np.random.default_rng((seed, r)).standard_normal(elems).astype(np.float32)
        out.append(bf16_round(x) if dtype == "bf16" else x)
    return out


def criterion_cases() -> list[dict]:
    """~160 randomized (n, length, chunk_bytes, max_in_flight) cases in the
    style of criterion 02 (tests/test_acceptance.py:86-137), lengths up to
    ~5e4 so the reference's socket ring generates them in seconds."""
    rng = np.random.default_rng(0x6A11)
    cases = [dict(n=2, elems=1), dict(n=8, elems=1), dict(n=8, elems=9), dict(n=4, elems=0),
             dict(n=3, elems=50_000), dict(n=8, elems=65_537)]
    while len(cases) < 120:
        cases.append(dict(n=2 + len(cases) % 7, elems=int(10 ** rng.uniform(0, 4.7))))
    out = []
    for i, c in enumerate(cases):
        nbytes = c["elems"] * 4
        if nbytes <= 4096:
            chunk = int(rng.integers(1, 65)) * 4
        else:
            chunk = max(4, (nbytes >> int(rng.integers(0, 9))) & ~3)
        kind = ["f32", "f32", "bf16", "special", "behind"][i % 5]
        out.append(dict(idx=i, kind=kind, n=c["n"], elems=c["elems"], chunk_bytes=chunk,
                        max_in_flight=int(rng.integers(1, 6)), seed=int(rng.integers(0, 2**31)),
                        scale_exp=int(rng.integers(-3, 4))))
    # default-geometry cases (one partition per small bucket, segment owners = slices)
    for j, (n, e) in enumerate([(2, 100_003), (4, 131_072), (8, 99_999), (5, 77_777)]):
        out.append(dict(idx=len(out), kind="f32", n=n, elems=e, chunk_bytes=8 * 1024 * 1024,
                        max_in_flight=4, seed=1000 + j, scale_exp=0))
    return out


def behind_set(spec: dict) -> list[int]:
    """Ring indices that are 'behind' (contribute zeros) in a 'behind' case."""
    if spec["kind"] != "behind" or spec["n"] < 2:
        return []
    rng = np.random.default_rng(spec["seed"] + 7)
    k = 1 + int(rng.integers(0, max(1, spec["n"] // 2)))
    return sorted(int(x) for x in rng.choice(spec["n"], size=min(k, spec["n"] - 1), replace=False))


def case_inputs(spec: dict, garbage_behind: bool = False) -> list[np.ndarray]:
    """Member buffers (fp32; bf16 cases as exact fp32 upcasts).  For 'behind'
    cases the behind members hold zeros (what the reference engine passes,
    replica.py:576) unless garbage_behind, which fills them with data that a
    contributor mask must ignore."""
    rng = np.random.default_rng(spec["seed"])
    n, e = spec["n"], spec["elems"]
    scale = np.float32(10.0 ** spec["scale_exp"])
    arrays = [(rng.standard_normal(e).astype(np.float32) * scale).astype(np.float32) for _ in range(n)]
    if spec["kind"] == "bf16":
        arrays = [bf16_round(a) for a in arrays]
    elif spec["kind"] == "special":
        for a in arrays:
            m = rng.random(e)
            a[m < 0.05] = np.float32(-0.0)
            a[(m >= 0.05) & (m < 0.08)] = np.float32(1e-40)  # subnormal
            a[(m >= 0.08) & (m < 0.10)] = np.float32(3e38) * np.float32(0.25)
    for b in behind_set(spec):
        arrays[b] = (rng.standard_normal(e).astype(np.float32) if garbage_behind
                     else np.zeros(e, dtype=np.float32))
    return arrays


def intra_cases() -> list[dict]:
    """Intra-replica reduce-scatter / all-gather cases (replica.py:241-262):
    the reference tests' shapes (tests/test_replica.py:61-97: hand values,
    n in 2..4 with a remainder-carrying last shard) plus segment_bounds
    splits (replica.py:731) and empty / uneven shards, n = 1..8."""
    rng = np.random.default_rng(0x1A7A)
    out = []

    def seg(total, n):
        base, rem = divmod(total, n)
        b, off = [], 0
        for r in range(n):
            ln = base + (1 if r < rem else 0)
            b.append([off, ln])
            off += ln
        return b

    for i in range(24):
        n = int(rng.integers(2, 5))
        total = int(rng.integers(n, 40))
        cut = total // n
        out.append(dict(n=n, total=total, seed=100 + i, kind="f32",
                        bounds=[[r * cut, cut if r < n - 1 else total - (n - 1) * cut] for r in range(n)]))
    for i, (n, total) in enumerate([(1, 17), (2, 1), (3, 2), (5, 1001), (7, 4097), (8, 65537), (8, 8),
                                    (4, 300_007), (6, 123_457), (2, 1 << 18)]):
        out.append(dict(n=n, total=total, seed=200 + i, kind="f32", bounds=seg(total, n)))
    for i, (n, total) in enumerate([(4, 99_999), (8, 40_000), (3, 7)]):
        out.append(dict(n=n, total=total, seed=300 + i, kind="bf16", bounds=seg(total, n)))
    # uneven, empty and unaligned shards (any caller-given bounds)
    for i in range(6):
        n = int(rng.integers(2, 9))
        total = int(rng.integers(0, 5000))
        cuts = sorted(int(c) for c in rng.integers(0, total + 1, size=n - 1))
        edges = [0, *cuts, total]
        out.append(dict(n=n, total=total, seed=400 + i, kind="f32",
                        bounds=[[edges[r], edges[r + 1] - edges[r]] for r in range(n)]))
    return out
