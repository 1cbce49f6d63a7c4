"""CPU oracle for the FTAR data plane — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker / the CPU baseline; the
product (paper_2602_00277_b200) never calls it and has no CPU fallback.

It restates, in numpy, the reference's arithmetic for the hot path:

* ``partition_plan`` / ``segments``   — build_partition_plan ftar.py:80-99 and
  segment_bounds ftar.py:102-112 (element units of the fp32 view).
* ``oracle_reduce``                  — the closed-form golden function of
  tests/test_ftar.py:20-40: for every segment, a float32 left fold of the
  members in ascending ring order starting at the segment's owner.  The
  reference's socket ring reproduces it bit for bit (criterion 02,
  tests/test_acceptance.py:86-137).
* ``oracle_reduce(..., contrib=)``   — behind replicas contribute a literal
  +0.0 buffer (replica.py:574-577).
* ``normalize``                      — grad *= f32(1/denom) (replica.py:622-626).
* ``sgd_momentum``                   — model.optimizer_step model.py:146-155
  (the §8f "next" row).
* ``decide``-free: membership parity is pinned against decision traces
  recorded from the reference itself (tests/golden/quorum_traces.json).

Parity status: PINNED — tests/test_oracle_golden.py checks this module against
golden vectors produced by running the reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np


def _balanced(total: int, parts: int) -> list[tuple[int, int]]:
    q, r = divmod(total, parts)
    out, off = [], 0
    for i in range(parts):
        ln = q + (1 if i < r else 0)
        out.append((off, ln))
        off += ln
    return out


def partition_plan(total_elems: int, chunk_bytes: int, max_in_flight: int, n: int) -> list[tuple[int, int]]:
    """ftar.py:80-99 in element units."""
    if total_elems == 0:
        return [(0, 0)]
    cap = max(1, (chunk_bytes * max_in_flight * n) // 4)
    return _balanced(total_elems, -(-total_elems // cap))


def segments(part_elems: int, n: int) -> list[tuple[int, int]]:
    """ftar.py:102-112."""
    return _balanced(part_elems, n)


def owners(total_elems: int, chunk_bytes: int, max_in_flight: int, n: int) -> np.ndarray:
    """Ring index whose copy starts each element's fold."""
    own = np.empty(total_elems, dtype=np.int32)
    for p_off, p_len in partition_plan(total_elems, chunk_bytes, max_in_flight, n):
        for j, (s_off, s_len) in enumerate(segments(p_len, n)):
            own[p_off + s_off:p_off + s_off + s_len] = j
    return own


def oracle_reduce(arrays, chunk_bytes: int, max_in_flight: int, contrib=None) -> np.ndarray:
    """tests/test_ftar.py:20-40 (fp32 left fold from the segment owner).

    ``arrays`` are the members' buffers in ring order (fp32, or bf16 given as
    their exact fp32 upcast).  ``contrib`` (optional, one bool per member)
    replaces non-contributors by +0.0, exactly what a behind replica's zero
    buffer contributes in the reference."""
    n = len(arrays)
    arrs = [np.asarray(a, dtype=np.float32) for a in arrays]
    if contrib is not None:
        arrs = [a if c else np.zeros_like(a) for a, c in zip(arrs, contrib)]
    total = arrs[0].size
    out = np.empty(total, dtype=np.float32)
    for p_off, p_len in partition_plan(total, chunk_bytes, max_in_flight, n):
        for owner, (s_off, s_len) in enumerate(segments(p_len, n)):
            lo, hi = p_off + s_off, p_off + s_off + s_len
            acc = arrs[owner][lo:hi].copy()
            for k in range(1, n):
                acc = acc + arrs[(owner + k) % n][lo:hi]
            out[lo:hi] = acc
    return out


def normalize(total: np.ndarray, denom: int) -> np.ndarray:
    """replica.py:622-626: multiply by the fp32-rounded reciprocal (NOT a divide)."""
    return total * np.float32(1.0 / denom)


def sgd_momentum(params: np.ndarray, momentum: np.ndarray, grad: np.ndarray, beta: float, lr: float):
    """model.py:146-155, in place: m *= f32(beta); m += g; p -= f32(lr) * m."""
    momentum *= np.float32(beta)
    momentum += grad
    params -= np.float32(lr) * momentum
    return params, momentum


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 to bf16 (round-to-nearest-even) and return the exact fp32
    upcast — how synthetic bf16 buckets are represented on the CPU side."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    nan = np.isnan(x)
    out = (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
    out = np.where(nan, np.float32(np.nan), out)
    return out.astype(np.float32)


def member_inputs(n: int, elems: int, seed: int = 0, dtype: str = "f32") -> list[np.ndarray]:
    """Synthetic per-replica buckets of SURVEY §8(d): x_r =
    default_rng((seed, r)).standard_normal(E) cast to the bucket dtype
    (bf16 returned as its fp32 upcast)."""
    out = []
    for r in range(n):
        x = np.random.default_rng((seed, r)).standard_normal(elems).astype(np.float32)
        out.append(bf16_round(x) if dtype == "bf16" else x)
    return out


# ---------------------------------------------------- intra-replica collectives


def intra_reduce_scatter(vecs, bounds) -> list[np.ndarray]:
    """replica.py:241-252 (IntraGroup.reduce_scatter): rank r's shard is
    vec_0[b_r] + vec_1[b_r] + ..., an fp32 left fold from rank 0 upward."""
    out = []
    for off, ln in bounds:
        acc = np.asarray(vecs[0], dtype=np.float32)[off:off + ln].copy()
        for v in vecs[1:]:
            acc += np.asarray(v, dtype=np.float32)[off:off + ln]
        out.append(acc)
    return out


def intra_all_gather(shards, bounds, total: int) -> np.ndarray:
    """replica.py:254-262 (IntraGroup.all_gather)."""
    full = np.empty(total, dtype=np.float32)
    for shard, (off, ln) in zip(shards, bounds):
        full[off:off + ln] = shard
    return full
