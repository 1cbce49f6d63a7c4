"""Golden fixtures for the intra-replica collectives, made by RUNNING THE
REFERENCE's IntraGroup (pkg/src/ftdp/replica.py:203-262) with rank threads,
exactly as tests/test_replica.py:34-97 does (dev container only).

    python tests/golden/make_intra_golden.py      # needs /root/reference

Writes intra_cases.json: per case (n, total, bounds, seed, kind) and the
sha256 of every rank's reduce_scatter shard and of the all_gather result.
Inputs are regenerated from the seed by tests/golden/gen.py:member_inputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

from gen import intra_cases, member_inputs  # noqa: E402

from ftdp.replica import IntraGroup  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def run_ranks(n, fn):
    out, errs = [None] * n, []

    def main(r):
        try:
            out[r] = fn(r)
        except BaseException as exc:  # noqa: BLE001
            errs.append(exc)

    ts = [threading.Thread(target=main, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    assert not errs, errs
    return out


def main():
    cases = []
    for spec in intra_cases():
        n, total, bounds = spec["n"], spec["total"], [tuple(b) for b in spec["bounds"]]
        vecs = member_inputs(n, total, spec["seed"], spec["kind"])
        g = IntraGroup(n)
        shards = run_ranks(n, lambda r: g.reduce_scatter(r, vecs[r].copy(), bounds))
        full = run_ranks(n, lambda r: g.all_gather(r, shards[r].copy(), bounds, total))
        assert all(np.array_equal(f, full[0]) for f in full)
        cases.append(dict(spec, rs_sha=[sha(s) for s in shards], ag_sha=sha(full[0])))
    with open(os.path.join(HERE, "intra_cases.json"), "w") as f:
        json.dump(cases, f, indent=0)
    print(f"{len(cases)} intra-replica cases")


if __name__ == "__main__":
    main()
