"""B200-native data plane of FT-HSDP's fault-tolerant all-reduce (FTAR) and
its non-blocking catch-up transfer (arXiv 2602.00277).

Drop-in modules mirroring the reference package ``ftdp`` for this path:

    ftar        PipelineConfig, build_partition_plan, segment_bounds, iter_chunks,
                classify_error, InflightMeter, RingGroup, ftar_all_reduce, LocalRing
    kernels     accumulate, copy_into, BACKEND, backends
    quorum      Decision, Report, QuorumEngine, StoreQuorum
    checkpoint  SnapshotStore, SnapshotUnavailable, fetch_shard, start_fetch, pick_donor
    errors      FtdpError, Recoverable, Fatal and the reason tags
    fabric      StoreFabric (one process per GPU), LocalFabric (in-process rings)

The data plane is libftar_b200.so (sm_100a CUDA, C-ABI in include/ftar_b200.h);
importing ``ftar``/``kernels``/``checkpoint`` loads it and fails loudly if it
is missing.  ``errors``, ``quorum`` and ``fabric`` are pure Python.
"""

__all__ = ["errors", "quorum", "fabric", "ftar", "kernels", "checkpoint"]
