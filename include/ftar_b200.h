/*
 * ftar_b200.h — C-ABI of the B200-native FTAR data plane (libftar_b200.so).
 *
 * This is the drop-in boundary beneath the reference's Python entry points.
 * Every entry point replaces one piece of the reference's CPU/TCP data plane;
 * the reference file:line each one stands in for is cited beside it
 * (paths relative to the reference package root, pkg/src/ftdp/).
 *
 * Plain pointers and sizes only: no torch types cross this boundary.  Device
 * pointers are CUDA device addresses on the context's device; `stream` is a
 * cudaStream_t passed as void*.  All calls are non-blocking except
 * ftar_ctx_destroy / ftar_wait / ftar_snap_wait.
 *
 * Status convention: functions return FTAR_OK (0) or a positive FTAR_ST_*
 * code.  The Python layer maps each code 1:1 onto the reference's error
 * taxonomy (errors.py:11-22): TIMEOUT/PEER_RESET/PEER_DOWN -> Recoverable,
 * PROTOCOL/NUMERICAL/INVARIANT -> Fatal.
 */
#ifndef FTAR_B200_H
#define FTAR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FTAR_MAX_MEMBERS 8

/* ---- status codes (done-word low byte; also C-ABI return values) ---- */
#define FTAR_OK            0
#define FTAR_ST_TIMEOUT    1   /* Recoverable(TIMEOUT)     ftar.py:382-386 */
#define FTAR_ST_PEER_RESET 2   /* Recoverable(PEER_RESET)  ftar.py:317-318 */
#define FTAR_ST_PEER_DOWN  3   /* Recoverable(PEER_DOWN)   ftar.py:194     */
#define FTAR_ST_PROTOCOL   4   /* Fatal(PROTOCOL_VIOLATION) ftar.py:388-397 */
#define FTAR_ST_NUMERICAL  5   /* Fatal(NUMERICAL)         ftar.py:351-352 */
#define FTAR_ST_INVARIANT  6   /* Fatal(INTERNAL_INVARIANT) ftar.py:311-312 */
#define FTAR_ST_ABORTED    7   /* host abort word honoured (maps to TIMEOUT) */
#define FTAR_ST_INJECTED   8   /* test hook: this member was told to die    */
#define FTAR_ST_UNAVAILABLE 9  /* SnapshotUnavailable      checkpoint.py:48-53 */
#define FTAR_ST_CUDA       10  /* CUDA runtime error (message via ftar_last_error) */
#define FTAR_ST_PENDING    255 /* op still running (ftar_poll only) */

/* ---- input dtypes ---- */
#define FTAR_DT_F32  0
#define FTAR_DT_BF16 1

/* ---- launch flags ---- */
#define FTAR_F_SCALE     1u   /* multiply the fp32 sum by `scale` (replica.py:622-626) */
#define FTAR_F_PROTOCOL  2u   /* in-process ring: run the two-shot flag protocol kernel
                                 (as one GPU per member would) instead of the one-shot */

typedef struct ftar_ctx ftar_ctx;

/* Error text of the last failing call on this thread. */
const char* ftar_last_error(void);
/* Library build string ("sm_100a ..."). */
const char* ftar_version(void);

/* ------------------------------------------------------------------ context
 * One context per (device, ring slot): the shared arena (result region,
 * staging double buffer, registered bucket pool, flag words) plus a pinned,
 * device-mapped control block holding the live mask, contributor mask, epoch
 * word, abort word, progress and done words.
 * Replaces RingGroup.__init__ ftar.py:167-178 (link state) — the arena is
 * what the TCP links were. `exportable` = 1 allocates the arena so that it
 * can be shared with other processes (CUDA IPC). */
int ftar_ctx_create(int device, uint64_t max_bucket_bytes, uint64_t pool_bytes,
                    int exportable, ftar_ctx** out);
int ftar_ctx_destroy(ftar_ctx* ctx);

/* Device address of the arena's registered-bucket pool and its size.
 * Buckets placed there are reduced zero-copy (no staging copy). */
int ftar_ctx_pool(ftar_ctx* ctx, uint64_t* dev_ptr, uint64_t* bytes);

/* IPC handle bytes of the arena (carried over the rendezvous that replaces
 * the HELLO_RING handshake, ftar.py:206-224). buf must hold >= 64 bytes. */
int ftar_ctx_export(ftar_ctx* ctx, void* buf, size_t buflen, size_t* written);

/* Map member `slot`'s arena from its exported handle (cached by slot until
 * ftar_ctx_unmap).  Importing a DIFFERENT handle into an occupied slot fails
 * (FTAR_ST_INVARIANT): slots are never silently re-pointed.  Replaces the
 * dial-right/accept-left of RingGroup.reconfig ftar.py:206-224. */
int ftar_ctx_import(ftar_ctx* ctx, int slot, const void* handle, size_t len,
                    uint64_t arena_bytes);
/* Single-process multi-GPU: map `other` (a context of this process on
 * another device) as member `slot` through peer access (no IPC). */
int ftar_ctx_link_local(ftar_ctx* ctx, int slot, ftar_ctx* other);
/* Drop a member mapping (RingGroup.close_links ftar.py:226-230); refused for
 * a slot of the current ring. */
int ftar_ctx_unmap(ftar_ctx* ctx, int slot);

/* Registered user buffers (any device allocation, e.g. a caching-allocator
 * tensor): the two-shot kernel reads a registered input in place (no staging
 * copy) and pushes results into a registered `out`.  Registration is a
 * collective of the ring (RingGroup.register): each member exports its
 * region (the owning block's IPC handle and the region's offset in it) and
 * imports every peer's before any call uses it.  Up to 16 regions per member.
 * Replaces the staging of buf for the reference's in-place call shape
 * (ftar.py:329-353 copies buf[p] into `work`). */
int ftar_region_register(ftar_ctx* ctx, const void* ptr, uint64_t bytes, int* rid, void* handle, size_t buflen,
                         uint64_t* offset);
int ftar_region_unregister(ftar_ctx* ctx, int rid);
int ftar_region_import(ftar_ctx* ctx, int slot, int rid, const void* handle, size_t len, uint64_t offset,
                       uint64_t bytes);

/* Write the quorum decision into the control words (quorum.py:49-75 ->
 * live mask = members, contributor mask = healthy, epoch = generation).
 * ring_slots[i] = slot (as given to ftar_ctx_import; self = -1) of the
 * member at ring index i (ring order = ascending replica id, ftar.py:202).
 * Resets the per-generation call sequence. */
int ftar_set_membership(ftar_ctx* ctx, const int* ring_slots, int n, int self_index,
                        uint32_t contrib_mask, uint64_t generation);

/* -------------------------------------------------------------- all-reduce
 * Launch one fault-tolerant all-reduce of `n_elems` elements on `stream`.
 * in:  device pointer, dtype FTAR_DT_F32 or FTAR_DT_BF16.
 * out: fp32 device pointer (== in for the reference's in-place fp32 call).
 * The fold order per element is the reference's (partition geometry from
 * chunk_bytes / max_in_flight, ftar.py:80-112; ring order from the owner of
 * the element's segment, tests/test_ftar.py:20-40).  Results are committed
 * to `out` all-or-nothing: on any error `out` is untouched (ftar.py:5-16).
 * Replaces ftar_all_reduce ftar.py:301-326 and _reduce_partition :329-353. */
int ftar_allreduce_launch(ftar_ctx* ctx, const void* in, int in_dtype, float* out,
                          uint64_t n_elems, uint64_t chunk_bytes, int max_in_flight,
                          float scale, uint32_t flags, void* stream);

/* Range form: reduce elements [base_elem, base_elem + n_elems) of a bucket of
 * `total_elems` elements, folding with the WHOLE bucket's partition geometry
 * (so a bucket reduced chunk by chunk — e.g. pipelined with host copies — is
 * bit-identical to one call).  in/out point at element base_elem. */
int ftar_allreduce_launch_range(ftar_ctx* ctx, const void* in, int in_dtype, float* out,
                                uint64_t n_elems, uint64_t base_elem, uint64_t total_elems,
                                uint64_t chunk_bytes, int max_in_flight, float scale,
                                uint32_t flags, void* stream);

/* §8f: the all-reduce with the SGD-momentum step fused in (model.py:146-155,
 * replica.py:622-633): g = sum x f32(scale); m' = f32(m*beta) + g;
 * p' = p - f32(lr*m'), every op separately rounded (bit-exact with the
 * reference).  Out of place (params_out/momentum_out) so that, as in the
 * reference, nothing is applied before the caller's commit vote; grad_out
 * (nullable) optionally receives g.  Each member updates its own copy. */
int ftar_allreduce_sgd_launch(ftar_ctx* ctx, const void* in, int in_dtype, float* grad_out,
                              uint64_t n_elems, uint64_t chunk_bytes, int max_in_flight, float scale,
                              uint32_t flags, const float* params, const float* momentum,
                              float* params_out, float* momentum_out, float lr, float beta,
                              void* stream);

/* §8f rank 2: the intra-replica collectives of an HSDP replica (R ranks,
 * one GPU each), replacing IntraGroup.reduce_scatter / all_gather
 * (replica.py:241-262; tests/test_replica.py:61-97).  `ctx` is a group whose
 * membership is the replica's ranks (ring index = rank).  Shard k of the
 * vector is elements [offs[k], offs[k] + lens[k]) (ftar.segment_bounds at
 * replica.py:731, or any caller-given bounds).
 *   op 1, reduce-scatter: in = this rank's full vector (`total` elements,
 *         f32 or bf16), out = this rank's fp32 shard (lens[rank] elements) =
 *         sum over ranks 0..R-1 of vec_k[shard], folded rank 0 upward
 *         (replica.py:247-249), bit-exact.
 *   op 2, all-gather: in = this rank's fp32 shard, out = the full fp32
 *         vector (`total` elements) on every rank (replica.py:254-262).
 * Completion (ftar_wait) implies every rank has finished reading this rank's
 * input, so the caller may reuse it (the reference's second barrier wait,
 * replica.py:206-208).  Unregistered inputs are staged into the arena. */
int ftar_intra_launch(ftar_ctx* ctx, int op, const void* in, int in_dtype, float* out,
                      uint64_t total, const uint64_t* offs, const uint64_t* lens, void* stream);

/* In-process form (all ranks on ONE device, one cooperative launch, waited
 * with ftar_wait_local) — the shape of the reference's threaded IntraGroup. */
int ftar_local_intra_launch(ftar_ctx** ctxs, int n, int op, const void* const* ins, int in_dtype,
                            float* const* outs, uint64_t total, const uint64_t* offs,
                            const uint64_t* lens, void* stream);

/* In-process ring: all `n` members live on ONE device and are driven by one
 * cooperative launch (the members' kernels wait on one another, so they
 * must be co-resident).  ctxs[i] is the member at ring index i.
 * fault_member/fault_after_tiles: test hook that makes one member stop
 * mid-reduce-scatter (-1 = none).  Mirrors bench._LoopbackRing
 * (bench.py:53-88), n RingGroups in one process. */
int ftar_local_allreduce_launch(ftar_ctx** ctxs, int n, const void* const* ins,
                                int in_dtype, float* const* outs, uint64_t n_elems,
                                uint64_t chunk_bytes, int max_in_flight, float scale,
                                uint32_t flags, uint32_t contrib_mask,
                                int fault_member, int fault_after_tiles, void* stream);

int ftar_local_allreduce_launch_range(ftar_ctx** ctxs, int n, const void* const* ins,
                                      int in_dtype, float* const* outs, uint64_t n_elems,
                                      uint64_t base_elem, uint64_t total_elems,
                                      uint64_t chunk_bytes, int max_in_flight, float scale,
                                      uint32_t flags, uint32_t contrib_mask, int fault_member,
                                      int fault_after_tiles, void* stream);

/* In-process form of ftar_allreduce_sgd_launch (protocol kernel, one device). */
int ftar_local_allreduce_sgd_launch(ftar_ctx** ctxs, int n, const void* const* ins, int in_dtype,
                                    float* const* grad_outs, uint64_t n_elems, uint64_t chunk_bytes,
                                    int max_in_flight, float scale, uint32_t flags,
                                    uint32_t contrib_mask, const float* const* params,
                                    const float* const* momentum, float* const* params_out,
                                    float* const* momentum_out, float lr, float beta, void* stream);

/* Poll the op in flight: *status = FTAR_ST_PENDING while running, else the
 * final code; *progress = work tiles completed (the per-chunk completion
 * counter the CPU polls, cf. _recv_chunk deadlines ftar.py:378-398). */
int ftar_poll(ftar_ctx* ctx, int* status, uint64_t* progress);
/* Set the abort word of every queued collective: kernels drain and report
 * FTAR_ST_ABORTED. */
int ftar_abort(ftar_ctx* ctx);
/* Number of launched collectives not yet collected by ftar_wait (<= 4:
 * callers may enqueue several buckets and wait for them in order). */
int ftar_inflight(ftar_ctx* ctx);
/* Block (GIL-free when called via ctypes) until the OLDEST queued
 * collective is done.  If the kernel has
 * started and progress does not advance for `progress_timeout_s`, write the
 * abort word (per-chunk deadline semantics, ftar.py:382-386).  Returns the
 * final status; *detail receives the ring index of the peer blamed (or -1). */
int ftar_wait(ftar_ctx* ctx, double progress_timeout_s, int* detail);
/* One watcher for an in-process ring (ftar_local_allreduce_launch): tracks
 * every member's progress word, aborts members that stall, fills
 * statuses[i] / details[i].  Returns FTAR_OK once all members are done. */
int ftar_wait_local(ftar_ctx** ctxs, int n, double progress_timeout_s, int* statuses, int* details);
/* CTAs per member for real (one process per GPU) and in-process launches;
 * 0 restores the default (env FTAR_CTAS / FTAR_LOCAL_CTAS, else 32). */
int ftar_set_tuning(int ctas, int local_ctas);
/* Elements each ring index reduces (the contiguous slice geometry), and the
 * grid used — for tests and the in-flight meter. */
int ftar_geometry(uint64_t n_elems, int n, uint64_t* slice_elems, int* ctas, int* threads);

/* The InflightMeter's figure (ftar.py:141-159) for a call of n_elems on an
 * n-member ring (one process per GPU; push = out-of-place into a peer-
 * addressable buffer): the most bytes one peer link can have outstanding
 * (*path: 0 none, 1 small push one-shot, 2 bulk-copy reduce-scatter,
 * 3 register path) and the CTAs of the launch. */
int ftar_inflight_bound(int n, uint64_t n_elems, int in_dtype, uint64_t chunk_bytes, int max_in_flight, int push,
                        uint64_t* bytes_per_link, int* ctas, int* path);

/* -------------------------------------------------------- operator plugin
 * kernels.accumulate / kernels.copy_into (kernels.py:16-48 ->
 * _ckernels.pyx:9-27) on device buffers: dst[i] += src[i] / dst[i] = src[i]. */
int ftar_accumulate(float* dst, const void* src, int src_dtype, uint64_t n, void* stream);
int ftar_copy_into(float* dst, const void* src, int src_dtype, uint64_t n, void* stream);

/* ---------------------------------------------------------------- catch-up
 * Retention-1 snapshot of (params, momentum) for one rank shard
 * (SnapshotStore checkpoint.py:56-80) held in an exportable device arena, and
 * a pull of it by a recovering replica over NVLink on a side stream
 * (fetch_shard checkpoint.py:117-144). */
typedef struct ftar_snap ftar_snap;
int ftar_snap_create(int device, uint64_t capacity_bytes, int exportable, ftar_snap** out);
int ftar_snap_destroy(ftar_snap* s);
int ftar_snap_export(ftar_snap* s, void* buf, size_t buflen, size_t* written);
/* Donor side: capture step's params||momentum (stream-ordered seqlock). */
int ftar_snap_capture(ftar_snap* s, uint64_t step, const void* params, uint64_t pbytes,
                      const void* momentum, uint64_t mbytes, void* stream);
/* Host read of the snapshot header (step, lengths); -1 step if empty. */
int ftar_snap_info(ftar_snap* s, int64_t* step, uint64_t* pbytes, uint64_t* mbytes);
/* Recovering side: map a donor's snapshot arena into `local` (slot cache;
 * a different handle in an occupied slot is refused). */
int ftar_snap_import(ftar_snap* local, int slot, const void* handle, size_t len,
                     uint64_t capacity_bytes);
/* Drop a donor mapping (a dead incarnation's snapshot stays pinned until its
 * last importer unmaps it). */
int ftar_snap_unmap(ftar_snap* local, int slot);
/* The mapped donor's snapshot header, read over NVLink: the step it holds
 * (-1 if none or mid-capture) and its lengths (checkpoint.py:76-80, 132-133). */
int ftar_snap_peer_info(ftar_snap* local, int slot, int64_t* step, uint64_t* pbytes, uint64_t* mbytes);

/* §8f rank 4 (persistent checkpoint, checkpoint.py:157-198): the snapshot's
 * device regions (params, then momentum) and its seqlock word.  A host
 * writer reads `seq` before and after streaming the regions to storage; an
 * odd or changed value means a capture ran in between (the copy is torn). */
int ftar_snap_region(ftar_snap* snap, void** params, void** momentum, uint64_t* pbytes,
                     uint64_t* mbytes, uint64_t* seq, int64_t* step);
/* Pull donor `slot`'s (-1 = local snapshot, for in-process donors) snapshot of
 * `want_step` into dst_params/dst_momentum with `ctas` CTAs on `stream`.
 * The op reports FTAR_ST_UNAVAILABLE (and *available) when the donor holds a
 * different step or re-captured during the pull. */
int ftar_snap_pull_launch(ftar_snap* local, int slot, const ftar_snap* src_local,
                          uint64_t want_step, void* dst_params, uint64_t pbytes,
                          void* dst_momentum, uint64_t mbytes, int ctas, void* stream);
/* Striped pull: chunk c comes from donor slots[c % nslots] (every healthy
 * replica holds the same retention-1 snapshot), spreading the catch-up over
 * all donors' NVLink egress.  nslots <= 8. */
int ftar_snap_pull_multi_launch(ftar_snap* local, const int* slots, int nslots,
                                const ftar_snap* src_local, uint64_t want_step, void* dst_params,
                                uint64_t pbytes, void* dst_momentum, uint64_t mbytes, int ctas,
                                void* stream);
/* Widen the pull in flight: a second grid of `ctas` CTAs on `stream` claims
 * chunks from the same counter (a catch-up runs narrow while the step's
 * collectives need NVLink, then wide).  No-op when the pull has finished. */
int ftar_snap_pull_boost(ftar_snap* local, int ctas, void* stream);
int ftar_snap_poll(ftar_snap* s, int* status, uint64_t* progress, int64_t* available);
int ftar_snap_abort(ftar_snap* s);
int ftar_snap_wait(ftar_snap* s, double progress_timeout_s, int64_t* available);

/* ------------------------------------------------------------- diagnostics
 * Streaming SM copy (dst/src may be peer addresses) with `ctas` CTAs, and
 * peer-access enabling for single-process multi-GPU probes.  Not on the
 * FTAR path; used to characterise NVLink pull vs push bandwidth. */
int ftar_probe_copy(void* dst, const void* src, uint64_t bytes, int ctas, void* stream);
/* The same copy by the TMA engine (cp.async.bulk global->shared->global),
 * one thread per CTA driving a `stages`-deep pipeline of `tile`-byte tiles. */
int ftar_probe_bulk(void* dst, const void* src, uint64_t bytes, int ctas, int tile, int stages, void* stream);
/* %globaltimer stamps of the last call's phases (start, entry passed,
 * reduce-scatter published, all-gather barrier passed, end). */
int ftar_phase_times(ftar_ctx* ctx, uint64_t* out, int n);
/* Diagnostic build: CTA 0's bulk-copy pipeline stamps of the last call
 * ([0,128) refill start, [128,256) refill issued, [256,384) tile landed for
 * warp 0, [384,512) for warp 1). */
int ftar_debug_trace(ftar_ctx* ctx, uint64_t* out, int n);
/* Per-CTA %globaltimer at the end of reduce-scatter / all-gather (last call). */
int ftar_debug_cta_times(ftar_ctx* ctx, uint64_t* rs_end, uint64_t* ag_end, int n);
int ftar_peer_enable(int device, int peer);
/* Fence-cost probe: c = a + b (b remote), load flavour `kind`, per-CTA
 * %globaltimer stamps (loop end, bar.sync, gpu fence, sys fence). */
/* Diagnostic: this GPU's %globaltimer offset to the host's CLOCK_MONOTONIC
 * (min over `reps` pairings), for cross-GPU phase timelines. */
int ftar_probe_clock(int device, int reps, int64_t* offset_ns);

int ftar_probe_fence(float* c, const float* a, const float* b, uint64_t n, int kind, int ctas,
                     uint64_t* stamps, int device, void* stream);
/* Access-pattern probe: mode 0 c=a+b, 1 c=b, 2 loads only, 3 all-local;
 * layout 0 grid-stride, 1 contiguous span per CTA. */
int ftar_probe_pattern(float* c, const float* a, const float* b, uint64_t n, int mode, int layout,
                       int unroll, int ctas, int device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FTAR_B200_H */
