// ftar_device.cuh — device-side data layout and memory-model helpers of the
// B200 FTAR data plane.  Everything a remote GPU may read lives in a member's
// ARENA (one cudaMalloc, exported with CUDA IPC); everything the host polls or
// writes lives in the pinned, device-mapped control block (HostCtl).
//
// Flag words are 64-bit: [generation:24][call seq:32][bits:8].  A flag only
// satisfies a wait when its (generation, seq) equals the waiter's, so a
// straggler from an abandoned attempt (older generation) can never complete a
// newer wait — the GPU analogue of the generation fencing at
// ftar.py:281-282 / 390-393.  Bulk data moves by peer PULLS, except in push
// mode (out-of-place calls into registered buffers, whose `out` is undefined
// after an error anyway).  Small control records (entry records, arrival
// flags) are pushed into the reader's header so every poll is local; each is
// bound to its call's tag (entry_sum), so a zombie of a dead attempt can delay
// a reader but never redirect it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace ftar {

constexpr int kMaxMembers = 8;
constexpr int kMaxRegions = 16;        // registered buffers per member (RingGroup.register)
constexpr int kThreads = 512;          // one CTA per SM (launch_bounds(512,1))
constexpr uint64_t kHdrBytes = 64 * 1024;
// small-bucket push one-shot: receive slots right after the header, at the
// same offset in every member's arena:
// [generation parity][call parity][sender] x kSmallMax bytes
constexpr uint64_t kSmallMax = 1ull << 20;
constexpr uint64_t kRecvOff = kHdrBytes;
constexpr uint64_t kRecvBytes = 2 * 2 * 8 * kSmallMax;
constexpr uint32_t kBitNonFinite = 1u;

// status codes (mirror include/ftar_b200.h)
enum : uint32_t {
  ST_OK = 0, ST_TIMEOUT = 1, ST_PEER_RESET = 2, ST_PEER_DOWN = 3, ST_PROTOCOL = 4,
  ST_NUMERICAL = 5, ST_INVARIANT = 6, ST_ABORTED = 7, ST_INJECTED = 8,
  ST_UNAVAILABLE = 9, ST_CUDA = 10
};

__host__ __device__ inline uint64_t mk_tag(uint64_t gen, uint64_t seq) {
  return ((gen & 0xffffffull) << 32) | (seq & 0xffffffffull);
}
__host__ __device__ inline uint64_t mk_flag(uint64_t tag, uint32_t bits) {
  return (tag << 8) | (bits & 0xffu);
}
__host__ __device__ inline uint64_t flag_tag(uint64_t f) { return f >> 8; }
__host__ __device__ inline uint64_t tag_gen(uint64_t t) { return t >> 32; }

// What member j announces when it enters a call, PUSHED into slot j of every
// peer's header (posted NVLink writes, one fence, then the flag), so each
// member polls and reads only its own memory: pulling the record cost one
// dependent NVLink round trip (~1.2 us) per field per peer — 25 us per call
// at N=4.  Peers validate it (the analogue of the (partition, ring_step,
// chunk, len) check at ftar.py:394-397): `fp` hashes what the member believes
// the call is (length, geometry, dtype, n, range); `sum` binds the offsets to
// the call's tag, so a stale writer from an aborted generation can never
// redirect a reader.
struct alignas(64) EntryIn {
  uint64_t flag;
  uint64_t fp;       // call fingerprint
  uint64_t in_off;   // input address - arena base (mod 2^64)
  uint64_t res_off;  // result region offset
  uint64_t out_off;  // push mode: `out` (element 0) - arena base; ~0 = not addressable
  uint64_t sum;      // entry_sum(tag, fp, in_off, res_off, out_off)
};

__host__ __device__ inline uint64_t entry_sum(uint64_t tag, uint64_t fp, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = tag * 0xD6E8FEB86659FD93ull ^ fp;
  h ^= (a + 0x9E3779B97F4A7C15ull) + (h << 6) + (h >> 2);
  h ^= (b + 0x632BE59BD9B4E019ull) + (h << 6) + (h >> 2);
  h ^= (c + 0x85EBCA77C2B2AE63ull) + (h << 6) + (h >> 2);
  return h;
}

struct alignas(128) ArenaHdr {
  EntryIn ent_in[kMaxMembers];      // member j's entry record for my current call
  uint64_t ent_ack[kMaxMembers];    // member j has read my entry record of call <tag> (PDL gate)
  alignas(128) uint64_t rs_done;    // flag: my slice is reduced (+kBitNonFinite)
  alignas(128) uint64_t poison;     // flag: I aborted this call (bits = reason)
  alignas(128) uint32_t rs_arrive;  // CTA arrival counters (local atomics)
  uint32_t done_arrive;
  uint32_t nonfinite;
  uint32_t err;
  int32_t err_peer;
  uint32_t pad0;
  uint64_t tiles_done;
  alignas(128) uint64_t dbg_rs_end[256];  // per-CTA %globaltimer at end of reduce-scatter
  uint64_t dbg_ag_end[256];               // per-CTA %globaltimer at end of all-gather
  uint64_t dbg_t1;                        // entry barrier passed (block 0)
  uint64_t dbg_fence[4];                  // last CTA: before/after the sys fence (RS, end)
  uint64_t tph[6];                        // phase stamps: [0] start [1] entry passed [2] RS published
                                          // [3] AG barrier passed [4] end (ftar_phase_times)
  alignas(128) uint64_t go;               // CTA 0 -> local CTAs: (tag << 8) | barrier passed
  uint64_t peer_in[kMaxMembers];          // entry barrier result: member inputs (my VA)
  uint64_t peer_res[kMaxMembers];         // and member result slices (my VA)
  uint32_t peer_bits;                     // RS barrier: OR of members' rs_done bits
  uint32_t vec_ok;
  alignas(128) uint64_t go2;              // direct mode: (tag << 8) | mask of members whose slice is reduced
  uint64_t peer_out[kMaxMembers];         // push mode: members' `out` element 0 (my VA)
  uint32_t push_ok;                       // push mode agreed for this call
  // push mode: member k finished writing its slice of call <tag> into my out,
  // one slot per call parity (with the early PDL trigger a peer can finish
  // call t and start call t+1's reduce-scatter before I have read its flag
  // of call t; call t+2 cannot start before my call t is done)
  alignas(128) uint64_t ag_in[2][kMaxMembers];
  // small one-shot: member k's whole input of call <tag> is in my recv slot,
  // and its call fingerprint (validated like an entry record); one slot per
  // call parity, as the payload slots: a peer that has finished call t may
  // already raise call t+1's flag while I still wait for or re-check its
  // flag of call t (call t+2 cannot start before my call t is done)
  alignas(128) uint64_t sm_in[2][kMaxMembers];
  uint64_t sm_meta[2][kMaxMembers];
  alignas(128) uint32_t sm_arrive[2];        // small one-shot: push-arrival counter per call parity
  alignas(128) uint64_t gen_word;            // the generation my host installed (ftar_set_membership):
                                             // a sender whose call is older stops before pushing here
  alignas(128) uint64_t dbg_trace[512];      // diagnostic build: CTA 0's per-tile pipeline stamps
};
static_assert(sizeof(ArenaHdr) <= kHdrBytes, "header too large");

// Pinned host memory mapped into the device: the control plane's words.
// epoch, live_mask and contrib_mask are read by every kernel at entry (one
// 16-byte load, ctl_mismatch): a mismatch with the launch is PROTOCOL.
struct alignas(64) HostCtl {
  volatile uint64_t epoch;         // host: current generation (quorum.py Decision.generation)
  volatile uint32_t live_mask;     // host: ring members (bit = ring index)
  volatile uint32_t contrib_mask;  // host: members contributing data (healthy)
  volatile uint64_t abort_tag;     // host -> device: abort the call with this tag
  volatile uint64_t started;       // device -> host: tag of the call that began
  volatile uint64_t progress;      // device -> host: work tiles completed
  volatile uint64_t done;          // device -> host: mk_flag(tag, status)
  volatile int64_t detail;         // device -> host: ring index blamed (-1 none)
  volatile int64_t available;      // device -> host: snapshot step available
  // (per-call phase stamps live in ArenaHdr::tph: kernel tails keep `done`
  // as their only PCIe write; ftar_phase_times copies the stamps out)
};

// Snapshot arena header (retention-1 seqlock, checkpoint.py:56-80).
struct alignas(128) SnapHdr {
  uint64_t seq;        // odd while a capture is writing
  int64_t step;        // -1 = nothing captured yet
  uint64_t pbytes, mbytes;
  alignas(128) uint64_t seq_min[kMaxMembers], seq_max[kMaxMembers];  // pull-side, per donor (local)
  uint32_t done_arrive, err;
  uint64_t bytes_done;
  alignas(128) uint64_t next_chunk;   // pull-side: chunks are claimed from this counter, so a
  uint64_t chunks_done;               // second (boost) launch shares the remaining work
};
constexpr uint64_t kSnapHdrBytes = 4096;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_sys32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint64_t ld_acquire_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
// Programmatic dependent launch: wait until the previous kernel on this stream
// has completed (no-op unless this grid was launched with PDL allowed), and
// let the next kernel start once every CTA of this grid has signalled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// 128-bit weak loads/stores that do not allocate in L1: peer data is streamed
// once, and local L1 would otherwise cache NVLink lines (L2 is bypassed for
// peer apertures).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// ---- bulk async copies (TMA engine, non-tensor: cp.async.bulk) + mbarriers.
// Peer (NVLink) addresses are ordinary global addresses to the copy engine:
// one thread moves a whole tile (peer global -> shared, shared -> peer
// global), so the SM's threads only fold; the bytes in flight per SM are the
// pipeline's stages, not its registers.  SASS: UBLKCP / SYNCS.*.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
// Bulk copies always complete (local or peer memory that stays mapped), so
// this wait is bounded only as a safety net: a copy that never lands is a
// programming error and traps the kernel instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t it = 1;; ++it) {
    if (mbar_try_wait(bar, parity)) return;
    if ((it & 1023u) == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 30ull * 1000000000ull) __trap();
    }
  }
}
// global (local or peer) -> shared; completes `bytes` of tx on `bar`
__device__ __forceinline__ void bulk_g2s(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(sdst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// shared -> global (local or peer), tracked by bulk groups
__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               ::"l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N committed groups may still be READING shared memory
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// at most N committed groups may still be incomplete (writes not yet performed)
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// generic-proxy smem writes -> visible to the async proxy (before a bulk store)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
// named barrier over `nthreads` threads (the consumer warps of a CTA)
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ bool nonfinite_bits(float x) {
  return (__float_as_uint(x) & 0x7f800000u) == 0x7f800000u;
}

// Element types of the bucket: the fp32 upcast of bf16 is exact.  The unit of
// vector work is 4 elements per lane, so that every warp-wide load (16 B/lane
// fp32, 8 B/lane bf16) and every fp32 store (16 B/lane) is fully coalesced:
// peer reads bypass L2, so a half-used sector is NVLink bandwidth thrown away.
__device__ __forceinline__ uint2 ld_stream64(const void* p) {
  uint2 r;
  asm volatile("ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// Predicated forms: `on` false issues no load at all (zeros), so a
// non-contributor's buffer costs no NVLink traffic and needs no branch
// between the batched loads.
__device__ __forceinline__ uint4 ld_stream_if(const void* p, bool on) {
  uint4 r;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %5, 0;\n"
      " mov.b32 %0, 0;\n mov.b32 %1, 0;\n mov.b32 %2, 0;\n mov.b32 %3, 0;\n"
      " @q ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n}\n"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "r"((int)on));
  return r;
}
__device__ __forceinline__ uint2 ld_stream64_if(const void* p, bool on) {
  uint2 r;
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n mov.b32 %0, 0;\n mov.b32 %1, 0;\n"
      " @q ld.global.L1::no_allocate.v2.u32 {%0,%1}, [%2];\n}\n"
      : "=r"(r.x), "=r"(r.y) : "l"(p), "r"((int)on));
  return r;
}

struct F32In {
  using T = float;
  using Raw = uint4;
  static constexpr int kBytes = 4;
  __device__ __forceinline__ static float scalar(const float* p, uint64_t e) { return p[e]; }
  __device__ __forceinline__ static Raw load4(const float* p, uint64_t e) { return ld_stream(p + e); }
  __device__ __forceinline__ static Raw load4_if(const float* p, uint64_t e, bool on) { return ld_stream_if(p + e, on); }
  __device__ __forceinline__ static Raw zero() { return make_uint4(0u, 0u, 0u, 0u); }
  __device__ __forceinline__ static void cvt4(const Raw& r, float (&v)[4]) {
    v[0] = __uint_as_float(r.x); v[1] = __uint_as_float(r.y);
    v[2] = __uint_as_float(r.z); v[3] = __uint_as_float(r.w);
  }
};
struct BF16In {
  using T = __nv_bfloat16;
  using Raw = uint2;
  static constexpr int kBytes = 2;
  __device__ __forceinline__ static float up(uint32_t h) { return __uint_as_float(h << 16); }
  __device__ __forceinline__ static float scalar(const __nv_bfloat16* p, uint64_t e) {
    return up(reinterpret_cast<const uint16_t*>(p)[e]);
  }
  __device__ __forceinline__ static Raw load4(const __nv_bfloat16* p, uint64_t e) { return ld_stream64(p + e); }
  __device__ __forceinline__ static Raw load4_if(const __nv_bfloat16* p, uint64_t e, bool on) {
    return ld_stream64_if(p + e, on);
  }
  __device__ __forceinline__ static Raw zero() { return make_uint2(0u, 0u); }
  __device__ __forceinline__ static void cvt4(const Raw& r, float (&v)[4]) {
    v[0] = __uint_as_float(r.x << 16); v[1] = __uint_as_float(r.x & 0xffff0000u);
    v[2] = __uint_as_float(r.y << 16); v[3] = __uint_as_float(r.y & 0xffff0000u);
  }
};

}  // namespace ftar
