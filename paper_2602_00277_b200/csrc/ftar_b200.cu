// ftar_b200.cu — sm_100a kernels and the C-ABI runtime of the B200 FTAR data
// plane (declared in include/ftar_b200.h).
//
// Hot path (replaces ftar.py:301-398 + kernels.py / _ckernels.pyx):
//   one persistent kernel per member and call, G CTAs x 512 threads:
//     1. entry    publish {input offset, call tag}; wait until every ring
//                 member has entered the same (generation, seq)
//     2. RS       reduce my contiguous slice: 128-bit NVLink loads of every
//                 live member's input, fp32 fold in the reference's order
//                 (per element: start at the owner of its partition segment,
//                 ascending ring index — tests/test_ftar.py:20-40), fused
//                 bf16->fp32 upcast, non-finite detection (warp vote) and the
//                 optional x f32(1/(h*R)) scale (replica.py:622-626); result
//                 to my arena's result region; last CTA publishes rs_done
//     3. barrier  wait for every member's rs_done; any non-finite -> NUMERICAL
//                 (nothing committed anywhere, ftar.py:351-352)
//     4. AG       pull every member's reduced slice over NVLink into `out`
//   Every wait is bounded (generation-tagged flag + peer poison word + host
//   abort word + device hard timeout), so a dead peer turns into a status,
//   never a hung GPU.  The host polls progress/done words in pinned memory.
#include "ftar_device.cuh"
#include "../../include/ftar_b200.h"

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <string>
#include <thread>
#include <vector>

using namespace ftar;

// ============================================================================
// device code
// ============================================================================

namespace {

__host__ __device__ __forceinline__ uint64_t umin(uint64_t a, uint64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ uint64_t umax(uint64_t a, uint64_t b) { return a > b ? a : b; }

constexpr uint32_t ST_FOLLOW = 254;  // stop because another CTA of mine failed
constexpr uint32_t kFlagDirect = 1u << 8;  // internal launch flag: RS writes my slice of out
constexpr uint32_t kFlagPush = 1u << 9;    // internal: all-gather by posted writes into peers' outs
constexpr uint32_t kFlagSGD = 1u << 10;    // internal: apply SGD-momentum to the reduced gradient
constexpr uint32_t kFlagSmallDirect = 1u << 11;  // internal: small one-shot folds straight into out

// Entry-record offsets that name a REGISTERED buffer instead of an arena
// offset: top two bits set, region id in bits 48..59, byte offset below.
// (Arena offsets the kernels dereference are always < 2^62.)
constexpr uint64_t kRegionTag = 3ull << 62;
__host__ __device__ __forceinline__ uint64_t region_ref(uint32_t rid, uint64_t off) {
  return kRegionTag | ((uint64_t)(rid & 0xfffu) << 48) | (off & ((1ull << 48) - 1));
}
__host__ __device__ __forceinline__ bool is_region_ref(uint64_t v) { return (v >> 62) == 3 && v != ~0ull; }

struct LaunchParams {
  char* base[kMaxMembers];       // arena base of ring member i, as mapped here
  HostCtl* ctl[kMaxMembers];     // control block of member i (device view)
  float* out[kMaxMembers];       // fp32 output of member i
  uint64_t in_off[kMaxMembers];  // member i's input address - its arena base
  uint64_t res_off[kMaxMembers]; // member i's result region offset
  uint64_t out_off[kMaxMembers]; // member i's out - arena base (push mode), ~0 = none
  uint64_t tag;
  uint64_t nelems;
  uint64_t slice;                // elements reduced per ring index (multiple of 8)
  uint64_t p_base, p_rem;        // partition lengths: p_rem of p_base+1, rest p_base
  uint64_t cap;                  // partition cap (elements), validated across members
  uint64_t ebase;                // element index of this call's element 0 in the bucket
  uint64_t total;                // bucket length (geometry)
  uint64_t hard_timeout_ns;
  const float* sgd_p[kMaxMembers];  // fused optimizer (§8f): member i's params / momentum in
  const float* sgd_m[kMaxMembers];
  float* sgd_po[kMaxMembers];        // updated params / momentum out (the caller swaps on commit,
  float* sgd_mo[kMaxMembers];        // as replica.py applies the optimizer only after the 2PC vote)
  float sgd_lr, sgd_beta;
  float scale;
  uint32_t flags;
  uint32_t contrib;              // bit i: ring index i contributes data (healthy)
  uint32_t workers;              // bit i: ring index i reduces a slice (contributors; all if none)
  uint32_t dtype;
  int self;                      // my ring index (real mode)
  int emulated;                  // 1: ring index = blockIdx.y (in-process ring)
  int fault_member;              // test hook (-1 none)
  int fault_after_tiles;
  int rs_layout;                 // 0: contiguous span per CTA, 1: grid-strided tiles
  int diag;                      // timing diagnostics: 1 = RS stores skipped, 2 = RS reads local only
  int rs_ctas;                   // CTAs that reduce (the rest only all-gather); <= gridDim.x
  uint32_t tma_stages;           // > 0: bulk-copy (TMA) data path with this many smem stages
  uint32_t early_trigger;        // 1: PDL trigger once the peers have read my entry record
  uint32_t entry_fence;          // 1: system fence between the entry record and its flag
  uint64_t my_in_va;             // real mode: my input as this process addresses it
  uint64_t region_va[kMaxMembers][kMaxRegions];  // member i's registered region r, mapped here (0 = none)
  uint32_t intra_op;             // intra-replica collective (kIntraRS / kIntraAG), 0 = FTAR
  uint64_t seg_off[kMaxMembers]; // intra: rank k's shard is elements [seg_off[k], +seg_len[k])
  uint64_t seg_len[kMaxMembers];
};

__device__ __forceinline__ uint32_t severity_code(uint32_t st) {
  uint32_t sev = (st == ST_INJECTED) ? 3u
               : (st == ST_PROTOCOL || st == ST_NUMERICAL || st == ST_INVARIANT) ? 2u : 1u;
  return (sev << 8) | st;
}

// Bounded wait for *flag to carry `tag`.  Exits early on: the member's poison
// word for this tag (it aborted -> PEER_RESET), a newer generation on the
// flag (I am stale -> PEER_RESET), a newer call of the same generation
// (sequence skew -> PROTOCOL), the host abort word, another CTA of mine
// failing (FOLLOW), or the device hard timeout.
// What a member believes the call is (validated against every peer's).
__device__ __forceinline__ uint64_t call_fingerprint(const LaunchParams& p, int n) {
  uint64_t h = p.nelems * 0x9E3779B97F4A7C15ull;
  h ^= (p.cap + 0x632BE59BD9B4E019ull) + (h << 6) + (h >> 2);
  h ^= ((uint64_t)p.dtype | ((uint64_t)n << 8)) + (h << 6) + (h >> 2);
  h ^= (p.ebase * 31 + p.total) + (h << 6) + (h >> 2);
  h ^= ((uint64_t)p.contrib * 0x94D049BB133111EBull) + (h << 6) + (h >> 2);  // members agree on who contributes
  return h;
}

// The control plane's words for this op, in ONE 16-byte PCIe read of the
// pinned control block: the epoch must be this call's generation and, for a
// real (one GPU per member) launch, the live mask and contributor mask must
// be the ones the launch was built from — a queued op never runs against a
// membership the control plane has since replaced.
struct CtlWords {
  uint64_t epoch, masks;
};
// the 16-byte PCIe read, issued on its own so that its latency overlaps
// whatever the caller issues next (the result is consumed by ctl_check)
__device__ __forceinline__ CtlWords ctl_load(const HostCtl* ctl) {
  CtlWords w;
  asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(w.epoch), "=l"(w.masks) : "l"(ctl) : "memory");
  return w;
}
__device__ __forceinline__ bool ctl_check(const CtlWords& w, uint64_t tag, int n, uint32_t contrib, bool real,
                                          bool check_contrib) {
  if (w.epoch != tag_gen(tag)) return true;
  if (!real) return false;
  const uint32_t all = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
  if ((uint32_t)w.masks != all) return true;
  return check_contrib && (uint32_t)(w.masks >> 32) != contrib;
}
__device__ __forceinline__ bool ctl_mismatch(const HostCtl* ctl, uint64_t tag, int n, uint32_t contrib, bool real,
                                             bool check_contrib) {
  uint64_t e, m;
  asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(e), "=l"(m) : "l"(ctl) : "memory");
  if (e != tag_gen(tag)) return true;
  if (!real) return false;
  const uint32_t all = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
  if ((uint32_t)m != all) return true;
  return check_contrib && (uint32_t)(m >> 32) != contrib;
}

// Zombie guard for kernels that PUSH data into peers' memory: lane j of warp
// 0 reads member j's gen_word (installed by its host at reconfig); a peer
// that has already moved to a newer generation means this call belongs to an
// abandoned ring (this member was dropped on timeout and is running late), so
// it must not write anything there.  Returns the mask of such peers.
__device__ __forceinline__ uint32_t newer_peers(const LaunchParams& p, int n, int me, uint64_t tag) {
  bool newer = false;
  const int j = threadIdx.x & 31;
  if (j < n && j != me)
    newer = ld_relaxed_sys(&reinterpret_cast<const ArenaHdr*>(p.base[j])->gen_word) > tag_gen(tag);
  return __ballot_sync(0xffffffffu, newer);
}

// Member i's reduce-scatter slice.  Only contributors (the workers) reduce:
// a behind replica (replica.py:574-577) owns no slice, issues no loads and
// is served by the others; the fold order is set by the segment owner, not
// by who executes it, so the bits do not change.
__device__ __forceinline__ void slice_of(const LaunchParams& p, int i, uint64_t E, uint64_t& lo, uint64_t& hi) {
  if (!((p.workers >> i) & 1u)) {
    lo = hi = E;
    return;
  }
  const uint64_t w = (uint64_t)__popc(p.workers & ((1u << i) - 1u));
  lo = umin(w * p.slice, E);
  hi = umin(lo + p.slice, E);
}

__device__ uint32_t wait_flag(const uint64_t* flag, uint64_t tag, const uint64_t* poison,
                              const HostCtl* ctl, const uint32_t* own_err, uint64_t t0,
                              uint64_t limit_ns, uint32_t* bits) {
  // Relaxed polls (no fence per poll: acquire loads from many spinning CTAs
  // slow down every other CTA's fences), one acquire load on success,
  // exponential-ish backoff so idle pollers leave NVLink and L2 alone.
  for (uint32_t it = 0;; ++it) {
    const uint64_t f = ld_relaxed_sys(flag);
    const uint64_t ft = flag_tag(f);
    if (ft == tag) {
      // acquire-only: one ld.acquire.sys re-read orders this thread's later
      // reads after the writer's release.  A fence.acq_rel.sys here would also
      // wait for this thread's own outstanding writes (e.g. a PCIe write to
      // the control block) - measured at ~2 us per flag.  A later tag read
      // here still orders correctly: the writer released it after this one.
      (void)ld_acquire_sys(flag);
      if (bits) *bits = (uint32_t)(f & 0xffu);
      return ST_OK;
    }
    // A peer's flag can only move past an op I am still waiting in if that
    // peer abandoned it (it cannot complete without me): a newer generation,
    // or an abort cascade within this one.  Either way the ring is reset;
    // mismatched calls are caught by the entry-record check, not here.
    if (ft > tag) return ST_PEER_RESET;
    if ((it & 15u) == 15u) {
      if (own_err && ld_relaxed_sys32(own_err) != 0) return ST_FOLLOW;
      if (globaltimer_ns() - t0 > limit_ns) return ST_TIMEOUT;
      // the slow checks (a remote load, a PCIe read of the host's abort word:
      // ~1.5 us each) run 4x less often so they rarely delay a flag's arrival
      if ((it & 63u) == 63u) {
        if (poison && flag_tag(ld_relaxed_sys(poison)) >= tag) return ST_PEER_RESET;
        if (ctl->abort_tag == tag) return ST_ABORTED;
      }
    }
    if (it > 4) __nanosleep(it < 64 ? 64 : 256);
  }
}

// Local fan-out: wait for CTA 0 of this member to post `want` on hdr->go.
// Only CTA 0 polls peers and the host; the others spin on one L2 word.
__device__ uint32_t wait_go(const ArenaHdr* hdr, uint64_t want, uint64_t t0, uint64_t limit_ns) {
  for (uint32_t it = 0;; ++it) {
    if (ld_relaxed_gpu(&hdr->go) == want) {
      (void)ld_acquire_gpu(&hdr->go);  // acquire-only (see wait_flag): no wait on this thread's writes
      return ST_OK;
    }
    if ((it & 15u) == 15u) {
      if (ld_relaxed_sys32(&hdr->err) != 0) return ST_FOLLOW;
      if (globaltimer_ns() - t0 > limit_ns) return ST_TIMEOUT;
    }
    if (it > 4) __nanosleep(it < 64 ? 64 : 256);
  }
}

// Direct mode: wait until CTA 0 has seen member k's slice reduced.
__device__ uint32_t wait_go_bit(const ArenaHdr* hdr, uint64_t tag, int k, uint64_t t0, uint64_t limit_ns) {
  for (uint32_t it = 0;; ++it) {
    const uint64_t v = ld_relaxed_gpu(&hdr->go2);
    if (flag_tag(v) == tag && ((v >> k) & 1u)) {
      (void)ld_acquire_gpu(&hdr->go2);  // acquire-only; go2 only gains bits within a call
      return ST_OK;
    }
    if ((it & 15u) == 15u) {
      if (ld_relaxed_sys32(&hdr->err) != 0) return ST_FOLLOW;
      if (globaltimer_ns() - t0 > limit_ns) return ST_TIMEOUT;
    }
    if (it > 4) __nanosleep(it < 64 ? 64 : 256);
  }
}

// Owner (segment index) of element e under the reference geometry
// (build_partition_plan ftar.py:80-99 + segment_bounds ftar.py:102-112), and
// the element index where that segment ends.
__device__ __forceinline__ void owner_of(uint64_t e_local, const LaunchParams& p, int n,
                                         int& owner, uint64_t& seg_end_local) {
  const uint64_t e = e_local + p.ebase;  // range calls fold with the whole bucket's geometry
  uint64_t seg_end;
  const uint64_t big = p.p_rem * (p.p_base + 1);
  if (e < (1ull << 31) && big < (1ull << 31) && p.p_base < (1ull << 31)) {
    // every bucket this library takes (< 2^31 elements): 32-bit divisions,
    // ~5x cheaper than the 64-bit routine (tools/fold_micro.cu: ~650 cycles)
    const uint32_t e32 = (uint32_t)e, big32 = (uint32_t)big, pb = (uint32_t)p.p_base, un = (uint32_t)n;
    uint32_t poff, L;
    if (e32 < big32) {
      poff = e32 / (pb + 1) * (pb + 1);
      L = pb + 1;
    } else {
      poff = big32 + (e32 - big32) / pb * pb;
      L = pb;
    }
    const uint32_t off = e32 - poff, sb = L / un, sr = L - sb * un, sbig = sr * (sb + 1);
    uint32_t j, send;
    if (off < sbig) {
      j = off / (sb + 1);
      send = (j + 1) * (sb + 1);
    } else {
      j = sr + (off - sbig) / sb;
      send = sbig + (j - sr + 1) * sb;
    }
    owner = (int)j;
    seg_end_local = (uint64_t)poff + send - p.ebase;
    return;
  }
  uint64_t poff, L;
  if (e < big) {
    const uint64_t pi = e / (p.p_base + 1);
    poff = pi * (p.p_base + 1);
    L = p.p_base + 1;
  } else {
    const uint64_t pi = (e - big) / p.p_base;
    poff = big + pi * p.p_base;
    L = p.p_base;
  }
  const uint64_t off = e - poff;
  const uint64_t sb = L / (uint64_t)n, sr = L % (uint64_t)n;
  const uint64_t sbig = sr * (sb + 1);
  uint64_t j, send;
  if (off < sbig) {
    j = off / (sb + 1);
    send = (j + 1) * (sb + 1);
  } else {
    j = sr + (off - sbig) / sb;
    send = sbig + (j - sr + 1) * sb;
  }
  owner = (int)j;
  seg_end = poff + send;
  seg_end_local = seg_end - p.ebase;
}

// Where folded values go: one fp32 array (result region or output), two
// (result region + my slice of `out`), or every member's output (in-process
// one-shot).  Arrays are indexed by global element; put4 writes 16 B/lane.
struct SinkOne {
  float* p;
  __device__ __forceinline__ void put1(uint64_t e, float x) const { p[e] = x; }
  __device__ __forceinline__ void put4(uint64_t e, const uint4& v) const { *reinterpret_cast<uint4*>(p + e) = v; }
};
struct SinkNone {  // diagnostics: results computed, never stored
  float* p;
  __device__ __forceinline__ void put1(uint64_t e, float x) const {
    if (__float_as_uint(x) == 0x7fc00001u) p[e] = x;
  }
  __device__ __forceinline__ void put4(uint64_t e, const uint4& v) const {
    if (v.x == 0x7fc00001u && v.y == 0x7fc00001u) *reinterpret_cast<uint4*>(p + e) = v;
  }
};
// Push mode: my folded slice goes to my `out` and, by posted NVLink writes,
// straight into every peer's `out` (the all-gather fused into the reduce).
template <int N>
struct SinkPush {
  float* const* outs;  // members' out (element 0), my VA; outs[me] local
  __device__ __forceinline__ void put1(uint64_t e, float x) const {
#pragma unroll
    for (int j = 0; j < N; ++j) outs[j][e] = x;
  }
  __device__ __forceinline__ void put4(uint64_t e, const uint4& v) const {
#pragma unroll
    for (int j = 0; j < N; ++j) st_stream(outs[j] + e, v);
  }
};
// SGD-momentum on the reduced gradient g, exactly model.optimizer_step
// (model.py:146-155): m = f32(m*beta); m = f32(m + g); p = f32(p - f32(lr*m)).
// Optionally the gradient itself goes to `g_out` too.
struct SgdRefs {
  const float* p;
  const float* m;
  float* po;
  float* mo;
  __device__ __forceinline__ SgdRefs at(uint64_t off) const { return {p + off, m + off, po + off, mo + off}; }
};
__device__ __forceinline__ void sgd4(const SgdRefs& r, uint64_t e, const uint4& gv, float lr, float beta) {
  const uint4 mv = ld_stream(r.m + e), pv = ld_stream(r.p + e);
  float gg[4] = {__uint_as_float(gv.x), __uint_as_float(gv.y), __uint_as_float(gv.z), __uint_as_float(gv.w)};
  float mm[4] = {__uint_as_float(mv.x), __uint_as_float(mv.y), __uint_as_float(mv.z), __uint_as_float(mv.w)};
  float pp[4] = {__uint_as_float(pv.x), __uint_as_float(pv.y), __uint_as_float(pv.z), __uint_as_float(pv.w)};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mm[i] = __fadd_rn(__fmul_rn(mm[i], beta), gg[i]);
    pp[i] = __fsub_rn(pp[i], __fmul_rn(lr, mm[i]));
  }
  st_stream(r.mo + e, make_uint4(__float_as_uint(mm[0]), __float_as_uint(mm[1]), __float_as_uint(mm[2]),
                                 __float_as_uint(mm[3])));
  st_stream(r.po + e, make_uint4(__float_as_uint(pp[0]), __float_as_uint(pp[1]), __float_as_uint(pp[2]),
                                 __float_as_uint(pp[3])));
}
__device__ __forceinline__ void sgd1(const SgdRefs& r, uint64_t e, float g, float lr, float beta) {
  const float mm = __fadd_rn(__fmul_rn(r.m[e], beta), g);
  const float pe = r.p[e];
  r.mo[e] = mm;
  r.po[e] = __fsub_rn(pe, __fmul_rn(lr, mm));
}
struct SinkSGD {  // my slice: result region (peers pull g) + fused update + optional g out
  float* res;
  float* gout;
  SgdRefs r;
  float lr, beta;
  __device__ __forceinline__ void put1(uint64_t e, float x) const {
    res[e] = x;
    if (gout) gout[e] = x;
    sgd1(r, e, x, lr, beta);
  }
  __device__ __forceinline__ void put4(uint64_t e, const uint4& v) const {
    *reinterpret_cast<uint4*>(res + e) = v;
    if (gout) st_stream(gout + e, v);
    sgd4(r, e, v, lr, beta);
  }
};
struct SinkTwo {
  float* p;
  float* q;
  __device__ __forceinline__ void put1(uint64_t e, float x) const { p[e] = x; q[e] = x; }
  __device__ __forceinline__ void put4(uint64_t e, const uint4& v) const {
    *reinterpret_cast<uint4*>(p + e) = v;
    st_stream(q + e, v);
  }
};
template <int N>
struct SinkAll {
  float* const* outs;
  __device__ __forceinline__ void put1(uint64_t e, float x) const {
#pragma unroll
    for (int j = 0; j < N; ++j) outs[j][e] = x;
  }
  __device__ __forceinline__ void put4(uint64_t e, const uint4& v) const {
#pragma unroll
    for (int j = 0; j < N; ++j) st_stream(outs[j] + e, v);
  }
};

// 4-element vectors each thread keeps in flight per source: ~16 loads per
// thread per round whatever the ring size.
template <int N, class In>
struct Unroll {
  // ~256 B of loads per thread; ~192 B from 5 members up, where the members'
  // source and push pointers also live in registers (launch_bounds(512, 1)
  // caps a thread at 128 registers; 256 B at N=8 spilled)
  static constexpr int kBudget = (N >= 6 && sizeof(typename In::Raw) == 8) ? 8 : (N >= 5 ? 12 : 16);
  static constexpr int U0 = (kBudget * 16 / (int)sizeof(typename In::Raw)) / N;
  // the register allocator's sweet spots (ptxas -v); N <= 2 keeps the deep
  // unroll: its bf16 form spills a little but measured 1-2% faster at >= 256 MiB
  static constexpr int kMaxU = N <= 2 ? 16 : (N == 3 ? 6 : 8);
  static constexpr int U = U0 < 1 ? 1 : (U0 > kMaxU ? kMaxU : U0);
};

// Reduce elements [a, b) whose fold starts at ring index s.  All threads of the
// CTA cooperate; each round a thread issues U x N coalesced vector loads
// (out-of-range vectors re-read a valid one and are masked; a
// non-contributor's loads are predicated off and read as +0.0) before the
// first add, so no branch separates the loads; scalars at the ragged edges.
// kAll: every member contributes (the common case), so the loads need no
// predicate: the predicated form's extra moves measured 4% on the HBM-bound
// in-process kernel.
template <int N, class In, int U, class Sink, bool kAll = false>
__device__ __forceinline__ void fold_range(const typename In::T* const* src, const Sink& sink,
                                           uint64_t a, uint64_t b, int s, uint32_t contrib,
                                           bool vec_ok, bool do_scale, float scale,
                                           uint32_t& nf) {
  using T = typename In::T;
  using Raw = typename In::Raw;
  const T* rs[N];
  bool cb[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int m = s + k;
    if (m >= N) m -= N;
    rs[k] = src[m];
    cb[k] = (contrib >> m) & 1u;
  }
  const int tid = threadIdx.x;
  auto scalar_elem = [&](uint64_t e) {
    float acc = cb[0] ? In::scalar(rs[0], e) : 0.0f;
#pragma unroll
    for (int k = 1; k < N; ++k) acc = __fadd_rn(acc, cb[k] ? In::scalar(rs[k], e) : 0.0f);
    nf |= nonfinite_bits(acc) ? 1u : 0u;
    if (do_scale) acc = __fmul_rn(acc, scale);
    sink.put1(e, acc);
  };
  if (!vec_ok) {
    for (uint64_t e = a + tid; e < b; e += kThreads) scalar_elem(e);
    return;
  }
  const uint64_t head = umin(b, (a + 3) & ~3ull);
  if (a + tid < head) scalar_elem(a + tid);
  const uint64_t vb = head >> 2, ve = b >> 2;
  if (vb < ve) {
    for (uint64_t v0 = vb + tid; v0 < ve; v0 += (uint64_t)kThreads * U) {
      Raw raw[U][N];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t v = v0 + (uint64_t)u * kThreads;
        // clamp: keep the load unconditional.  An out-of-range vector
        // re-reads this thread's own first vector: clamping every thread to
        // the same vector (vb) piled up to 512 x (U-1) x N loads on ONE line
        // at the end of every short range (~3.5 us of the small kernel's fold)
        const uint64_t vv = v < ve ? v : v0;
#pragma unroll
        for (int k = 0; k < N; ++k) raw[u][k] = kAll ? In::load4(rs[k], vv * 4) : In::load4_if(rs[k], vv * 4, cb[k]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t v = v0 + (uint64_t)u * kThreads;
        float acc[4], x[4];
        In::cvt4(raw[u][0], acc);
#pragma unroll
        for (int k = 1; k < N; ++k) {
          In::cvt4(raw[u][k], x);
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], x[i]);
        }
        if (v < ve) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            nf |= nonfinite_bits(acc[i]) ? 1u : 0u;
            if (do_scale) acc[i] = __fmul_rn(acc[i], scale);
          }
          sink.put4(v * 4, make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]),
                                      __float_as_uint(acc[2]), __float_as_uint(acc[3])));
        }
      }
    }
  }
  const uint64_t tail = umax(head, ve << 2);
  if (tail + tid < b) scalar_elem(tail + tid);
}

// Fold [lo, hi) in grid-strided tiles (the CTAs' working set stays one
// compact window, which keeps NVLink/TLB locality), caching the current owner
// run so owner_of only runs when a tile crosses a segment boundary.
template <int N, class In, class Sink, bool kOneForm = false>
__device__ __forceinline__ int fold_tiles(const LaunchParams& p, const typename In::T* const* src,
                                          const Sink& sink, uint64_t lo, uint64_t hi, bool vec_ok,
                                          bool do_scale, uint32_t& nf, HostCtl* ctl, int max_tiles,
                                          int layout = -1, int rs_ctas = -1) {
  // layout / rs_ctas override p.rs_layout / p.rs_ctas when >= 0
  constexpr int U = Unroll<N, In>::U;
  const uint64_t TL = (uint64_t)kThreads * 4 * U;
  int done = 0;
  int s = 0;
  uint64_t sbeg = 1, send = 0;  // cached run [sbeg, send) with owner s
  const int rc = rs_ctas >= 0 ? rs_ctas : p.rs_ctas;
  const uint64_t G = (rc > 0 && rc < (int)gridDim.x) ? (uint64_t)rc : gridDim.x;
  if (blockIdx.x >= G) return 0;  // all-gather-only CTA
  uint64_t first = lo + (uint64_t)blockIdx.x * TL, step = G * TL;
  if ((layout >= 0 ? layout : p.rs_layout) == 0) {  // one contiguous span per CTA
    const uint64_t per = ((hi - lo + G - 1) / G + 7) & ~7ull;
    first = umin(lo + (uint64_t)blockIdx.x * per, hi);
    hi = umin(first + per, hi);
    step = TL;
  }
  for (uint64_t a = first; a < hi; a += step) {
    if (done >= max_tiles) return -1;
    const uint64_t b = umin(a + TL, hi);
    uint64_t cur = a;
    while (cur < b) {
      if (cur < sbeg || cur >= send) {
        owner_of(cur, p, N, s, send);
        sbeg = cur;
      }
      const uint64_t end = umin(send, b);
      // kOneForm: only the predicated form (half the code: latency-bound
      // callers pay for instruction-cache misses, not for the predicates)
      if (!kOneForm && ((p.contrib >> 0) & ((1u << N) - 1u)) == ((1u << N) - 1u))
        fold_range<N, In, U, Sink, true>(src, sink, cur, end, s, p.contrib, vec_ok, do_scale, p.scale, nf);
      else
        fold_range<N, In, U, Sink, false>(src, sink, cur, end, s, p.contrib, vec_ok, do_scale, p.scale, nf);
      cur = end;
    }
    ++done;
    if (threadIdx.x == 0 && (done & 63) == 0) ctl->progress = ((uint64_t)blockIdx.x << 32) | (uint64_t)done;
  }
  return done;
}

// The small one-shot's local fold: every thread finds the owner of each of
// its vectors itself, so a bucket cut into N short segments (a 1 KB bucket
// at N=4: four 64-element segments) is folded in ONE round of loads instead
// of one round per segment (fold_tiles walks segments one after another:
// 4 x (owner_of + load round trip) = 3.6 us of the small kernel at 1 KB).
// Same fold order and fusions as fold_range: start at the segment owner,
// then ascending ring index; a vector that straddles two segments is folded
// element by element.
template <int N, class In, class Sink>
__device__ __forceinline__ void fold_small(const LaunchParams& p, const typename In::T* const* src, const Sink& sink,
                                           uint64_t E, bool vec_ok, bool do_scale, uint32_t& nf) {
  using Raw = typename In::Raw;
  constexpr int U = Unroll<N, In>::U;
  const uint32_t contrib = p.contrib;
  const float scale = p.scale;
  const uint64_t gt = (uint64_t)blockIdx.x * kThreads + threadIdx.x, gs = (uint64_t)gridDim.x * kThreads;
  // owner_of costs ~600 cycles: cache the current segment run [sbeg, send)
  // (a thread's elements ascend, so most share a segment)
  uint64_t sbeg = 1, send = 0;
  int sown = 0;
  auto owner_at = [&](uint64_t e) {
    if (e < sbeg || e >= send) {
      owner_of(e, p, N, sown, send);
      sbeg = e;
    }
    return sown;
  };
  auto one = [&](uint64_t e) {
    const int own = owner_at(e);
    float acc = 0.0f;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      int m = own + k;
      if (m >= N) m -= N;
      const float x = ((contrib >> m) & 1u) ? In::scalar(src[m], e) : 0.0f;
      acc = k == 0 ? x : __fadd_rn(acc, x);
    }
    nf |= nonfinite_bits(acc) ? 1u : 0u;
    return do_scale ? __fmul_rn(acc, scale) : acc;
  };
  if (!vec_ok) {
    for (uint64_t e = gt; e < E; e += gs) sink.put1(e, one(e));
    return;
  }
  const uint64_t nv = E >> 2;
  // tiles of kThreads x U vectors, grid-strided over the CTAs (each CTA reads
  // one compact block per round, as fold_tiles does)
  const uint64_t tlv = (uint64_t)kThreads * U;
  for (uint64_t tv = (uint64_t)blockIdx.x * tlv; tv < nv; tv += (uint64_t)gridDim.x * tlv) {
    const uint64_t v0 = tv + threadIdx.x;
    if (v0 >= nv) break;  // (later tiles start further on)
    Raw raw[U][N];
    int own[U];
    bool whole[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = v0 + (uint64_t)u * kThreads;
      const uint64_t e = (v < nv ? v : v0) * 4;  // out of range: re-read my first vector
      own[u] = owner_at(e);
      whole[u] = e + 4 <= send;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        int m = own[u] + k;
        if (m >= N) m -= N;
        raw[u][k] = In::load4_if(src[m], e, (contrib >> m) & 1u);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = v0 + (uint64_t)u * kThreads;
      if (v >= nv) continue;
      float acc[4], x[4];
      if (whole[u]) {
        In::cvt4(raw[u][0], acc);
#pragma unroll
        for (int k = 1; k < N; ++k) {
          In::cvt4(raw[u][k], x);
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], x[i]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          nf |= nonfinite_bits(acc[i]) ? 1u : 0u;
          if (do_scale) acc[i] = __fmul_rn(acc[i], scale);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = one(v * 4 + i);
      }
      sink.put4(v * 4, make_uint4(__float_as_uint(acc[0]), __float_as_uint(acc[1]), __float_as_uint(acc[2]),
                                  __float_as_uint(acc[3])));
    }
  }
  const uint64_t e = (nv << 2) + gt;  // the < 4-element ragged tail
  if (e < E) sink.put1(e, one(e));
}

// Grid-stride fp32 copy (the all-gather pull), 16-byte vectors, UA loads in
// flight per thread before the stores.
// Byte copy of [0, bytes) with 16-byte vectors when aligned.
__device__ __forceinline__ void copy_bytes_grid(char* dst, const char* src, uint64_t bytes,
                                                uint64_t first, uint64_t stride) {
  const bool vec = ((reinterpret_cast<uint64_t>(dst) | reinterpret_cast<uint64_t>(src)) & 15u) == 0;
  if (!vec) {
    for (uint64_t i = first; i < bytes; i += stride) dst[i] = src[i];
    return;
  }
  const uint64_t nv = bytes >> 4;
  constexpr int UA = 8;
  for (uint64_t v = first; v < nv; v += stride * UA) {
    uint4 r[UA];
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const uint64_t i = v + (uint64_t)u * stride;
      if (i < nv) r[u] = ld_stream(src + i * 16);
    }
#pragma unroll
    for (int u = 0; u < UA; ++u) {
      const uint64_t i = v + (uint64_t)u * stride;
      if (i < nv) *reinterpret_cast<uint4*>(dst + i * 16) = r[u];
    }
  }
  const uint64_t t = (nv << 4) + first;
  if (t < bytes && first < 16) dst[t] = src[t];
}

// All-gather pull of a reduced slice straight into the optimizer update
// (gradient never stored unless dst != nullptr).
template <int UA>
__device__ __forceinline__ void pull_sgd(float* dst, const float* src, const SgdRefs& r, uint64_t cnt,
                                         bool vec_ok, float lr, float beta) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t first = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (!vec_ok) {
    for (uint64_t e = first; e < cnt; e += stride) {
      const float g = src[e];
      if (dst) dst[e] = g;
      sgd1(r, e, g, lr, beta);
    }
    return;
  }
  const uint64_t nv = cnt >> 2;
  if (nv) {
    for (uint64_t v = first; v < nv; v += stride * UA) {
      uint4 rv[UA];
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        const uint64_t i = v + (uint64_t)u * stride;
        rv[u] = ld_stream(src + (i < nv ? i : 0) * 4);
      }
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        const uint64_t i = v + (uint64_t)u * stride;
        if (i < nv) {
          if (dst) *reinterpret_cast<uint4*>(dst + i * 4) = rv[u];
          sgd4(r, i * 4, rv[u], lr, beta);
        }
      }
    }
  }
  const uint64_t t = (nv << 2) + first;
  if (t < cnt && first < 4) {
    const float g = src[t];
    if (dst) dst[t] = g;
    sgd1(r, t, g, lr, beta);
  }
}

template <int UA>
__device__ __forceinline__ void copy_f32(float* dst, const float* src, uint64_t cnt, bool vec_ok) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t first = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  if (!vec_ok) {
    for (uint64_t e = first; e < cnt; e += stride) dst[e] = src[e];
    return;
  }
  const uint64_t nv = cnt >> 2;
  if (nv) {
    for (uint64_t v = first; v < nv; v += stride * UA) {
      uint4 r[UA];
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        const uint64_t i = v + (uint64_t)u * stride;
        r[u] = ld_stream(src + (i < nv ? i : 0) * 4);
      }
#pragma unroll
      for (int u = 0; u < UA; ++u) {
        const uint64_t i = v + (uint64_t)u * stride;
        if (i < nv) *reinterpret_cast<uint4*>(dst + i * 4) = r[u];
      }
    }
  }
  const uint64_t t = (nv << 2) + first;
  if (t < cnt && first < 4) dst[t] = src[t];
}

// ---------------------------------------------------------------- bulk-copy (TMA) data path
// The reduce-scatter with the TMA engine moving every remote input byte.  Per
// CTA, a ring of S smem stages; stage s holds one tile (tma_tile(N, in)
// elements) of every contributing PEER's input, landed by cp.async.bulk
// (peer -> shared) on mbarrier full[s].  Warp 15 is the producer: its lane 0
// keeps S-1 tiles of loads in flight, reloading a stage as soon as the 15
// consumer warps have arrived on its empty[s] mbarrier, so the bytes in
// flight per SM are ~(S-1) x (N-1) x tile, not a register budget: 16-32 CTAs
// saturate NVLink where the register-staged loop needed 64-128
// (tools/tma_probe.py: 47 vs 28 GB/s per CTA).  The producer is a warp of its
// own because issuing a bulk copy blocks the issuing thread ~0.2 us; folded
// into a consumer it set the whole CTA's pace (1.3 us per tile,
// tools/tma_fold_probe.py trace).  The 15 consumer warps fold V 4-element
// vectors each per tile: this member's own copy is read straight from its
// buffer (local HBM, prefetched into registers before the tile lands), the
// peers' from shared memory, in the reference order from the segment owner
// with the fused cast / scale / non-finite vote, and the result goes from
// registers by posted 16-byte stores to every destination: the result
// region, my `out`, and in push mode every peer's `out` (the all-gather fused
// in; a bulk store to a peer only releases its smem after the remote write).
// The producer tracks the segment owner incrementally (owner_of's 64-bit
// divisions only when a tile crosses a segment end).  Non-contributors' tiles
// are never loaded (their +0.0 is folded from a register).  Needs every
// segment to be >= one tile (at most one owner change per tile) and 16-byte
// aligned buffers; anything else takes fold_tiles.
constexpr uint32_t kTmaMetaBytes = 1024;              // mbarriers + per-stage tile metadata
// dynamic smem per CTA (1 CTA / SM): 227 KB less room for the kernel's
// static shared variables and the 1 KB alignment of the dynamic window
constexpr uint32_t kTmaSmemMax = 227 * 1024 - 2048;
constexpr uint32_t kTmaMaxStages = 16;
constexpr uint32_t kTmaConsumers = kThreads - 32;     // warps 0..14 fold, warp 15 produces
constexpr int kTmaProducer = kThreads - 32;           // thread that issues the bulk copies

// vectors per consumer thread per tile: ~24 KB of peer data per stage, so
// that >= 8 stages (>= 8 bulk copies) are in flight per SM where the ring is
// small — one copy lands at ~10 GB/s and an SM's copy engine needs several
// in flight to reach its ~47 GB/s (tools/tma_probe.py, tma_fold_probe.py)
__host__ __device__ constexpr uint32_t tma_vecs(int n, int in_bytes) {
  const uint32_t per_vec = (uint32_t)(n > 1 ? n - 1 : 1) * kTmaConsumers * 4u * (uint32_t)in_bytes;
  const uint32_t v = 24576u / per_vec;
  return v < 1 ? 1u : (v > 4 ? 4u : v);
}
__host__ __device__ constexpr uint32_t tma_tile(int n, int in_bytes) {
  return kTmaConsumers * 4u * tma_vecs(n, in_bytes);
}

struct TmaMeta {            // what the producer recorded for the tile in a stage
  uint64_t a;               // first element (call-local)
  uint32_t cnt;             // elements (multiple of 8)
  int s0, s1;               // owner of [a, bnd) and of [bnd, a + cnt)
  uint32_t bnd;             // boundary offset within the tile (>= cnt: none)
};
// smem map: [0,128) full[16] | [128,256) empty[16] | [256,640) meta[16] | stages
__device__ __forceinline__ uint64_t* tma_full(char* smem) { return reinterpret_cast<uint64_t*>(smem); }
__device__ __forceinline__ uint64_t* tma_empty(char* smem) { return reinterpret_cast<uint64_t*>(smem + 128); }
__device__ __forceinline__ TmaMeta* tma_meta(char* smem) { return reinterpret_cast<TmaMeta*>(smem + 256); }

__host__ __device__ __forceinline__ uint64_t tma_stage_off() { return kTmaMetaBytes; }
// one stage = a tile of every PEER's input (this member's own copy is read
// from global memory): peer k sits in slot k - (k > me)
__host__ __device__ __forceinline__ uint64_t tma_stage_bytes(int n, int in_bytes) {
  return (uint64_t)(n > 1 ? n - 1 : 1) * tma_tile(n, in_bytes) * (uint64_t)in_bytes;
}
__device__ __forceinline__ uint32_t tma_slot(int k, int me) { return (uint32_t)(k - (k > me ? 1 : 0)); }
__host__ __device__ __forceinline__ uint32_t tma_stages_for(int n, int in_bytes) {
  const uint64_t s = (kTmaSmemMax - tma_stage_off()) / tma_stage_bytes(n, in_bytes);
  return (uint32_t)(s > kTmaMaxStages ? kTmaMaxStages : s);
}
__host__ __device__ __forceinline__ uint64_t tma_smem_bytes(int n, int in_bytes, uint32_t stages) {
  return tma_stage_off() + (uint64_t)stages * tma_stage_bytes(n, in_bytes);
}

// The producer's cached owner run [sbeg, send) -> owner (fold_tiles does the same).
struct OwnerRun {
  uint64_t sbeg = 1, send = 0;
  int owner = 0;
};

// Issue the bulk loads of the tile at element `a` (cnt elements) into stage
// j % S (j = the CTA-local sequence number, which also sets the phases).
template <int N, class In>
__device__ __forceinline__ void tma_issue(const LaunchParams& p, const typename In::T* const* src, int me, char* smem,
                                          uint32_t S, uint64_t a, uint32_t cnt, uint64_t j, OwnerRun& run) {
  constexpr uint32_t TE = tma_tile(N, In::kBytes);
  uint64_t* full = tma_full(smem);
  TmaMeta* meta = tma_meta(smem);
  const uint32_t s = (uint32_t)(j % S);
  if (a < run.sbeg || a >= run.send) {
    owner_of(a, p, N, run.owner, run.send);
    run.sbeg = a;
  }
  TmaMeta m;
  m.a = a;
  m.cnt = cnt;
  m.s0 = run.owner;
  m.s1 = run.owner;
  m.bnd = 0xffffffffu;
  if (run.send < a + cnt) {  // one owner change inside the tile (segments >= a tile)
    const uint64_t b = run.send;
    owner_of(b, p, N, run.owner, run.send);
    run.sbeg = b;
    m.s1 = run.owner;
    m.bnd = (uint32_t)(b - a);
  }
  meta[s] = m;
  const uint32_t bytes = cnt * (uint32_t)In::kBytes;
  const uint32_t peers = p.contrib & ((1u << N) - 1u) & ~(1u << me);
  char* stage = smem + tma_stage_off() + (uint64_t)s * tma_stage_bytes(N, In::kBytes);
  if (peers == 0) {
    mbar_arrive(&full[s]);
    return;
  }
  mbar_expect_tx(&full[s], bytes * (uint32_t)__popc(peers));
#pragma unroll
  for (int k = 0; k < N; ++k)
    if ((peers >> k) & 1u) bulk_g2s(stage + (uint64_t)tma_slot(k, me) * TE * In::kBytes, src[k] + a, bytes, &full[s]);
}

// Fold one 4-element vector (elements off..off+3 of the tile) whose fold
// starts at ring index `own`: member `me`'s copy from registers (`mine`),
// every other contributor's from the stage.
template <int N, class In>
__device__ __forceinline__ void tma_fold_vec(const char* stage, uint32_t off, int own, int me, uint32_t contrib,
                                             const typename In::Raw& mine, float (&acc)[4]) {
  using Raw = typename In::Raw;
  constexpr uint32_t TE = tma_tile(N, In::kBytes);
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int m = own + k;
    if (m >= N) m -= N;
    float x[4];
    if (!((contrib >> m) & 1u)) {
      x[0] = x[1] = x[2] = x[3] = 0.0f;
    } else if (m == me) {
      In::cvt4(mine, x);
    } else {
      In::cvt4(*reinterpret_cast<const Raw*>(stage + ((uint64_t)tma_slot(m, me) * TE + off) * In::kBytes), x);
    }
    if (k == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = x[i];
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = __fadd_rn(acc[i], x[i]);
    }
  }
}
template <int N, class In>
__device__ __forceinline__ float tma_fold_one(const char* stage, uint32_t off, int own, int me, uint32_t contrib,
                                              const typename In::T* mine_g, uint64_t e) {
  constexpr uint32_t TE = tma_tile(N, In::kBytes);
  float acc = 0.0f;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int m = own + k;
    if (m >= N) m -= N;
    float x = 0.0f;
    if ((contrib >> m) & 1u) {
      const uint64_t at = (uint64_t)tma_slot(m, me) * TE + off;
      if (m == me) x = In::scalar(mine_g, e);
      else if (In::kBytes == 4) x = *reinterpret_cast<const float*>(stage + at * 4);
      else x = __uint_as_float((uint32_t)*reinterpret_cast<const uint16_t*>(stage + at * 2) << 16);
    }
    acc = k == 0 ? x : __fadd_rn(acc, x);
  }
  return acc;
}

// Reduce my slice [lo, hi) through the bulk-copy pipeline; every result
// vector goes to `sink` (put4 / put1 by call-local element).  The < 8-element
// ragged tail of the slice is folded by the last CTA with fold_range.
// Returns tiles done, or -1 when the fault hook stopped it.
template <int N, class In, class Sink>
__device__ int fold_tiles_tma(const LaunchParams& p, const typename In::T* const* src, int me, const Sink& sink,
                              uint64_t lo, uint64_t hi, bool do_scale, uint32_t& nf, HostCtl* ctl, int max_tiles,
                              char* smem) {
  using Raw = typename In::Raw;
  constexpr uint32_t TE = tma_tile(N, In::kBytes);
  constexpr uint32_t V = tma_vecs(N, In::kBytes);
  const int tid = threadIdx.x;
  const uint32_t S = p.tma_stages;
  uint64_t* full = tma_full(smem);
  uint64_t* empty = tma_empty(smem);
  const TmaMeta* meta = tma_meta(smem);
  const uint64_t G = (p.rs_ctas > 0 && p.rs_ctas < (int)gridDim.x) ? (uint64_t)p.rs_ctas : gridDim.x;
  if (blockIdx.x >= G) return 0;
  const uint64_t len = hi > lo ? hi - lo : 0;
  const uint64_t lenv = len & ~7ull;  // bulk-copied part (16-byte granules for bf16 and fp32)
  const uint64_t ntiles = (lenv + TE - 1) / TE;
  const uint64_t per = (ntiles + G - 1) / G;
  const uint64_t t0 = umin(blockIdx.x * per, ntiles), t1 = umin(t0 + per, ntiles);
  const uint64_t cnt = t1 - t0;
  const float scale = p.scale;
  const uint64_t run = umin(cnt, (uint64_t)(max_tiles < 0 ? 0 : max_tiles));  // the fault hook stops early
  const uint64_t end = lo + lenv;
  const bool i_contribute = (p.contrib >> me) & 1u;
  const typename In::T* const mine_g = src[me];
#ifdef FTAR_DIAGNOSTICS
  uint64_t* trace = (p.diag >= 3 && blockIdx.x == 0 && (p.emulated == 0 || blockIdx.y == 0))
                        ? reinterpret_cast<ArenaHdr*>(p.base[p.emulated ? blockIdx.y : p.self])->dbg_trace
                        : nullptr;
#endif
  if (tid >= (int)kTmaConsumers) {
    // ---- producer warp (the kernel initialised the mbarriers at entry)
    if (tid == kTmaProducer) {
      OwnerRun orun;
      for (uint64_t j = 0; j < run; ++j) {
        if (j >= S) mbar_wait(&empty[j % S], (uint32_t)(((j / S) - 1) & 1));  // tile j-S left the stage
#ifdef FTAR_DIAGNOSTICS
        if (trace && j < 128) trace[j] = globaltimer_ns();
#endif
        const uint64_t a = lo + (t0 + j) * TE;
        tma_issue<N, In>(p, src, me, smem, S, a, (uint32_t)umin(TE, end - a), j, orun);
#ifdef FTAR_DIAGNOSTICS
        if (trace && j < 128) trace[128 + j] = globaltimer_ns();
#endif
      }
    }
  } else {
    // ---- consumer warps
    // this member's own copy comes from local HBM by plain loads, issued one
    // tile ahead so their latency hides behind the previous tile's fold
    Raw mine[V], ahead[V];
    auto load_mine = [&](uint64_t jj, Raw (&dst)[V]) {
      const uint64_t a = lo + (t0 + jj) * TE;
      const uint32_t tcnt = (uint32_t)umin(TE, end - a);
#pragma unroll
      for (uint32_t v = 0; v < V; ++v) {
        const uint32_t off = (v * kTmaConsumers + (uint32_t)tid) * 4;
        // past the tile's end: re-read a vector of the tile spread by thread
        // (one shared address would queue every such load on one line)
        dst[v] = In::load4_if(mine_g, a + (off < tcnt ? off : ((uint32_t)tid * 4) % tcnt), i_contribute);
      }
    };
    if (run > 0) load_mine(0, ahead);
    for (uint64_t j = 0; j < run; ++j) {
      const uint32_t s = (uint32_t)(j % S);
#pragma unroll
      for (uint32_t v = 0; v < V; ++v) mine[v] = ahead[v];
      if (j + 1 < run) load_mine(j + 1, ahead);
      mbar_wait(&full[s], (uint32_t)((j / S) & 1));
#ifdef FTAR_DIAGNOSTICS
      if (trace && tid == 0 && j < 128) trace[256 + j] = globaltimer_ns();
      if (trace && tid == 32 && j < 128) trace[384 + j] = globaltimer_ns();
#endif
      const TmaMeta m = meta[s];
      const char* stage = smem + tma_stage_off() + (uint64_t)s * tma_stage_bytes(N, In::kBytes);
      float acc[V][4];
#pragma unroll
      for (uint32_t v = 0; v < V; ++v) {
        const uint32_t off = (v * kTmaConsumers + (uint32_t)tid) * 4;
        acc[v][0] = acc[v][1] = acc[v][2] = acc[v][3] = 0.f;
#ifdef FTAR_DIAGNOSTICS
        if (off < m.cnt && p.diag != 4) {  // diag 4: loads only
#else
        if (off < m.cnt) {
#endif
          if (off + 4 <= m.bnd || off >= m.bnd) {
            tma_fold_vec<N, In>(stage, off, off >= m.bnd ? m.s1 : m.s0, me, p.contrib, mine[v], acc[v]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              acc[v][i] = tma_fold_one<N, In>(stage, off + i, off + i >= m.bnd ? m.s1 : m.s0, me, p.contrib,
                                              mine_g, m.a + off + i);
          }
        }
      }
      // this warp is done with the stage: let the producer reload it
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[s]);
#pragma unroll
      for (uint32_t v = 0; v < V; ++v) {
        const uint32_t off = (v * kTmaConsumers + (uint32_t)tid) * 4;
        if (off < m.cnt) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            nf |= nonfinite_bits(acc[v][i]) ? 1u : 0u;
            if (do_scale) acc[v][i] = __fmul_rn(acc[v][i], scale);
          }
#ifdef FTAR_DIAGNOSTICS
          if (p.diag != 3)  // diag 3: no stores
#endif
            sink.put4(m.a + off, make_uint4(__float_as_uint(acc[v][0]), __float_as_uint(acc[v][1]),
                                            __float_as_uint(acc[v][2]), __float_as_uint(acc[v][3])));
        }
      }
      if (tid == 0 && ((j + 1) & 63) == 0) ctl->progress = ((uint64_t)blockIdx.x << 32) | (uint64_t)(j + 1);
    }
  }
  // every stage is consumed (the all-gather copies reuse the ring with the
  // sequence continuing at `run`)
  __syncthreads();
  if (run < cnt) return -1;
  if (lenv < len && blockIdx.x == G - 1) {  // ragged tail (< 8 elements): plain loads
    int s0;
    uint64_t send;
    uint64_t cur = lo + lenv;
    while (cur < hi) {
      owner_of(cur, p, N, s0, send);
      const uint64_t e2 = umin(send, hi);
      fold_range<N, In, 1>(src, sink, cur, e2, s0, p.contrib, false, do_scale, scale, nf);
      cur = e2;
    }
  }
  return (int)cnt;
}

// All-gather pull of one member's fp32 slice with the TMA engine: the CTAs
// split [0, cnt) into contiguous spans; thread 0 streams each span through
// the smem stages (peer -> shared -> my out).  The < 4-element tail is copied
// by plain loads.
__device__ void tma_copy_span(float* dst, const float* src, uint64_t cnt, char* smem, uint32_t S_bytes_stages,
                              uint32_t tile_bytes, uint32_t& phase_base) {
  uint64_t* full = tma_full(smem);
  char* stages = smem + tma_stage_off();
  const uint32_t S = S_bytes_stages;
  const uint64_t te = tile_bytes / 4;
  const uint64_t cntv = cnt & ~3ull;
  const uint64_t ntiles = (cntv + te - 1) / te;
  const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = umin((uint64_t)blockIdx.x * per, ntiles), t1 = umin(t0 + per, ntiles);
  if (threadIdx.x == 0) {
    const uint64_t n = t1 - t0;
    const uint64_t L = S - 1;
    for (uint64_t j = 0; j < n + L; ++j) {
      if (j < n) {
        const uint64_t g = phase_base + j;  // global sequence through the stage ring
        const uint32_t s = (uint32_t)(g % S);
        if (j >= S) bulk_wait_read<0>();
        const uint64_t a = (t0 + j) * te;
        const uint32_t bytes = (uint32_t)(umin(te, cntv - a) * 4);
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(stages + (uint64_t)s * tile_bytes, src + a, bytes, &full[s]);
      }
      if (j >= L) {
        const uint64_t jj = j - L;
        const uint64_t g = phase_base + jj;
        const uint32_t s = (uint32_t)(g % S);
        mbar_wait(&full[s], (uint32_t)((g / S) & 1));
        const uint64_t a = (t0 + jj) * te;
        const uint32_t bytes = (uint32_t)(umin(te, cntv - a) * 4);
        bulk_s2g(dst + a, stages + (uint64_t)s * tile_bytes, bytes);
        bulk_commit();
      }
    }
    bulk_wait_read<0>();
    phase_base += (uint32_t)n;
    for (uint64_t e = cntv; e < cnt; ++e)
      if (blockIdx.x == 0) dst[e] = src[e];
  }
}

template <int N, class In>
__global__ void __launch_bounds__(kThreads, 1) allreduce_kernel(const __grid_constant__ LaunchParams p) {
  using T = typename In::T;
  const int me = p.emulated ? (int)blockIdx.y : p.self;
  char* const mybase = p.base[me];
  ArenaHdr* const hdr = reinterpret_cast<ArenaHdr*>(mybase);
  HostCtl* const ctl = p.ctl[me];
  const uint64_t tag = p.tag;
  const uint64_t E = p.nelems;
  const int tid = threadIdx.x;
  uint64_t lo, hi;
  slice_of(p, me, E, lo, hi);
  // direct: my reduced slice goes straight into `out` (out-of-place calls);
  // res_off then addresses element `lo` of my out inside my arena, so peers
  // pull my slice from there (p.res_off is already that when out is registered)
  const bool direct = (p.flags & kFlagDirect) != 0;

  __shared__ const T* s_src[N];
  __shared__ const float* s_res[N];
  __shared__ float* s_out[N];
  __shared__ int s_push;
  __shared__ uint32_t s_status;
  __shared__ int s_blame;
  __shared__ uint32_t s_nf;
  __shared__ int s_vec_ok;
  __shared__ uint64_t s_t0;

  __shared__ uint64_t s_pin[N], s_pres[N], s_pout[N];  // CTA 0: entry results, staged for the fan-out
  __shared__ uint32_t s_pushok;
  __shared__ uint32_t s_newer;
  extern __shared__ __align__(1024) char dsmem[];  // bulk-copy stages (p.tma_stages > 0)

  if (tid == 0) {
    s_status = ST_OK;
    s_blame = -1;
    s_nf = 0;
    s_push = 0;
    s_t0 = globaltimer_ns();
    if (p.tma_stages) {
      for (uint32_t s = 0; s < p.tma_stages; ++s) {
        mbar_init(tma_full(dsmem) + s, 1);
        mbar_init(tma_empty(dsmem) + s, kTmaConsumers / 32);
      }
      fence_mbar_init();
    }
  }
  // push mode writes into peers' outputs: never from an abandoned generation.
  // (Warp 1 in CTA 0, whose warp 0 runs the entry concurrently: the remote
  // reads cost an NVLink round trip.)  s_newer is read after __syncthreads.
  const int zw = blockIdx.x == 0 ? 1 : 0;
  if ((tid >> 5) == zw) {
    const uint32_t m = (!p.emulated && (p.flags & kFlagPush)) ? newer_peers(p, N, me, tag) : 0u;
    if ((tid & 31) == 0) s_newer = m;
  }
  if (blockIdx.x == 0 && tid < 32) {
    // ---- 1a. entry (may overlap the previous call's tail: PDL) ------------
    // Until griddepcontrol.wait below this touches only this call's control
    // slot, slot `me` of the peers' ent_in[] and my own ent_in[] (no earlier
    // call reads those any more) - never the rest of my header, which the
    // previous kernel on this stream may still be resetting.
    __syncwarp();
    if (tid == 0) {
      // Epoch fence: an op queued under an older decision must not run
      // against the membership the control plane has since installed.  The
      // PCIe read is issued first and checked after the entry pushes, so its
      // ~1.5 us overlaps them and the flags' flight.  (A stale op that
      // already published is harmless: its tag matches no current peer call,
      // and it poisons itself below.)
      const CtlWords cw = ctl_load(ctl);
      if (N > 1) {
        // push my entry record into slot `me` of every peer's header: posted
        // writes, then the flags (the peers poll locally)
        const uint64_t fp = call_fingerprint(p, N);
        const uint64_t oo = (p.flags & kFlagPush) ? p.out_off[me] : ~0ull;
        const uint64_t sum = entry_sum(tag, fp, p.in_off[me], p.res_off[me], oo);
        for (int jj = 1; jj < N; ++jj) {
          EntryIn* e = &reinterpret_cast<ArenaHdr*>(p.base[(me + jj) % N])->ent_in[me];
          st_relaxed_sys(&e->fp, fp);
          st_relaxed_sys(&e->in_off, p.in_off[me]);
          st_relaxed_sys(&e->res_off, p.res_off[me]);
          st_relaxed_sys(&e->out_off, oo);
          st_relaxed_sys(&e->sum, sum);
        }
        // No fence between the record and its flag: the reader re-reads the
        // record until its checksum (over this call's tag) holds, which
        // costs nothing once the writes land, where a system fence waits a
        // full NVLink round trip for their acks (FTAR_ENTRY_FENCE=1 restores it)
        if (p.entry_fence) fence_acq_rel_sys();
        for (int jj = 1; jj < N; ++jj)
          st_relaxed_sys(&reinterpret_cast<ArenaHdr*>(p.base[(me + jj) % N])->ent_in[me].flag, mk_flag(tag, 0));
      }
      if (ctl_check(cw, tag, N, p.contrib, !p.emulated, true)) {
        s_status = ST_PROTOCOL;
        s_blame = me;
      }
      ctl->started = tag;
    }
    __syncwarp();
    // lane j waits for member j's record and validates it (all peers at once)
    const int j = tid;
    uint32_t st = ST_OK;
    uint64_t oo = 0;
    if (s_status == ST_OK && j < N) {
      if (j == me) {
        s_pin[j] = p.emulated ? reinterpret_cast<uint64_t>(mybase) + p.in_off[me] : p.my_in_va;
        s_pres[j] = reinterpret_cast<uint64_t>(mybase) + p.res_off[me];
        s_pout[j] = reinterpret_cast<uint64_t>(p.out[me]);
      } else {
        const uint64_t want_fp = call_fingerprint(p, N);
        ArenaHdr* ph = reinterpret_cast<ArenaHdr*>(p.base[j]);
        EntryIn* e = &hdr->ent_in[j];  // local: member j pushed it here
        // own_err = null: hdr->err still belongs to the previous call here
        st = wait_flag(&e->flag, tag, &ph->poison, ctl, nullptr, s_t0, p.hard_timeout_ns, nullptr);
        if (st == ST_OK) {
          // the flag can overtake the record (no writer fence): re-read until
          // the record is this call's (its checksum covers the tag).  A writer
          // that died mid-record leaves it torn: its poison word, the host's
          // abort or the call's hard timeout end the wait, as in wait_flag.
          uint64_t fp, in_off, res_off, sum;
          for (uint32_t it = 0;; ++it) {
            fp = ld_relaxed_sys(&e->fp);
            in_off = ld_relaxed_sys(&e->in_off);
            res_off = ld_relaxed_sys(&e->res_off);
            oo = ld_relaxed_sys(&e->out_off);
            sum = ld_relaxed_sys(&e->sum);
            if (sum == entry_sum(tag, fp, in_off, res_off, oo)) break;
            if ((it & 63u) == 63u) {
              if (flag_tag(ld_relaxed_sys(&ph->poison)) >= tag) st = ST_PEER_RESET;
              else if (ctl->abort_tag == tag) st = ST_ABORTED;
              else if (globaltimer_ns() - s_t0 > p.hard_timeout_ns) st = ST_TIMEOUT;
              if (st != ST_OK) break;
            }
            if (it > 4) __nanosleep(64);
          }
          if (st == ST_OK && fp != want_fp) st = ST_PROTOCOL;  // a different call
          // arena offsets, or references to member j's registered buffers
          // (mapped here by RingGroup.register); an unmapped region is a
          // protocol error, never a guess
          // (in-process rings pass raw offsets, which may be "negative")
          auto resolve = [&](uint64_t off) -> uint64_t {
            if (p.emulated || !is_region_ref(off)) return reinterpret_cast<uint64_t>(p.base[j]) + off;
            const uint32_t rid = (uint32_t)(off >> 48) & 0xfffu;
            const uint64_t va = rid < kMaxRegions ? p.region_va[j][rid] : 0;
            return va ? va + (off & ((1ull << 48) - 1)) : 0;
          };
          s_pin[j] = resolve(in_off);
          s_pres[j] = reinterpret_cast<uint64_t>(p.base[j]) + res_off;
          s_pout[j] = oo == ~0ull ? 0 : resolve(oo);
          const bool unmapped = !p.emulated && ((is_region_ref(in_off) && s_pin[j] == 0) ||
                                                (oo != ~0ull && is_region_ref(oo) && s_pout[j] == 0));
          if (st == ST_OK && unmapped) st = ST_PROTOCOL;
          // tell member j its record is consumed (after the loads above: the
          // store is control-dependent on their values)
          if (st == ST_OK) st_relaxed_sys(&ph->ent_ack[me], tag);
        }
      }
    }
    const uint32_t bad = __ballot_sync(0xffffffffu, st != ST_OK);
    // push mode only if every member accepts pushes
    const uint32_t nopush = __ballot_sync(0xffffffffu, j < N && j != me && oo == ~0ull);
    const uint32_t st_first = __shfl_sync(0xffffffffu, st, bad ? __ffs(bad) - 1 : 0);
    if (tid == 0) {
      if (bad) {
        s_status = st_first;
        s_blame = __ffs(bad) - 1;
      }
      s_pushok = ((p.flags & kFlagPush) && !nopush) ? 1u : 0u;
    }
    // Early PDL trigger (push mode only).  The next call on this stream may
    // run its entry (which writes only the entry slots and its own control
    // slot) as soon as every peer has consumed my record of this call -- it
    // then overlaps this call's whole reduce-scatter instead of only its
    // completion tail.  Its record lets a peer that has finished this call
    // start the next one's reduce-scatter while I am still in this one:
    //  - push mode: that peer writes only my out of the next call (stream
    //    order makes that the next call's buffer) and the ag_in slot of the
    //    next call's parity;
    //  - pull mode would let it overwrite its result region while I still
    //    pull this call's slice from it, so pull-mode calls (including the
    //    fused optimizer) keep the end-of-call trigger.
    // A peer that does not ack within 100 us just leaves the trigger to the
    // end of the call.
    __syncwarp();
    if (N > 1 && !p.emulated && !bad && p.early_trigger && s_pushok) {
      bool acked = true;
      if (j < N && j != me) {
        acked = false;
        const uint64_t ta = globaltimer_ns();
        for (uint32_t it = 0;; ++it) {
          if (ld_relaxed_sys(&hdr->ent_ack[j]) == tag) {
            acked = true;
            break;
          }
          if ((it & 15u) == 15u && globaltimer_ns() - ta > 100000ull) break;
          if (it > 4) __nanosleep(64);
        }
      }
      if (__all_sync(0xffffffffu, acked) && tid == 0) pdl_trigger();
    }
  }
  // CTAs other than 0 gate nothing the next call's entry touches
  if (blockIdx.x != 0 && tid == 0 && p.early_trigger) pdl_trigger();
  // The previous kernel on this stream (if it let us start early) has now
  // completed and its writes are visible; a no-op for ordinary launches.
  pdl_wait();
  __syncthreads();

  // ---- 1b. fan the entry result out to my CTAs ----------------------------
  if (blockIdx.x == 0) {
    if (tid == 0) {
      hdr->tph[0] = s_t0;
      if (s_status == ST_OK) {
        for (int k = 0; k < N; ++k) {
          hdr->peer_in[k] = s_pin[k];
          hdr->peer_res[k] = s_pres[k];
          hdr->peer_out[k] = s_pout[k];
        }
        const uint32_t push_ok = s_pushok;
        hdr->push_ok = push_ok;
        uint64_t orbits = reinterpret_cast<uint64_t>(p.out[me]);
        for (int k = 0; k < N; ++k) orbits |= s_pin[k] | s_pres[k];
        if (push_ok)
          for (int k = 0; k < N; ++k) orbits |= s_pout[k];
        if (p.flags & kFlagSGD)
          orbits |= reinterpret_cast<uint64_t>(p.sgd_p[me]) | reinterpret_cast<uint64_t>(p.sgd_m[me]) |
                    reinterpret_cast<uint64_t>(p.sgd_po[me]) | reinterpret_cast<uint64_t>(p.sgd_mo[me]);
        const uint32_t vec_ok = (orbits & 15u) == 0;
        hdr->vec_ok = vec_ok;
        st_release_gpu(&hdr->go, mk_flag(tag, 1));
        s_vec_ok = (int)vec_ok;
        s_push = direct && N > 1 && push_ok != 0;
      }
      hdr->tph[1] = globaltimer_ns();
      hdr->dbg_t1 = hdr->tph[1];
    }
    __syncthreads();
    if (s_status == ST_OK && tid < N) {
      s_src[tid] = reinterpret_cast<const T*>(s_pin[tid]);
      s_res[tid] = reinterpret_cast<const float*>(s_pres[tid]);
      s_out[tid] = reinterpret_cast<float*>(s_pout[tid]);
    }
  } else {
    if (tid == 0 && s_status == ST_OK) {
      const uint32_t st = wait_go(hdr, mk_flag(tag, 1), s_t0, p.hard_timeout_ns);
      if (st != ST_OK) s_status = st;
    }
    __syncthreads();
    // one L2 round trip: the 3N+1 words are read by different threads
    if (s_status == ST_OK) {
      if (tid < N) s_src[tid] = reinterpret_cast<const T*>(ld_relaxed_gpu(&hdr->peer_in[tid]));
      else if (tid < 2 * N) s_res[tid - N] = reinterpret_cast<const float*>(ld_relaxed_gpu(&hdr->peer_res[tid - N]));
      else if (tid < 3 * N) s_out[tid - 2 * N] = reinterpret_cast<float*>(ld_relaxed_gpu(&hdr->peer_out[tid - 2 * N]));
      else if (tid == 3 * N) {
        s_vec_ok = (int)ld_relaxed_sys32(&hdr->vec_ok);
        s_push = direct && N > 1 && ld_relaxed_sys32(&hdr->push_ok) != 0;
      }
    }
  }
  __syncthreads();

  if (tid == 0 && s_newer && s_status == ST_OK) {  // I am a zombie of an older ring: push nothing
    s_status = ST_PEER_RESET;
    s_blame = __ffs(s_newer) - 1;
  }
  __syncthreads();
  // ---- 2. reduce-scatter of my slice: one contiguous span per CTA --------
  uint32_t nf = 0;
  int done = 0;
  // the bulk-copy path runs when every buffer is 16-byte aligned (known only
  // after the entry records) and the call is not a fused-optimizer one
  // (the fused optimizer keeps the register path: its epilogue's extra HBM
  // traffic in the consumers made the bulk path slower, config 5 at N=4:
  // 14.0 vs 10.2 ms per 2 GB step)
  const bool tma = p.tma_stages != 0 && s_vec_ok != 0 && (p.flags & kFlagSGD) == 0 && (p.diag == 0 || p.diag >= 3);
  uint32_t gseq = 0;  // thread 0: stage-ring sequence number (mbarrier phases) across RS and AG
  if (s_status == ST_OK) {
    const bool vec_ok = s_vec_ok != 0;
    const bool do_scale = (p.flags & FTAR_F_SCALE) != 0;
    const int max_tiles = (p.fault_member == me) ? p.fault_after_tiles : 0x7fffffff;
    float* const res = const_cast<float*>(s_res[me]) - lo;  // indexed by global element
    if (tma) {
      if (s_push)
        done = fold_tiles_tma<N, In>(p, s_src, me, SinkPush<N>{s_out}, lo, hi, do_scale, nf, ctl, max_tiles, dsmem);
      else if (direct && res != p.out[me])
        done = fold_tiles_tma<N, In>(p, s_src, me, SinkTwo{res, p.out[me]}, lo, hi, do_scale, nf, ctl, max_tiles, dsmem);
      else
        done = fold_tiles_tma<N, In>(p, s_src, me, SinkOne{res}, lo, hi, do_scale, nf, ctl, max_tiles, dsmem);
      gseq = done > 0 ? (uint32_t)done : 0u;
#ifdef FTAR_DIAGNOSTICS
      // timing diagnostics that change results (the diagnostic library
      // variant only, built by _build.build(diag=True); never the product)
    } else if (p.diag == 1) {
      done = fold_tiles<N, In>(p, s_src, SinkNone{res}, lo, hi, vec_ok, do_scale, nf, ctl, max_tiles);
    } else if (p.diag == 2) {
      __shared__ const T* s_loc[N];
      if (tid < N) s_loc[tid] = s_src[me];
      __syncthreads();
      done = fold_tiles<N, In>(p, s_loc, SinkOne{res}, lo, hi, vec_ok, do_scale, nf, ctl, max_tiles);
#endif
    } else if (p.flags & kFlagSGD) {
      done = fold_tiles<N, In>(p, s_src,
                               SinkSGD{res, direct ? p.out[me] : nullptr, SgdRefs{p.sgd_p[me], p.sgd_m[me], p.sgd_po[me], p.sgd_mo[me]},
                                       p.sgd_lr, p.sgd_beta},
                               lo, hi, vec_ok, do_scale, nf, ctl, max_tiles);
    } else if (s_push) {
      done = fold_tiles<N, In>(p, s_src, SinkPush<N>{s_out}, lo, hi, vec_ok, do_scale, nf, ctl, max_tiles);
    } else if (direct && res != p.out[me]) {
      done = fold_tiles<N, In>(p, s_src, SinkTwo{res, p.out[me]}, lo, hi, vec_ok, do_scale, nf, ctl, max_tiles);
    } else {
      done = fold_tiles<N, In>(p, s_src, SinkOne{res}, lo, hi, vec_ok, do_scale, nf, ctl, max_tiles);
    }
    if (done < 0 && tid == 0) s_status = ST_INJECTED;
  }
  if (tid == 0 && blockIdx.x < 256) hdr->dbg_rs_end[blockIdx.x] = globaltimer_ns();
  if (__any_sync(0xffffffffu, nf != 0) && (tid & 31) == 0) atomicOr(&s_nf, 1u);
  __syncthreads();
  if (tid == 0) {
    const uint32_t st = s_status;
    if (st == ST_OK && s_nf) atomicOr(&hdr->nonfinite, 1u);
    if (st != ST_OK && st != ST_FOLLOW) {
      atomicMax(&hdr->err, severity_code(st));
      hdr->err_peer = s_blame;
      if (st != ST_INJECTED) st_release_sys(&hdr->poison, mk_flag(tag, st));
    }
    if (done > 0) atomicAdd(reinterpret_cast<unsigned long long*>(&hdr->tiles_done), (unsigned long long)done);
    // arrival: gpu-scope release (the CTA's writes, ordered by the bar.sync
    // above, before the counter); the last CTA then publishes with ONE
    // sys-scope fence + release store, which is cumulative over everything
    // the counter chain made it observe.  Per-CTA sys fences cost ~100 us.
    if (gridDim.x > 1) __threadfence();  // my CTA's writes before the arrival counter
    const uint32_t old = gridDim.x > 1 ? atomicAdd(&hdr->rs_arrive, 1u) : 0u;
    if (old == gridDim.x - 1) {
      // ONE sys-scope acq_rel fence: acquires the other CTAs' writes through
      // the counter and releases everything before the relaxed flag stores
      hdr->dbg_fence[0] = globaltimer_ns();
      fence_acq_rel_sys();
      hdr->dbg_fence[1] = globaltimer_ns();
      if (ld_relaxed_sys32(&hdr->err) == 0) {
        const uint32_t bits = ld_relaxed_sys32(&hdr->nonfinite) ? kBitNonFinite : 0u;
        st_relaxed_sys(&hdr->rs_done, mk_flag(tag, bits));
        if (s_push) {
          // my whole slice is in every peer's out: tell them (the fence above
          // made all my CTAs' posted writes visible first)
          for (int j = 0; j < N; ++j) {
            if (j == me) continue;
            ArenaHdr* ph = reinterpret_cast<ArenaHdr*>(p.base[j]);
            st_relaxed_sys(&ph->ag_in[tag & 1][me], mk_flag(tag, bits));
          }
        }
        hdr->tph[2] = globaltimer_ns();
      }
      ctl->progress = hdr->tiles_done;
    }
  }

  // ---- 3. reduce-scatter -> all-gather barrier (CTA 0 polls, fans out) ---
  // In-place calls: a full barrier (nothing is committed unless every slice
  // is reduced and finite).  Out-of-place (direct) calls: `out` is scratch
  // until success, so CTA 0 publishes members one by one (go2 mask) and each
  // CTA pulls a slice as soon as its owner is done.
  if (s_push) {
    // push mode: peers wrote their slices into my out; CTA 0 waits for
    // every peer's ag_in flag (local polls; their poison words remote)
    if (blockIdx.x == 0 && tid == 0 && s_status == ST_OK) {
      uint32_t bits = ld_relaxed_sys32(&hdr->nonfinite) ? kBitNonFinite : 0u;
      for (int jj = 1; jj < N; ++jj) {
        const int j = (me + jj) % N;
        ArenaHdr* ph = reinterpret_cast<ArenaHdr*>(p.base[j]);
        uint32_t b = 0;
        const uint32_t st = wait_flag(&hdr->ag_in[tag & 1][j], tag, &ph->poison, ctl, &hdr->err, s_t0,
                                      p.hard_timeout_ns, &b);
        if (st != ST_OK) {
          s_status = st;
          s_blame = j;
          break;
        }
        bits |= b;
      }
      hdr->tph[3] = globaltimer_ns();
      if (s_status == ST_OK && (bits & kBitNonFinite)) s_status = ST_NUMERICAL;
    }
    __syncthreads();
  } else if (!direct) {
    if (tid == 0 && s_status == ST_OK) {
      if (blockIdx.x == 0) {
        uint32_t bits = 0;
        for (int jj = 0; jj < N; ++jj) {
          const int j = (me + jj) % N;
          ArenaHdr* ph = reinterpret_cast<ArenaHdr*>(p.base[j]);
          uint32_t b = 0;
          uint32_t st = wait_flag(&ph->rs_done, tag, j == me ? nullptr : &ph->poison, ctl,
                                  &hdr->err, s_t0, p.hard_timeout_ns, &b);
          if (st != ST_OK) {
            s_status = st;
            s_blame = j;
            break;
          }
          bits |= b;
        }
        if (s_status == ST_OK) {
          hdr->peer_bits = bits;
          st_release_gpu(&hdr->go, mk_flag(tag, 2));
        }
        hdr->tph[3] = globaltimer_ns();
      } else {
        const uint32_t st = wait_go(hdr, mk_flag(tag, 2), s_t0, p.hard_timeout_ns);
        if (st != ST_OK) s_status = st;
      }
      if (s_status == ST_OK && (ld_relaxed_sys32(&hdr->peer_bits) & kBitNonFinite)) s_status = ST_NUMERICAL;
    }
    __syncthreads();
  } else if (blockIdx.x == 0) {
    if (tid == 0 && s_status == ST_OK) {
      uint32_t bits = 0, mask = 0;
      for (int jj = 1; jj <= N; ++jj) {  // peers first, my own slice (already in out) last
        const int j = (me + jj) % N;
        ArenaHdr* ph = reinterpret_cast<ArenaHdr*>(p.base[j]);
        uint32_t b = 0;
        uint32_t st = wait_flag(&ph->rs_done, tag, j == me ? nullptr : &ph->poison, ctl,
                                &hdr->err, s_t0, p.hard_timeout_ns, &b);
        if (st != ST_OK) {
          s_status = st;
          s_blame = j;
          break;
        }
        bits |= b;
        mask |= 1u << j;
        st_release_gpu(&hdr->go2, mk_flag(tag, mask));
      }
      hdr->tph[3] = globaltimer_ns();
      if (s_status == ST_OK && (bits & kBitNonFinite)) s_status = ST_NUMERICAL;
    }
    __syncthreads();
  }

  // ---- 4. all-gather pull (commit) ---------------------------------------
  if (!s_push && (s_status == ST_OK || (direct && s_status == ST_NUMERICAL))) {
    float* const out = p.out[me];
    const bool vec_ok = s_vec_ok != 0;
    // every CTA starts on a different peer so all links stay busy
    for (int i = 0; i < N; ++i) {
      const int k = (int)((me + 1 + blockIdx.x + i) % N);
      if ((direct || (p.flags & kFlagSGD)) && k == me) continue;  // done during the reduce-scatter
      if (direct && blockIdx.x != 0) {
        if (tid == 0) {
          const uint32_t st = wait_go_bit(hdr, tag, k, s_t0, p.hard_timeout_ns);
          if (st != ST_OK) s_status = st;
        }
        __syncthreads();
        if (s_status != ST_OK) break;
      }
      uint64_t klo, khi;
      slice_of(p, k, E, klo, khi);
      if (klo >= khi) continue;
      if (p.flags & kFlagSGD)
        pull_sgd<8>(direct ? out + klo : nullptr, s_res[k], SgdRefs{p.sgd_p[me], p.sgd_m[me], p.sgd_po[me], p.sgd_mo[me]}.at(klo),
                    khi - klo, vec_ok, p.sgd_lr, p.sgd_beta);
      else if (tma)
        tma_copy_span(out + klo, s_res[k], khi - klo, dsmem, p.tma_stages,
                      (uint32_t)tma_stage_bytes(N, In::kBytes), gseq);
      else
        copy_f32<8>(out + klo, s_res[k], khi - klo, vec_ok);
    }
    if (tma && tid == 0) bulk_wait<0>();  // my out is complete before the arrival below
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < 256) hdr->dbg_ag_end[blockIdx.x] = globaltimer_ns();

  // ---- 5. completion -----------------------------------------------------
  if (tid == 0) {
    // this CTA is done with every data buffer of the call (push mode: CTA 0
    // only gets here once all peers' slices are in my out), so the next call
    // on the stream may start its entry while the tail below drains
    pdl_trigger();
    const uint32_t st = s_status;
    if (st != ST_OK && st != ST_FOLLOW) {
      atomicMax(&hdr->err, severity_code(st));
      hdr->err_peer = s_blame;
      if (st != ST_INJECTED && st != ST_NUMERICAL) st_release_sys(&hdr->poison, mk_flag(tag, st));
    }
    if (gridDim.x > 1) __threadfence();
    const uint32_t old = gridDim.x > 1 ? atomicAdd(&hdr->done_arrive, 1u) : 0u;
    if (old == gridDim.x - 1) {
      // Only my own CTAs write err/nonfinite/tiles: a gpu-scope acquire through
      // the arrival counter suffices.  Nothing published here is read by a
      // peer, and the outputs reach stream-ordered consumers at kernel
      // completion, so the success path needs no sys fence (~1.5 us each);
      // `detail` is only read after a failed `done`, so only errors fence it.
      hdr->dbg_fence[2] = globaltimer_ns();
      fence_acq_rel_gpu();
      hdr->dbg_fence[3] = globaltimer_ns();
      const uint32_t err = ld_relaxed_gpu32(&hdr->err);
      const uint64_t tiles = hdr->tiles_done;
      const int64_t blame = hdr->err_peer;
      (void)tiles;
      // the phase stamps stay in device memory (ftar_phase_times reads them);
      // `done` is the tail's only PCIe write: griddepcontrol.wait in the next
      // call waits for this grid's writes to flush, host-memory ones included
      hdr->tph[4] = globaltimer_ns();
      hdr->rs_arrive = 0;
      hdr->done_arrive = 0;
      hdr->nonfinite = 0;
      hdr->err = 0;
      hdr->err_peer = -1;
      hdr->tiles_done = 0;
      if (err) {
        ctl->detail = blame;
        __threadfence_system();
      }
      ctl->done = mk_flag(tag, err & 0xffu);
    }
  }
}


// ---------------------------------------------------------------- small buckets
// Push one-shot (input <= kSmallMax bytes): every member posts its whole
// input into every peer's receive slot [generation parity][seq parity][sender]
// and raises sm_in[sender] (with a call fingerprint in sm_meta); then waits for
// the N-1 peers' flags and folds all N copies LOCALLY in the reference order
// into the result region, committing to `out` only if every sum is finite.
// One flag wait per call instead of entry + reduce-scatter barriers; nobody
// ever reads a peer's memory, and the seq-parity double buffer makes the
// receive slots safe to reuse without an entry barrier (a member cannot start
// call c+2 before every member finished call c+1, hence consumed call c).
// The generation parity keeps a zombie of an abandoned generation (a member
// dropped on timeout that resumes and pushes late, with its old ring index)
// out of the slots the regrouped ring uses; after the fold every sender's
// flag and fingerprint are re-read, so a late write that did land in time is
// reported (PEER_RESET) instead of committed.

__device__ __forceinline__ uint64_t small_slot(uint64_t tag, int sender) {
  const uint64_t genp = tag_gen(tag) & 1ull, parity = tag & 1ull;
  return kRecvOff + ((genp * 2 + parity) * kMaxMembers + (uint64_t)sender) * kSmallMax;
}

template <int N, class In>
__global__ void __launch_bounds__(kThreads, 1) small_allreduce_kernel(const __grid_constant__ LaunchParams p) {
  using T = typename In::T;
  constexpr int U = Unroll<N, In>::U;
  const int me = p.emulated ? (int)blockIdx.y : p.self;
  char* const mybase = p.base[me];
  ArenaHdr* const hdr = reinterpret_cast<ArenaHdr*>(mybase);
  HostCtl* const ctl = p.ctl[me];
  const uint64_t tag = p.tag;
  const uint64_t E = p.nelems;
  const uint64_t bytes = E * (uint64_t)In::kBytes;
  const uint64_t parity = tag & 1ull;
  const int tid = threadIdx.x;
  const T* const my_in = reinterpret_cast<const T*>(reinterpret_cast<uint64_t>(mybase) + p.in_off[me]);
  __shared__ const T* s_src[N];
  __shared__ uint32_t s_status, s_nf;
  __shared__ int s_blame;
  __shared__ uint64_t s_t0;
  __shared__ uint64_t s_t1;
  __shared__ uint32_t s_newer, s_ctlbad;
#ifdef FTAR_DIAGNOSTICS
  // per-step stamps of CTA 0 (tools/small_probe.py): dbg_trace[0..9]
  uint64_t* const strace = (blockIdx.x == 0 && (p.emulated == 0 || blockIdx.y == 0)) ? hdr->dbg_trace : nullptr;
#define SMALL_STAMP(k) \
  if (strace && tid == 0) strace[k] = globaltimer_ns();
#else
#define SMALL_STAMP(k)
#endif
  SMALL_STAMP(0)
  if (tid >= 32 && tid < 64) {
    // zombie guard on warp 1 (remote reads, overlapping the previous
    // kernel's tail and warp 0's PCIe read): a member dropped from the ring
    // must not push into the regrouped one
    const uint32_t newer = p.emulated ? 0u : newer_peers(p, N, me, tag);
    if (tid == 32) s_newer = newer;
  }
  if (tid == 0) {
    s_nf = 0;
    s_t0 = globaltimer_ns();
    s_t1 = 0;
    s_ctlbad = 0;
    if (blockIdx.x == 0) {
      // Epoch fence (a PCIe read, overlapping the previous kernel's tail):
      // a stale op's pushes carry a tag no current peer call waits for, and
      // it poisons itself.
      if (ctl_mismatch(ctl, tag, N, p.contrib, !p.emulated, true)) s_ctlbad = 1;
      ctl->started = tag;
    }
  }
  __syncthreads();
  if (tid == 0) {
    s_status = s_newer ? ST_PEER_RESET : (s_ctlbad ? ST_PROTOCOL : ST_OK);
    s_blame = s_newer ? __ffs(s_newer) - 1 : (s_ctlbad ? me : -1);
  }
  SMALL_STAMP(1)
  // The input may be the output of the previous kernel on this stream (an
  // in-place chain, or an intra-replica reduce-scatter feeding this call):
  // griddepcontrol.launch_dependents does not make that kernel's writes
  // visible, so nothing reads my input before griddepcontrol.wait.
  pdl_wait();
  __syncthreads();
  SMALL_STAMP(2)
  const uint64_t fp = call_fingerprint(p, N);
  const bool contributes = (p.contrib >> me) & 1u;
  // 1. push my input to every peer (grid-stride 16-byte copies)
  if (contributes && bytes && s_status == ST_OK) {
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    const uint64_t first = (uint64_t)blockIdx.x * kThreads + tid;
    for (int jj = 1; jj < N; ++jj) {
      const int j = (me + jj) % N;
      copy_bytes_grid(p.base[j] + small_slot(tag, me), reinterpret_cast<const char*>(my_in), bytes, first, stride);
    }
  }
  __syncthreads();
  SMALL_STAMP(3)
  if (tid == 0) {
    if (gridDim.x > 1) __threadfence();
    const uint32_t old = gridDim.x > 1 ? atomicAdd(&hdr->sm_arrive[parity], 1u) : 0u;
    if (old == gridDim.x - 1) hdr->sm_arrive[parity] = 0;  // untouched until the call after next
    if (old == gridDim.x - 1 && s_status != ST_PEER_RESET) {  // (a zombie raises no flags either)
      for (int jj = 1; jj < N; ++jj)
        st_relaxed_sys(&reinterpret_cast<ArenaHdr*>(p.base[(me + jj) % N])->sm_meta[parity][me], fp);
      fence_acq_rel_sys();  // all my CTAs' posted writes (and the fingerprints) before the flags
      for (int jj = 1; jj < N; ++jj)
        st_relaxed_sys(&reinterpret_cast<ArenaHdr*>(p.base[(me + jj) % N])->sm_in[parity][me], mk_flag(tag, 0));
      s_t1 = globaltimer_ns();
    }
  }
  SMALL_STAMP(4)
  __syncthreads();
  if (tid == 0 && blockIdx.x == 0) {
    hdr->tph[0] = s_t0;
    hdr->tph[1] = s_t1 ? s_t1 : globaltimer_ns();
  }
  // 2. wait for every peer's push (each CTA's thread 0 polls local flags)
  if (tid == 0 && s_status == ST_OK) {
    for (int jj = 1; jj < N; ++jj) {
      const int j = (me + jj) % N;
      ArenaHdr* ph = reinterpret_cast<ArenaHdr*>(p.base[j]);
      uint32_t st = wait_flag(&hdr->sm_in[parity][j], tag, &ph->poison, ctl, &hdr->err, s_t0, p.hard_timeout_ns,
                              nullptr);
      if (st == ST_OK && ld_relaxed_sys(&hdr->sm_meta[parity][j]) != fp) st = ST_PROTOCOL;
      if (st != ST_OK) {
        s_status = st;
        s_blame = j;
        break;
      }
    }
    for (int j = 0; j < N; ++j)
      s_src[j] = j == me ? my_in : reinterpret_cast<const T*>(mybase + small_slot(tag, j));
    if (blockIdx.x == 0) hdr->tph[2] = globaltimer_ns();
  }
  __syncthreads();
  SMALL_STAMP(5)
  // 3. fold locally (reference order) into out directly (out-of-place calls:
  // out is undefined after an error) or into the staging region (in place)
  const bool sdirect = (p.flags & kFlagSmallDirect) != 0;
  float* const res = sdirect ? p.out[me] : reinterpret_cast<float*>(mybase + p.res_off[me]);
  uint32_t nf = 0;
  if (s_status == ST_OK) {
    uint64_t orbits = reinterpret_cast<uint64_t>(res) | reinterpret_cast<uint64_t>(p.out[me]);
    for (int j = 0; j < N; ++j) orbits |= reinterpret_cast<uint64_t>(s_src[j]);
    const bool vec_ok = (orbits & 15u) == 0;
#ifdef FTAR_DIAGNOSTICS
    if (strace && tid == 0) {
      // one dependent load of a peer-written slot and of my input
      const uint64_t t0 = globaltimer_ns();
      const float a = *(volatile const float*)s_src[(me + 1) % N];
      const uint64_t t1 = globaltimer_ns();
      const float b = *(volatile const float*)s_src[me];
      const uint64_t t2 = globaltimer_ns();
      strace[10] = t1 - t0;
      strace[11] = t2 - t1;
      strace[14] = __float_as_uint(a + b);
    }
#endif
    fold_small<N, In>(p, s_src, SinkOne{res}, E, vec_ok, (p.flags & FTAR_F_SCALE) != 0, nf);
#ifdef FTAR_DIAGNOSTICS
    if (strace && tid == 0) strace[12] = globaltimer_ns();
    if (p.diag == 5) {  // the same fold again: warm instruction cache, TLB and L2
      uint32_t nf2 = 0;
      fold_small<N, In>(p, s_src, SinkOne{res}, E, vec_ok, (p.flags & FTAR_F_SCALE) != 0, nf2);
      if (strace && tid == 0) strace[13] = globaltimer_ns();
    }
#endif
  }
  __syncthreads();
  SMALL_STAMP(6)
  if (tid < 32 && s_status == ST_OK) {
    // every copy I folded must still be the one its sender flagged for this
    // call: a zombie's late push is followed by its (older) flag (lane j
    // re-reads member j's flag and fingerprint; all peers at once)
    const int j = tid;
    const bool stale = j < N && j != me &&
                       (flag_tag(ld_relaxed_sys(&hdr->sm_in[parity][j])) != tag ||
                        ld_relaxed_sys(&hdr->sm_meta[parity][j]) != fp);
    const uint32_t bad = __ballot_sync(0xffffffffu, stale);
    if (tid == 0 && bad) {
      s_status = ST_PEER_RESET;
      s_blame = __ffs(bad) - 1;
    }
  }
  if (__any_sync(0xffffffffu, nf != 0) && (tid & 31) == 0) atomicOr(&s_nf, 1u);
  __syncthreads();
  SMALL_STAMP(7)
  if (tid == 0 && s_nf) atomicOr(&hdr->nonfinite, 1u);
  if (tid == 0 && s_status != ST_OK && s_status != ST_FOLLOW) {
    atomicMax(&hdr->err, severity_code(s_status));
    hdr->err_peer = s_blame;
    st_release_sys(&hdr->poison, mk_flag(tag, s_status));
  }
  // commit needs every CTA's fold: a grid-wide arrival, then the last CTA copies
  if (tid == 0) {
    if (gridDim.x > 1) __threadfence();
    const uint32_t old = gridDim.x > 1 ? atomicAdd(&hdr->done_arrive, 1u) : 0u;
    s_blame = (old == gridDim.x - 1) ? 1 : 0;  // reuse as "am last"
    // PDL: a CTA is done with the data buffers here, except the last one of a
    // staged (in-place) call, which still copies the sums into out - the next
    // call's input may alias that out, so it triggers after the copy
    if (!s_blame || sdirect) pdl_trigger();
  }
  __syncthreads();
  SMALL_STAMP(8)
  if (s_blame == 1) {
    if (tid == 0) fence_acq_rel_gpu();
    __syncthreads();
    uint32_t err = ld_relaxed_gpu32(&hdr->err);
    if (err == 0 && ld_relaxed_gpu32(&hdr->nonfinite)) err = severity_code(ST_NUMERICAL);
    if (err == 0 && !sdirect) {
      // copy the staged sums into out (one CTA; small buckets only)
      const bool vec = ((reinterpret_cast<uint64_t>(res) | reinterpret_cast<uint64_t>(p.out[me])) & 15u) == 0;
      float* out = p.out[me];
      if (vec) {
        const uint64_t nv = E >> 2;
        for (uint64_t v = tid; v < nv; v += kThreads)
          *reinterpret_cast<uint4*>(out + v * 4) = *reinterpret_cast<const uint4*>(res + v * 4);
        for (uint64_t e = (nv << 2) + tid; e < E; e += kThreads) out[e] = res[e];
      } else {
        for (uint64_t e = tid; e < E; e += kThreads) out[e] = res[e];
      }
    }
    __syncthreads();
    if (tid == 0 && !sdirect) pdl_trigger();
    if (tid == 0) {
      // as in allreduce_kernel: no sys fence on the success path
      const int64_t blame = hdr->err_peer;
      hdr->tph[3] = hdr->tph[2];
      hdr->tph[4] = globaltimer_ns();  // device memory only: `done` is the one PCIe write
#ifdef FTAR_DIAGNOSTICS
      hdr->dbg_trace[9] = hdr->tph[4];
#endif
      hdr->rs_arrive = 0;
      hdr->done_arrive = 0;
      hdr->nonfinite = 0;
      hdr->err = 0;
      hdr->err_peer = -1;
      if (err) {
        ctl->detail = blame;
        __threadfence_system();
      }
      ctl->done = mk_flag(tag, err & 0xffu);
    }
  }
}
#undef SMALL_STAMP

// ------------------------------------------------- intra-replica collectives
// IntraGroup.reduce_scatter / all_gather (replica.py:241-262)
// across the R GPUs of one replica (HSDP, R > 1), over NVLink peer loads.
//   RS: rank r's shard = vec_0[b_r] + vec_1[b_r] + ... + vec_{R-1}[b_r], the
//       fold running rank 0 upward on every rank (replica.py:247-249,
//       tests/test_replica.py:71-86), fp32 (bf16 inputs upcast exactly).
//   AG: full[b_k] = shard_k for every rank k (replica.py:254-262).
// Same entry protocol as allreduce_kernel (pushed, tag-bound entry records).
// A closing barrier - every peer has finished reading my input - lets the
// caller reuse its buffer on return, like the reference's second barrier wait
// (replica.py:206-208).
constexpr uint32_t kIntraRS = 1, kIntraAG = 2;

__device__ __forceinline__ uint64_t intra_fingerprint(const LaunchParams& p, int n) {
  uint64_t h = call_fingerprint(p, n) ^ ((uint64_t)p.intra_op * 0xC2B2AE3D27D4EB4Full);
  for (int k = 0; k < n; ++k) h ^= (p.seg_off[k] * 131 + p.seg_len[k] + 0x165667B19E3779F9ull) + (h << 6) + (h >> 2);
  return h;
}

template <int N, class In>
__global__ void __launch_bounds__(kThreads, 1) intra_kernel(const __grid_constant__ LaunchParams p) {
  using T = typename In::T;
  constexpr int U = Unroll<N, In>::U;
  const int me = p.emulated ? (int)blockIdx.y : p.self;
  char* const mybase = p.base[me];
  ArenaHdr* const hdr = reinterpret_cast<ArenaHdr*>(mybase);
  HostCtl* const ctl = p.ctl[me];
  const uint64_t tag = p.tag;
  const int tid = threadIdx.x;
  const bool ag = p.intra_op == kIntraAG;
  __shared__ uint64_t s_pin[N];
  __shared__ const T* s_src[N];
  __shared__ uint32_t s_status;
  __shared__ int s_blame;
  __shared__ uint64_t s_t0;

  if (tid == 0) {
    s_status = ST_OK;
    s_blame = -1;
    s_t0 = globaltimer_ns();
  }
  // ---- 1. entry: publish my record, collect every peer's (warp 0, CTA 0)
  if (blockIdx.x == 0 && tid < 32) {
    __syncwarp();
    const uint64_t fp = intra_fingerprint(p, N);
    if (tid == 0) {
      const uint64_t sum = entry_sum(tag, fp, p.in_off[me], 0, ~0ull);
      for (int jj = 1; jj < N; ++jj) {
        EntryIn* e = &reinterpret_cast<ArenaHdr*>(p.base[(me + jj) % N])->ent_in[me];
        st_relaxed_sys(&e->fp, fp);
        st_relaxed_sys(&e->in_off, p.in_off[me]);
        st_relaxed_sys(&e->res_off, 0);
        st_relaxed_sys(&e->out_off, ~0ull);
        st_relaxed_sys(&e->sum, sum);
      }
      if (N > 1) fence_acq_rel_sys();
      for (int jj = 1; jj < N; ++jj)
        st_relaxed_sys(&reinterpret_cast<ArenaHdr*>(p.base[(me + jj) % N])->ent_in[me].flag, mk_flag(tag, 0));
      if (ctl_mismatch(ctl, tag, N, p.contrib, !p.emulated, false)) {
        s_status = ST_PROTOCOL;
        s_blame = me;
      }
      ctl->started = tag;
    }
    __syncwarp();
    const int j = tid;
    uint32_t st = ST_OK;
    if (s_status == ST_OK && j < N) {
      if (j == me) {
        s_pin[j] = reinterpret_cast<uint64_t>(mybase) + p.in_off[me];
      } else {
        ArenaHdr* ph = reinterpret_cast<ArenaHdr*>(p.base[j]);
        EntryIn* e = &hdr->ent_in[j];
        // own_err = null: under PDL hdr->err still belongs to the previous call
        st = wait_flag(&e->flag, tag, &ph->poison, ctl, nullptr, s_t0, p.hard_timeout_ns, nullptr);
        if (st == ST_OK) {
          const uint64_t efp = ld_relaxed_sys(&e->fp), in_off = ld_relaxed_sys(&e->in_off);
          const uint64_t r0 = ld_relaxed_sys(&e->res_off), oo = ld_relaxed_sys(&e->out_off);
          const uint64_t sum = ld_relaxed_sys(&e->sum);
          if (efp != fp) st = ST_PROTOCOL;  // a different collective or different bounds
          else if (sum != entry_sum(tag, efp, in_off, r0, oo)) st = ST_PEER_RESET;
          s_pin[j] = reinterpret_cast<uint64_t>(p.base[j]) + in_off;
        }
      }
    }
    const uint32_t bad = __ballot_sync(0xffffffffu, st != ST_OK);
    const uint32_t st_first = __shfl_sync(0xffffffffu, st, bad ? __ffs(bad) - 1 : 0);
    if (tid == 0 && bad) {
      s_status = st_first;
      s_blame = __ffs(bad) - 1;
    }
  }
  // PDL: the entry above touched only the entry slots and my control slot;
  // from here on the previous kernel on this stream has completed
  pdl_wait();
  __syncthreads();
  // ---- 2. fan out to my CTAs
  if (blockIdx.x == 0) {
    if (tid == 0) {
      hdr->tph[0] = s_t0;
      if (s_status == ST_OK) {
        for (int k = 0; k < N; ++k) hdr->peer_in[k] = s_pin[k];
        st_release_gpu(&hdr->go, mk_flag(tag, 1));
      }
      hdr->tph[1] = globaltimer_ns();
    }
    __syncthreads();
    if (s_status == ST_OK && tid < N) s_src[tid] = reinterpret_cast<const T*>(s_pin[tid]);
  } else {
    if (tid == 0 && s_status == ST_OK) {
      const uint32_t st = wait_go(hdr, mk_flag(tag, 1), s_t0, p.hard_timeout_ns);
      if (st != ST_OK) s_status = st;
    }
    __syncthreads();
    if (s_status == ST_OK && tid < N) s_src[tid] = reinterpret_cast<const T*>(ld_relaxed_gpu(&hdr->peer_in[tid]));
  }
  __syncthreads();

  // ---- 3. the collective
  if (s_status == ST_OK) {
    float* const out = p.out[me];
    if (!ag) {
      const uint64_t off = p.seg_off[me], len = p.seg_len[me];
      uint64_t orbits = reinterpret_cast<uint64_t>(out - off);
      for (int k = 0; k < N; ++k) orbits |= reinterpret_cast<uint64_t>(s_src[k]);
      const bool vec_ok = (orbits & 15u) == 0;
      // one contiguous span of my shard per CTA, folded in tiles
      const uint64_t G = gridDim.x;
      const uint64_t per = ((len + G - 1) / G + 7) & ~7ull;
      const uint64_t a0 = off + umin((uint64_t)blockIdx.x * per, len);
      const uint64_t a1 = off + umin((uint64_t)blockIdx.x * per + per, len);
      const uint64_t TL = (uint64_t)kThreads * 4 * U;
      uint32_t nf = 0;
      for (uint64_t a = a0; a < a1; a += TL)
        fold_range<N, In, U, SinkOne, true>(s_src, SinkOne{out - off}, a, umin(a + TL, a1), 0, 0xffffffffu, vec_ok,
                                            false, 1.0f, nf);
    } else {
      // every CTA starts on a different rank so all links stay busy
      for (int i = 0; i < N; ++i) {
        const int k = (int)((me + 1 + blockIdx.x + i) % N);
        const float* src = reinterpret_cast<const float*>(s_src[k]);
        float* dst = out + p.seg_off[k];
        const bool vec_ok = ((reinterpret_cast<uint64_t>(src) | reinterpret_cast<uint64_t>(dst)) & 15u) == 0;
        copy_f32<8>(dst, src, p.seg_len[k], vec_ok);
      }
    }
  }
  __syncthreads();
  // ---- 4. closing barrier: I am done reading every peer's input
  if (tid == 0) {
    if (s_status != ST_OK && s_status != ST_FOLLOW) {
      atomicMax(&hdr->err, severity_code(s_status));
      hdr->err_peer = s_blame;
      st_release_sys(&hdr->poison, mk_flag(tag, s_status));
    }
    if (gridDim.x > 1) __threadfence();
    const uint32_t old = gridDim.x > 1 ? atomicAdd(&hdr->rs_arrive, 1u) : 0u;
    if (old == gridDim.x - 1) {
      fence_acq_rel_gpu();
      if (ld_relaxed_gpu32(&hdr->err) == 0) {
        // every CTA's loads have returned (their values are stored): tell the
        // peers they may let their callers reuse the buffers I read
        for (int jj = 1; jj < N; ++jj)
          st_relaxed_sys(&reinterpret_cast<ArenaHdr*>(p.base[(me + jj) % N])->ag_in[tag & 1][me], mk_flag(tag, 0));
      }
      hdr->tph[2] = globaltimer_ns();
    }
  }
  if (blockIdx.x == 0 && tid == 0 && s_status == ST_OK) {
    for (int jj = 1; jj < N; ++jj) {
      const int j = (me + jj) % N;
      const uint32_t st = wait_flag(&hdr->ag_in[tag & 1][j], tag, &reinterpret_cast<ArenaHdr*>(p.base[j])->poison, ctl,
                                    &hdr->err, s_t0, p.hard_timeout_ns, nullptr);
      if (st != ST_OK) {
        s_status = st;
        s_blame = j;
        break;
      }
    }
    hdr->tph[3] = globaltimer_ns();
  }
  __syncthreads();
  // ---- 5. completion (as allreduce_kernel: no sys fence on success)
  if (tid == 0) {
    pdl_trigger();  // done with every buffer (CTA 0: after the closing barrier)
    const uint32_t st = s_status;
    if (st != ST_OK && st != ST_FOLLOW) {
      atomicMax(&hdr->err, severity_code(st));
      hdr->err_peer = s_blame;
      st_release_sys(&hdr->poison, mk_flag(tag, st));
    }
    if (gridDim.x > 1) __threadfence();
    const uint32_t old = gridDim.x > 1 ? atomicAdd(&hdr->done_arrive, 1u) : 0u;
    if (old == gridDim.x - 1) {
      fence_acq_rel_gpu();
      const uint32_t err = ld_relaxed_gpu32(&hdr->err);
      const int64_t blame = hdr->err_peer;
      hdr->tph[4] = globaltimer_ns();  // device memory only: `done` is the one PCIe write
      hdr->rs_arrive = 0;
      hdr->done_arrive = 0;
      hdr->nonfinite = 0;
      hdr->err = 0;
      hdr->err_peer = -1;
      hdr->tiles_done = 0;
      if (err) {
        ctl->detail = blame;
        __threadfence_system();
      }
      ctl->done = mk_flag(tag, err & 0xffu);
    }
  }
}

// ---------------------------------------------------------------- operators
template <class In>
__global__ void __launch_bounds__(256) accumulate_kernel(float* __restrict__ dst,
                                                         const typename In::T* __restrict__ src,
                                                         uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride)
    dst[e] = __fadd_rn(dst[e], In::scalar(src, e));
}
template <class In>
__global__ void __launch_bounds__(256) copy_into_kernel(float* __restrict__ dst,
                                                        const typename In::T* __restrict__ src,
                                                        uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride)
    dst[e] = In::scalar(src, e);
}

// ---------------------------------------------------------------- catch-up
__global__ void snap_mark_kernel(SnapHdr* h, int64_t step, uint64_t pb, uint64_t mb, int begin) {
  if (begin) {
    h->seq = h->seq + 1;  // odd: capture in progress
    __threadfence_system();
  } else {
    h->step = step;
    h->pbytes = pb;
    h->mbytes = mb;
    __threadfence_system();
    st_release_sys(&h->seq, h->seq + 1);  // even: stable
  }
}

__global__ void __launch_bounds__(kThreads) snap_copy_kernel(char* dst, const char* p, uint64_t pb,
                                                             const char* m, uint64_t mb) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t first = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  copy_bytes_grid(dst, p, pb, first, stride);
  copy_bytes_grid(dst + pb, m, mb, first, stride);
}

// Pull a snapshot (over NVLink when the sources are peer mappings) in 1 MiB
// chunks striped across `nsrc` donors (all healthy replicas hold the same
// retention-1 snapshot, so chunk c can come from donor c % nsrc and no single
// donor's NVLink egress carries the whole catch-up).  Honours the host abort
// word, publishes progress, and validates every donor's seqlock across the
// whole pull (a re-capture mid-pull = torn = SnapshotUnavailable).
constexpr uint64_t kPullChunk = 1ull << 20;

struct PullSrcs {
  const char* arena[kMaxMembers];
  int n;
};

// The bulk-copy (TMA) form of a pull: thread 0 streams a CTA's chunks through
// kPullStages x kPullTile smem stages (donor -> shared -> my buffer), one
// continuous pipeline over all of them; ~47 GB/s per CTA against ~28 for the
// register copy (tools/tma_probe.py), so a budget of k CTAs is a bandwidth cap
// of ~47k GB/s.  Used when every region is 16-byte aligned.
constexpr uint32_t kPullTile = 32 * 1024;
constexpr uint32_t kPullStages = 6;
constexpr uint32_t kPullSmem = 1024 + kPullStages * kPullTile;

struct BulkStream {  // thread 0's pipeline state
  char* smem;
  uint64_t issued = 0, completed = 0;
  char* pend_dst[kPullStages];
  uint32_t pend_bytes[kPullStages];
  __device__ void complete_one() {
    const uint64_t t = completed++;
    const uint32_t s = (uint32_t)(t % kPullStages);
    mbar_wait(reinterpret_cast<uint64_t*>(smem) + s, (uint32_t)((t / kPullStages) & 1));
    bulk_s2g(pend_dst[s], smem + 1024 + (uint64_t)s * kPullTile, pend_bytes[s]);
    bulk_commit();
  }
  __device__ void push(char* dst, const char* src, uint32_t bytes) {
    const uint32_t s = (uint32_t)(issued % kPullStages);
    if (issued >= kPullStages) bulk_wait_read<0>();  // the store of the tile that used stage s has read it
    uint64_t* full = reinterpret_cast<uint64_t*>(smem) + s;
    mbar_expect_tx(full, bytes);
    bulk_g2s(smem + 1024 + (uint64_t)s * kPullTile, src, bytes, full);
    pend_dst[s] = dst;
    pend_bytes[s] = bytes;
    ++issued;
    if (issued - completed > kPullStages - 1) complete_one();
  }
  __device__ void copy(char* dst, const char* src, uint64_t bytes) {
    for (uint64_t o = 0; o < bytes; o += kPullTile) push(dst + o, src + o, (uint32_t)umin(kPullTile, bytes - o));
  }
  __device__ void flush() {
    while (completed < issued) complete_one();
    bulk_wait<0>();
  }
};

// Pull kernel.  Chunks are CLAIMED from lhdr->next_chunk (atomicAdd), not
// assigned by block index, so ftar_snap_pull_boost can launch a second grid
// of the same pull that takes over part of what is left: a catch-up runs at a
// small CTA budget while the step's collectives need the links, then at full
// width.  Each CTA adds the chunks it claimed to chunks_done once they have
// landed; the CTA that completes the count validates every donor's seqlock
// and publishes `done`.  (ftar_snap_pull_multi_launch resets the counters on
// the pull stream before the first grid.)
__global__ void snap_pull_reset_kernel(SnapHdr* h) {
  h->next_chunk = 0;
  h->chunks_done = 0;
  h->err = 0;
  for (int d = 0; d < kMaxMembers; ++d) {
    h->seq_min[d] = ~0ull;
    h->seq_max[d] = 0;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
snap_pull_kernel(const __grid_constant__ PullSrcs src, SnapHdr* lhdr, HostCtl* ctl, uint64_t tag, int64_t want,
                 char* dp, uint64_t pb, char* dm, uint64_t mb, int bulk) {
  __shared__ uint32_t s_st;
  __shared__ uint64_t s_c;
  extern __shared__ __align__(1024) char psmem[];
  const int tid = threadIdx.x;
  if (bulk && tid == 0) {
    for (uint32_t i = 0; i < kPullStages; ++i) mbar_init(reinterpret_cast<uint64_t*>(psmem) + i, 1);
    fence_mbar_init();
  }
  const uint64_t total = pb + mb;
  const uint64_t nchunks = (total + kPullChunk - 1) / kPullChunk;
  if (tid == 0) {
    if (blockIdx.x == 0) ctl->started = tag;
    s_st = ST_OK;
    for (int d = 0; d < src.n; ++d) {
      const SnapHdr* sh = reinterpret_cast<const SnapHdr*>(src.arena[d]);
      const uint64_t seq = ld_acquire_sys(&sh->seq);
      const int64_t step = (int64_t)ld_relaxed_sys(reinterpret_cast<const uint64_t*>(&sh->step));
      const uint64_t spb = ld_relaxed_sys(&sh->pbytes), smb = ld_relaxed_sys(&sh->mbytes);
      if ((seq & 1u) || step != want || spb != pb || smb != mb) {
        s_st = ST_UNAVAILABLE;
        ctl->available = (seq & 1u) ? -1 : step;
      }
      atomicMin(reinterpret_cast<unsigned long long*>(&lhdr->seq_min[d]), (unsigned long long)seq);
      atomicMax(reinterpret_cast<unsigned long long*>(&lhdr->seq_max[d]), (unsigned long long)seq);
    }
  }
  __syncthreads();
  uint64_t mine = 0;  // chunks this CTA claimed (thread 0)
  auto claim = [&]() -> uint64_t {  // thread 0
    if (s_st != ST_OK || ctl->abort_tag == tag || ld_relaxed_sys32(&lhdr->err) != 0) {
      if (s_st == ST_OK) s_st = ST_ABORTED;
      // take everything left so the count still completes
      const uint64_t k = atomicExch(reinterpret_cast<unsigned long long*>(&lhdr->next_chunk),
                                    (unsigned long long)nchunks);
      if (k < nchunks) mine += nchunks - k;
      return nchunks;
    }
    const uint64_t c = atomicAdd(reinterpret_cast<unsigned long long*>(&lhdr->next_chunk), 1ull);
    if (c < nchunks) ++mine;
    return c;
  };
  if (bulk) {
    if (tid == 0) {
      BulkStream bs;
      bs.smem = psmem;
      uint32_t it = 0;
      for (uint64_t c = claim(); c < nchunks; c = claim(), ++it) {
        const char* data = src.arena[c % (uint64_t)src.n] + kSnapHdrBytes;
        const uint64_t a = c * kPullChunk, b = umin(a + kPullChunk, total);
        if (a < pb) bs.copy(dp + a, data + a, umin(b, pb) - a);
        if (b > pb) {
          const uint64_t s0 = umax(a, pb);
          bs.copy(dm + (s0 - pb), data + s0, b - s0);
        }
        if ((it & 7u) == 7u) ctl->progress = ((uint64_t)blockIdx.x << 32) | it;
      }
      bs.flush();  // every copy landed (also on abort: nothing may write smem after exit)
    }
  } else {
    uint32_t it = 0;
    for (;; ++it) {
      if (tid == 0) s_c = claim();
      __syncthreads();
      const uint64_t c = s_c;
      __syncthreads();
      if (c >= nchunks) break;
      const char* data = src.arena[c % (uint64_t)src.n] + kSnapHdrBytes;
      const uint64_t a = c * kPullChunk, b = umin(a + kPullChunk, total);
      // a chunk may straddle params|momentum
      if (a < pb) copy_bytes_grid(dp + a, data + a, umin(b, pb) - a, tid, kThreads);
      if (b > pb) {
        const uint64_t s0 = umax(a, pb);
        copy_bytes_grid(dm + (s0 - pb), data + s0, b - s0, tid, kThreads);
      }
      if (tid == 0 && (it & 7u) == 7u) ctl->progress = ((uint64_t)blockIdx.x << 32) | it;
    }
  }
  __syncthreads();
  if (tid == 0) {
    for (int d = 0; d < src.n; ++d) {
      const SnapHdr* sh = reinterpret_cast<const SnapHdr*>(src.arena[d]);
      const uint64_t seq2 = ld_acquire_sys(&sh->seq);
      atomicMax(reinterpret_cast<unsigned long long*>(&lhdr->seq_max[d]), (unsigned long long)seq2);
    }
    if (s_st != ST_OK) atomicMax(&lhdr->err, s_st);
    __threadfence();  // my chunks (and my err / seq words) before the count
    const uint64_t old = mine ? atomicAdd(reinterpret_cast<unsigned long long*>(&lhdr->chunks_done),
                                          (unsigned long long)mine)
                              : nchunks + 1;
    const bool finisher = (old < nchunks && old + mine >= nchunks) || (nchunks == 0 && blockIdx.x == 0);
    if (finisher) {
      __threadfence_system();
      uint32_t err = ld_relaxed_sys32(&lhdr->err);
      for (int d = 0; d < src.n; ++d) {
        const uint64_t smin = ld_relaxed_sys(&lhdr->seq_min[d]), smax = ld_relaxed_sys(&lhdr->seq_max[d]);
        if (err == ST_OK && smin != smax) {  // this donor re-captured mid-pull: torn
          err = ST_UNAVAILABLE;
          const SnapHdr* sh = reinterpret_cast<const SnapHdr*>(src.arena[d]);
          ctl->available = (int64_t)ld_relaxed_sys(reinterpret_cast<const uint64_t*>(&sh->step));
        }
      }
      ctl->progress = total;
      __threadfence_system();
      ctl->done = mk_flag(tag, err);
    }
  }
}

// ---------------------------------------------------------------- in-process one-shot
// All members of an in-process ring live on this GPU, so no member has to
// wait for another: one cooperative grid folds every element from all member
// inputs (same reference fold order and fusions as the protocol kernel),
// stages the fp32 sums once, and — only if every sum is finite — broadcasts
// them to all member outputs.  HBM traffic: n*in + 4 (stage write) + 4 (stage
// read) + n*4 bytes per element, vs the minimum n*(in+4).
struct LocalParams {
  const void* in[kMaxMembers];
  float* out[kMaxMembers];
  HostCtl* ctl[kMaxMembers];
  float* stage;             // nullptr: direct mode (outputs never alias inputs)
  uint32_t* flags;          // [0] nonfinite
  uint32_t* arrive;         // direct mode: CTA arrival counter (no grid barrier)
  uint64_t tag[kMaxMembers];
  uint64_t nelems;
  uint64_t p_base, p_rem;
  uint64_t ebase;
  float scale;
  uint32_t flags_in;
  uint32_t contrib;
  uint32_t stages;          // local_bulk_kernel: smem pipeline stages
};

// Direct mode's completion: the last CTA to arrive publishes every member's
// status (outputs were written during the fold; no grid barrier needed).
template <int N>
__device__ __forceinline__ void local_direct_finish(const LocalParams& p, uint32_t nf_cta, uint64_t ntiles) {
  if (threadIdx.x != 0) return;
  if (nf_cta) atomicOr(p.flags, 1u);
  __threadfence();
  if (atomicAdd(p.arrive, 1u) == gridDim.x - 1) {
    fence_acq_rel_gpu();
    const bool nonfinite = ld_relaxed_gpu32(p.flags) != 0;
    *p.flags = 0;
    *p.arrive = 0;
    for (int j = 0; j < N; ++j) {
      p.ctl[j]->progress = ntiles + 1;
      if (nonfinite) p.ctl[j]->detail = -1;
    }
    if (nonfinite) __threadfence_system();
    for (int j = 0; j < N; ++j) p.ctl[j]->done = mk_flag(p.tag[j], nonfinite ? ST_NUMERICAL : ST_OK);
  }
}

template <int N, class In>
__global__ void __launch_bounds__(kThreads, 1) local_oneshot_kernel(const __grid_constant__ LocalParams p) {
  using T = typename In::T;
  constexpr int U = Unroll<N, In>::U;
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ const T* s_src[N];
  __shared__ uint32_t s_nf;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_nf = 0;
    for (int j = 0; j < N; ++j) s_src[j] = static_cast<const T*>(p.in[j]);
    if (blockIdx.x == 0)
      for (int j = 0; j < N; ++j) p.ctl[j]->started = p.tag[j];
  }
  __syncthreads();
  LaunchParams g{};
  g.p_base = p.p_base;
  g.p_rem = p.p_rem;
  g.ebase = p.ebase;
  uint64_t orbits = reinterpret_cast<uint64_t>(p.stage);
  for (int j = 0; j < N; ++j) orbits |= reinterpret_cast<uint64_t>(p.in[j]) | reinterpret_cast<uint64_t>(p.out[j]);
  const bool vec_ok = (orbits & 15u) == 0;
  const bool do_scale = (p.flags_in & FTAR_F_SCALE) != 0;
  const uint64_t E = p.nelems;
  const uint64_t TL = (uint64_t)kThreads * 8 * U;
  const uint64_t ntiles = (E + TL - 1) / TL;
  uint32_t nf = 0;
  const bool direct = p.stage == nullptr;
  const bool all = (p.contrib & ((1u << N) - 1u)) == ((1u << N) - 1u);
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t a = t * TL, b = umin(a + TL, E);
    uint64_t cur = a;
    while (cur < b) {
      int s;
      uint64_t send;
      owner_of(cur, g, N, s, send);
      const uint64_t end = umin(send, b);
      if (direct)
        all ? fold_range<N, In, U, SinkAll<N>, true>(s_src, SinkAll<N>{p.out}, cur, end, s, p.contrib, vec_ok, do_scale,
                                                       p.scale, nf)
            : fold_range<N, In, U, SinkAll<N>, false>(s_src, SinkAll<N>{p.out}, cur, end, s, p.contrib, vec_ok,
                                                        do_scale, p.scale, nf);
      else
        all ? fold_range<N, In, U, SinkOne, true>(s_src, SinkOne{p.stage}, cur, end, s, p.contrib, vec_ok, do_scale,
                                                  p.scale, nf)
            : fold_range<N, In, U, SinkOne, false>(s_src, SinkOne{p.stage}, cur, end, s, p.contrib, vec_ok, do_scale,
                                                   p.scale, nf);
      cur = end;
    }
  }
  if (__any_sync(0xffffffffu, nf != 0) && (tid & 31) == 0) atomicOr(&s_nf, 1u);
  __syncthreads();
  if (direct) {
    // Direct mode wrote every output during the fold (outputs are undefined
    // after a non-finite sum, as for out-of-place calls), so only the status
    // needs every CTA: an arrival counter instead of a grid barrier, which
    // also lets this mode launch without the cooperative-launch overhead.
    local_direct_finish<N>(p, s_nf, ntiles);
    return;
  }
  if (tid == 0 && s_nf) atomicOr(p.flags, 1u);
  grid.sync();
  const bool bad = ld_relaxed_sys32(p.flags) != 0;
  if (!bad && !direct) {
    const uint64_t stride = (uint64_t)gridDim.x * kThreads;
    const uint64_t first = (uint64_t)blockIdx.x * kThreads + tid;
    if (vec_ok) {
      const uint64_t nv = E >> 2;
      constexpr int UB = 4;
      for (uint64_t v = first; v < nv; v += stride * UB) {
        uint4 r[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const uint64_t i = v + (uint64_t)u * stride;
          if (i < nv) r[u] = ld_stream(p.stage + i * 4);
        }
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const uint64_t i = v + (uint64_t)u * stride;
            if (i < nv) st_stream(p.out[j] + i * 4, r[u]);
          }
      }
      const uint64_t tl = (nv << 2) + first;
      if (tl < E && first < 4)
        for (int j = 0; j < N; ++j) p.out[j][tl] = p.stage[tl];
    } else {
      for (uint64_t e = first; e < E; e += stride) {
        const float x = p.stage[e];
        for (int j = 0; j < N; ++j) p.out[j][e] = x;
      }
    }
  }
  grid.sync();
  if (blockIdx.x == 0 && tid == 0) {
    const uint32_t st = bad ? ST_NUMERICAL : ST_OK;
    *p.flags = 0;
    __threadfence_system();
    for (int j = 0; j < N; ++j) {
      p.ctl[j]->detail = -1;
      p.ctl[j]->progress = ntiles + 1;
      p.ctl[j]->done = mk_flag(p.tag[j], st);
    }
  }
}

// In-process one-shot, direct mode, through the bulk-copy engine.  The
// register form above alternates a burst of loads with a burst of stores, so
// HBM sees reads and writes in phases; here warp 15 keeps S-1 stages of every
// member's tile in flight (cp.async.bulk global -> shared, mbarrier
// complete_tx) while warps 0..14 fold the landed stage in the reference order
// and stream the sums to every member's output.  Tiles are grid-strided so
// all CTAs work in one compact window of each input.
__host__ __device__ constexpr uint32_t lb_vecs(int n, int in_bytes) {
  // ~32 KB per stage over all n members (>= 6 stages in 227 KB up to n = 4)
  const uint32_t per_vec = (uint32_t)n * kTmaConsumers * 4u * (uint32_t)in_bytes;
  const uint32_t v = 32768u / per_vec;
  return v < 1 ? 1u : (v > 4 ? 4u : v);
}
__host__ __device__ constexpr uint32_t lb_tile(int n, int in_bytes) {
  return kTmaConsumers * 4u * lb_vecs(n, in_bytes);
}
__host__ __device__ __forceinline__ uint64_t lb_stage_bytes(int n, int in_bytes) {
  return (uint64_t)n * lb_tile(n, in_bytes) * (uint64_t)in_bytes;
}
__host__ __device__ __forceinline__ uint32_t lb_stages_for(int n, int in_bytes) {
  const uint64_t s = (kTmaSmemMax - tma_stage_off()) / lb_stage_bytes(n, in_bytes);
  return (uint32_t)(s > kTmaMaxStages ? kTmaMaxStages : s);
}

template <int N, class In>
__device__ __forceinline__ float lb_fold_one(const char* stage, uint32_t off, int own, uint32_t contrib) {
  constexpr uint32_t TE = lb_tile(N, In::kBytes);
  float acc = 0.0f;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    int m = own + k;
    if (m >= N) m -= N;
    float x = 0.0f;
    if ((contrib >> m) & 1u) {
      const uint64_t at = (uint64_t)m * TE + off;
      if (In::kBytes == 4) x = *reinterpret_cast<const float*>(stage + at * 4);
      else x = __uint_as_float((uint32_t)*reinterpret_cast<const uint16_t*>(stage + at * 2) << 16);
    }
    acc = k == 0 ? x : __fadd_rn(acc, x);
  }
  return acc;
}

template <int N, class In>
__global__ void __launch_bounds__(kThreads, 1) local_bulk_kernel(const __grid_constant__ LocalParams p) {
  using T = typename In::T;
  using Raw = typename In::Raw;
  constexpr uint32_t V = lb_vecs(N, In::kBytes);
  constexpr uint32_t TE = lb_tile(N, In::kBytes);
  extern __shared__ __align__(1024) char smem[];
  __shared__ uint32_t s_nf;
  const int tid = threadIdx.x;
  const uint32_t S = p.stages;
  uint64_t* full = tma_full(smem);
  uint64_t* empty = tma_empty(smem);
  TmaMeta* meta = tma_meta(smem);
  if (tid == 0) {
    s_nf = 0;
    for (uint32_t s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaConsumers / 32);
    }
    fence_mbar_init();
    if (blockIdx.x == 0)
      for (int j = 0; j < N; ++j) p.ctl[j]->started = p.tag[j];
  }
  __syncthreads();
  LaunchParams g{};
  g.p_base = p.p_base;
  g.p_rem = p.p_rem;
  g.ebase = p.ebase;
  const uint32_t contrib = p.contrib & ((1u << N) - 1u);
  const bool do_scale = (p.flags_in & FTAR_F_SCALE) != 0;
  const uint64_t E = p.nelems, Ev = E & ~7ull;  // bulk part: 16-byte granules
  const uint64_t ntiles = (Ev + TE - 1) / TE;
  const uint64_t G = gridDim.x;
  const uint64_t run = blockIdx.x < ntiles ? (ntiles - blockIdx.x + G - 1) / G : 0;
  uint32_t nf = 0;
  if (tid >= (int)kTmaConsumers) {
    if (tid == kTmaProducer) {
      OwnerRun orun;
      for (uint64_t j = 0; j < run; ++j) {
        const uint32_t s = (uint32_t)(j % S);
        if (j >= S) mbar_wait(&empty[s], (uint32_t)(((j / S) - 1) & 1));
        const uint64_t a = (blockIdx.x + j * G) * TE;
        const uint32_t cnt = (uint32_t)umin(TE, Ev - a);
        if (a < orun.sbeg || a >= orun.send) {
          owner_of(a, g, N, orun.owner, orun.send);
          orun.sbeg = a;
        }
        TmaMeta m;
        m.a = a;
        m.cnt = cnt;
        m.s0 = m.s1 = orun.owner;
        m.bnd = 0xffffffffu;
        if (orun.send < a + cnt) {  // one owner change inside the tile (segments >= a tile)
          const uint64_t b = orun.send;
          owner_of(b, g, N, orun.owner, orun.send);
          orun.sbeg = b;
          m.s1 = orun.owner;
          m.bnd = (uint32_t)(b - a);
        }
        meta[s] = m;
        char* stage = smem + tma_stage_off() + (uint64_t)s * lb_stage_bytes(N, In::kBytes);
        if (contrib == 0) {
          mbar_arrive(&full[s]);
          continue;
        }
        const uint32_t bytes = cnt * (uint32_t)In::kBytes;
        mbar_expect_tx(&full[s], bytes * (uint32_t)__popc(contrib));
#pragma unroll
        for (int k = 0; k < N; ++k)
          if ((contrib >> k) & 1u)
            bulk_g2s(stage + (uint64_t)k * TE * In::kBytes, static_cast<const T*>(p.in[k]) + a, bytes, &full[s]);
      }
    }
  } else {
    for (uint64_t j = 0; j < run; ++j) {
      const uint32_t s = (uint32_t)(j % S);
      mbar_wait(&full[s], (uint32_t)((j / S) & 1));
      const TmaMeta m = meta[s];
      const char* stage = smem + tma_stage_off() + (uint64_t)s * lb_stage_bytes(N, In::kBytes);
      float acc[V][4];
#pragma unroll
      for (uint32_t v = 0; v < V; ++v) {
        const uint32_t off = (v * kTmaConsumers + (uint32_t)tid) * 4;
        acc[v][0] = acc[v][1] = acc[v][2] = acc[v][3] = 0.f;
        if (off < m.cnt) {
          if (off + 4 <= m.bnd || off >= m.bnd) {
            const int own = off >= m.bnd ? m.s1 : m.s0;
#pragma unroll
            for (int k = 0; k < N; ++k) {
              int mm = own + k;
              if (mm >= N) mm -= N;
              float x[4];
              if ((contrib >> mm) & 1u)
                In::cvt4(*reinterpret_cast<const Raw*>(stage + ((uint64_t)mm * TE + off) * In::kBytes), x);
              else
                x[0] = x[1] = x[2] = x[3] = 0.0f;
#pragma unroll
              for (int i = 0; i < 4; ++i) acc[v][i] = k == 0 ? x[i] : __fadd_rn(acc[v][i], x[i]);
            }
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              acc[v][i] = lb_fold_one<N, In>(stage, off + i, off + i >= m.bnd ? m.s1 : m.s0, contrib);
          }
        }
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[s]);
#pragma unroll
      for (uint32_t v = 0; v < V; ++v) {
        const uint32_t off = (v * kTmaConsumers + (uint32_t)tid) * 4;
        if (off < m.cnt) {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            nf |= nonfinite_bits(acc[v][i]) ? 1u : 0u;
            if (do_scale) acc[v][i] = __fmul_rn(acc[v][i], p.scale);
          }
          const uint4 r = make_uint4(__float_as_uint(acc[v][0]), __float_as_uint(acc[v][1]),
                                     __float_as_uint(acc[v][2]), __float_as_uint(acc[v][3]));
#pragma unroll
          for (int k = 0; k < N; ++k) st_stream(p.out[k] + m.a + off, r);
        }
      }
    }
    // the < 8-element ragged tail: plain loads by the last CTA's first warp
    if (Ev < E && blockIdx.x == G - 1 && tid < 32) {
      const T* srcs[N];
#pragma unroll
      for (int k = 0; k < N; ++k) srcs[k] = static_cast<const T*>(p.in[k]);
      for (uint64_t e = Ev + tid; e < E; e += 32) {
        int own;
        uint64_t send;
        owner_of(e, g, N, own, send);
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          int mm = own + k;
          if (mm >= N) mm -= N;
          const float x = ((contrib >> mm) & 1u) ? In::scalar(srcs[mm], e) : 0.0f;
          acc = k == 0 ? x : __fadd_rn(acc, x);
        }
        nf |= nonfinite_bits(acc) ? 1u : 0u;
        if (do_scale) acc = __fmul_rn(acc, p.scale);
#pragma unroll
        for (int k = 0; k < N; ++k) p.out[k][e] = acc;
      }
    }
  }
  if (__any_sync(0xffffffffu, nf != 0) && (tid & 31) == 0) atomicOr(&s_nf, 1u);
  __syncthreads();
  local_direct_finish<N>(p, s_nf, ntiles);
}

// ---------------------------------------------------------------- diagnostics
// Streaming copy used to characterise the NVLink path (pull = remote src,
// push = remote dst) at a given CTA count; not on the FTAR path.
__global__ void __launch_bounds__(kThreads) probe_copy_kernel(char* dst, const char* src, uint64_t bytes) {
  const uint64_t stride = (uint64_t)gridDim.x * kThreads;
  const uint64_t first = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
  copy_bytes_grid(dst, src, bytes, first, stride);
}

// Bulk-copy probe (diagnostic): the same copy moved by the TMA engine, one
// thread per CTA driving an S-stage pipeline of `tile`-byte bulk loads
// (global -> shared, mbarrier tx) and bulk stores (shared -> global), one
// contiguous span per CTA.  src or dst may be a peer address.
template <int S>
__global__ void __launch_bounds__(32, 1) probe_bulk_kernel(char* dst, const char* src, uint64_t bytes,
                                                           uint32_t tile) {
  extern __shared__ __align__(1024) char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  char* buf = smem + 1024;
  if (threadIdx.x != 0) return;
  const uint64_t ntiles = bytes / tile;
  const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = umin((uint64_t)blockIdx.x * per, ntiles), t1 = umin(t0 + per, ntiles);
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  fence_mbar_init();
  const uint64_t cnt = t1 - t0;
  constexpr uint64_t L = S - 1;  // loads lead stores by S-1 tiles
  for (uint64_t j = 0; j < cnt + L; ++j) {
    if (j < cnt) {
      const int s = (int)(j % S);
      if (j >= S) bulk_wait_read<0>();  // the store of tile j-S has read slot s
      mbar_expect_tx(&full[s], tile);
      bulk_g2s(buf + (uint64_t)s * tile, src + (t0 + j) * tile, tile, &full[s]);
    }
    if (j >= L) {
      const uint64_t t = j - L;
      const int s = (int)(t % S);
      mbar_wait(&full[s], (uint32_t)((t / S) & 1));
      bulk_s2g(dst + (t0 + t) * tile, buf + (uint64_t)s * tile, tile);
      bulk_commit();
    }
  }
  bulk_wait<0>();
}

// Access-pattern probe (diagnostic): elements are fp32; a = local, b = remote.
//  mode 0: c[i] = a[i] + b[i]    (reduce-scatter-like, N = 2)
//  mode 1: c[i] = b[i]           (all-gather-like)
//  mode 2: s += a[i] + b[i], no store (loads only)
//  mode 3: c[i] = a[i] + a2[i]   (all local)
// layout 0: grid-stride 16-byte vectors; layout 1: contiguous span per CTA.
// `unroll` vectors per thread in flight per source.
template <int UNR>
__global__ void __launch_bounds__(kThreads, 1) probe_pattern_kernel(float* c, const float* a, const float* b,
                                                                    uint64_t n, int mode, int layout) {
  const uint64_t nv = n >> 2;
  uint64_t first, stride, end;
  if (layout == 0) {
    first = (uint64_t)blockIdx.x * kThreads + threadIdx.x;
    stride = (uint64_t)gridDim.x * kThreads;
    end = nv;
  } else {
    const uint64_t per = (nv + gridDim.x - 1) / gridDim.x;
    const uint64_t lo = umin((uint64_t)blockIdx.x * per, nv);
    first = lo + threadIdx.x;
    stride = kThreads;
    end = umin(lo + per, nv);
  }
  float acc = 0.f;
  for (uint64_t v = first; v < end; v += stride * UNR) {
    uint4 ra[UNR], rb[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t i = v + (uint64_t)u * stride;
      const uint64_t ii = i < end ? i : first;
      ra[u] = ld_stream(a + ii * 4);
      rb[u] = ld_stream((mode == 3 ? a + (nv - 1 - ii) * 4 : b + ii * 4));
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const uint64_t i = v + (uint64_t)u * stride;
      if (i < end) {
        uint4 r = rb[u];
        if (mode != 1) {
          r.x = __float_as_uint(__uint_as_float(ra[u].x) + __uint_as_float(rb[u].x));
          r.y = __float_as_uint(__uint_as_float(ra[u].y) + __uint_as_float(rb[u].y));
          r.z = __float_as_uint(__uint_as_float(ra[u].z) + __uint_as_float(rb[u].z));
          r.w = __float_as_uint(__uint_as_float(ra[u].w) + __uint_as_float(rb[u].w));
        }
        if (mode == 2) acc += __uint_as_float(r.x);
        else *reinterpret_cast<uint4*>(c + i * 4) = r;
      }
    }
  }
  if (mode == 2 && acc == 123456.f) c[0] = acc;
}

// Fence-cost probe (diagnostic): c = a + b with remote b, load flavour LK
// (0 L1::no_allocate, 1 default ld.global, 2 ld.global.nc), then per-CTA
// stamps: [0] loop end (warp 0), [1] after bar.sync, [2] after gpu fence,
// [3] after sys fence.
template <int LK>
__device__ __forceinline__ uint4 ld_kind(const float* p) {
  if (LK == 0) return ld_stream(p);
  if (LK == 1) return *reinterpret_cast<const uint4*>(p);
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
template <int LK>
__global__ void __launch_bounds__(kThreads, 1) probe_fence_kernel(float* c, const float* a, const float* b,
                                                                  uint64_t n, uint64_t* stamps) {
  const uint64_t nv = n >> 2;
  const uint64_t per = (nv + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = umin((uint64_t)blockIdx.x * per, nv), hi = umin(lo + per, nv);
  constexpr int U = 8;
  for (uint64_t v = lo + threadIdx.x; v < hi; v += (uint64_t)kThreads * U) {
    uint4 ra[U], rb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = v + (uint64_t)u * kThreads;
      const uint64_t ii = i < hi ? i : lo;
      ra[u] = ld_kind<LK>(a + ii * 4);
      rb[u] = ld_kind<LK>(b + ii * 4);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = v + (uint64_t)u * kThreads;
      if (i < hi) {
        uint4 r;
        r.x = __float_as_uint(__uint_as_float(ra[u].x) + __uint_as_float(rb[u].x));
        r.y = __float_as_uint(__uint_as_float(ra[u].y) + __uint_as_float(rb[u].y));
        r.z = __float_as_uint(__uint_as_float(ra[u].z) + __uint_as_float(rb[u].z));
        r.w = __float_as_uint(__uint_as_float(ra[u].w) + __uint_as_float(rb[u].w));
        *reinterpret_cast<uint4*>(c + i * 4) = r;
      }
    }
  }
  uint64_t* st = stamps + blockIdx.x * 4;
  if (threadIdx.x == 0) st[0] = globaltimer_ns();
  __syncthreads();
  if (threadIdx.x == 0) {
    st[1] = globaltimer_ns();
    __threadfence();
    st[2] = globaltimer_ns();
    __threadfence_system();
    st[3] = globaltimer_ns();
  }
}

__global__ void snap_init_kernel(SnapHdr* h) {
  h->seq = 0;
  h->step = -1;
  h->pbytes = h->mbytes = 0;
  for (int d = 0; d < kMaxMembers; ++d) {
    h->seq_min[d] = ~0ull;
    h->seq_max[d] = 0;
  }
  h->done_arrive = 0;
  h->err = 0;
  h->bytes_done = 0;
}

}  // namespace

// ============================================================================
// host runtime (C-ABI)
// ============================================================================

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return FTAR_ST_CUDA;
}
#define CK(call)                                  \
  do {                                            \
    cudaError_t _e = (call);                      \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

constexpr int kMaxSlots = 256;
constexpr int kQueue = 4;

int g_ctas = 0;         // real-mode CTAs per member (0 = default)
int g_local_ctas = 0;   // in-process ring CTAs per member (0 = default)

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
// Launch shape (tuned on 2x/4x B200, tools/tune_allreduce.py + bench.py):
// pull mode 64 CTAs that all reduce; push mode 128 CTAs.
int real_ctas(bool push = false) {
  if (g_ctas > 0) return g_ctas;
  return push ? env_int("FTAR_CTAS_PUSH", 128) : env_int("FTAR_CTAS", 64);
}
int rs_ctas_knob() { return env_int("FTAR_RS_CTAS", 0); }
// buckets up to this many input bytes take the single-barrier push one-shot
uint64_t small_bytes() {
  const int v = env_int("FTAR_SMALL_BYTES", 1 << 20);
  return std::min<uint64_t>(v < 0 ? 0 : (uint64_t)v, kSmallMax);
}
// programmatic dependent launch of the two-shot kernel (FTAR_PDL=0 disables)
bool pdl_on() { return env_int("FTAR_PDL", 1) != 0; }
// bulk-copy (TMA) data path for the two-shot kernel (FTAR_TMA=0 disables)
bool tma_on() { return env_int("FTAR_TMA", 1) != 0; }
// ... for slices of at least this many input bytes (tools/tune_tma.py, N=4:
// the register path wins at <= 4 MiB slices, the bulk path from 16 MiB)
uint64_t tma_min_slice() { return (uint64_t)env_int("FTAR_TMA_MIN_SLICE_MIB", 16) << 20; }
// CTAs of the bulk-copy path: ~128 KB of my slice per CTA, at most
// FTAR_CTAS_TMA (default 48 from N=3, a third of the SMs: N=4 f32 busbw
// 597 / 661 / 680 GB/s at 64 MiB / 256 MiB / 1 GiB; 16 CTAs already give 648
// at 256 MiB.  At N=2 each stage holds a single peer's tile and 96 CTAs are
// needed: 652 -> 666 GB/s f32 and 436 -> 453 bf16 at 256 MiB, 128 no better;
// tools/tune_tma.py, profiles/r02/tune/ctas_n2.jsonl)
int tma_ctas(int n, uint64_t slice_bytes) {
  const int cap = g_ctas > 0 ? g_ctas : env_int("FTAR_CTAS_TMA", n <= 2 ? 96 : 48);
  const uint64_t per = (uint64_t)env_int("FTAR_TMA_BYTES_PER_CTA", 128 << 10);
  return (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)std::max(cap, 1), (slice_bytes + per - 1) / per));
}
// CTAs of the small one-shot: ~20 KB of the bucket each, at most 48 (N=4,
// 1 MiB f32: 21.7 us per call at 16 CTAs, 19.3 at 48; bf16 24.5 -> 20.9;
// tools/tune_tma.py --mib 1, profiles/r02/tune/small_ctas_n4.jsonl)
int small_ctas(uint64_t bytes) {
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(48, (bytes + 20479) / 20480));
}

// The data path and grid of one call (launch_real and ftar_inflight_bound
// share it, so the in-flight meter reports the path the call really takes).
enum PathKind { kPathNone = 0, kPathSmall = 1, kPathBulk = 2, kPathRegister = 3 };
struct PathChoice {
  int kind;
  int ctas;
  uint32_t stages;  // bulk-copy pipeline stages (0: not the bulk path)
};
PathChoice choose_path(int n, const LaunchParams& p, uint64_t esz, bool small, bool sgd, bool push) {
  // the fused optimizer's all-gather also streams params + momentum through
  // HBM: 128 CTAs (tools/sgd_bench.py, N=4, 128 Mi bf16 elements per bucket:
  // 1.19 ms at 64 CTAs, 1.04 at 128, 1.11 at 148; the plain all-reduce 0.89)
  const int sgd_ctas = g_ctas > 0 ? g_ctas : env_int("FTAR_CTAS_SGD", 128);
  PathChoice pc{kPathRegister, sgd ? sgd_ctas : real_ctas(push), 0};
  // fewer CTAs for small slices (CTA arrival + fences dominate): ~64 KB of
  // my slice per CTA, at least 1, at most the tuned shape
  const uint64_t per = (uint64_t)env_int("FTAR_BYTES_PER_CTA", 64 << 10);
  const uint64_t want = (p.slice * esz + per - 1) / per;
  if (g_ctas <= 0 && want < (uint64_t)pc.ctas) pc.ctas = (int)std::max<uint64_t>(1, want);
  if (small) {
    pc.kind = kPathSmall;
    pc.ctas = g_ctas > 0 ? g_ctas : small_ctas(p.nelems * esz);
  } else if (!sgd && n >= 2 && tma_on() && p.p_base / (uint64_t)n >= tma_tile(n, (int)esz) &&
             (p.slice * esz >= tma_min_slice() || g_ctas > 0)) {
    // every segment spans >= one tile and the slice is large: the bulk-copy data path
    pc.kind = kPathBulk;
    pc.stages = tma_stages_for(n, (int)esz);
    pc.ctas = tma_ctas(n, p.slice * esz);
  }
  return pc;
}
int rs_layout() { return env_int("FTAR_RS_LAYOUT", 0); }
#ifdef FTAR_DIAGNOSTICS
int diag_mode() { return env_int("FTAR_DIAG", 0); }
#else
int diag_mode() { return 0; }  // the product library has no result-changing diagnostics
#endif

// Host wait policy: pure spinning (pause) for the first 50 ms of a wait —
// sleep_for() of a few us really sleeps ~50 us (timer slack), which would add
// that much to every collective — then yield, then 100 us sleeps.
inline void host_backoff(uint64_t it, double waited_s) {
  if (waited_s < 0.05) {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
  } else if (waited_s < 0.5) {
    std::this_thread::yield();
  } else {
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
  (void)it;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

struct ftar_ctx {
  int device = 0;
  bool exportable = false;
  char* arena = nullptr;
  uint64_t arena_bytes = 0;
  uint64_t max_bucket_bytes = 0;
  uint64_t res_off = 0, stage_off[2] = {0, 0}, pool_off = 0, pool_bytes = 0;
  // control blocks: a FIFO of kQueue slots, one per queued collective, so a
  // caller can enqueue several buckets before waiting (the GPU then runs
  // them back to back); ctl_h/ctl_d point at the most recently launched one
  HostCtl* ctl_hs = nullptr;
  HostCtl* ctl_ds = nullptr;
  HostCtl* ctl_h = nullptr;
  HostCtl* ctl_d = nullptr;
  uint64_t q_tag[kQueue] = {};
  int q_head = 0, q_count = 0;
  char* peer[kMaxSlots] = {};
  cudaIpcMemHandle_t peer_handle[kMaxSlots] = {};  // what each slot maps (import refuses a different one)
  uint64_t peer_bytes[kMaxSlots] = {};
  bool peer_local[kMaxSlots] = {};  // linked in-process (no IPC handle to close)
  int ring_slots[kMaxMembers] = {};
  int n = 1, self = 0;
  uint32_t contrib = 1;
  uint64_t gen = 0, seq = 0;
  uint64_t cur_tag = 0;
  uint64_t hard_timeout_ns = 120ull * 1000000000ull;
  bool warmed = false;  // this ring size's kernels loaded (warm_ring_kernels)
  // registered buffers (RingGroup.register): mine by region id, and every
  // peer slot's as mapped here (one IPC mapping per peer allocation block)
  uint64_t my_region_ptr[kMaxRegions] = {};
  uint64_t my_region_bytes[kMaxRegions] = {};
  uint64_t peer_region_va[kMaxSlots][kMaxRegions] = {};
  struct BlockMap {
    cudaIpcMemHandle_t h;
    char* va;
    int slot;
  };
  std::vector<BlockMap> blocks;

  int find_region(const void* ptr, uint64_t bytes, uint64_t* off) const {
    const uint64_t a = reinterpret_cast<uint64_t>(ptr);
    for (int r = 0; r < kMaxRegions; ++r)
      if (my_region_bytes[r] && a >= my_region_ptr[r] && a + bytes <= my_region_ptr[r] + my_region_bytes[r]) {
        *off = a - my_region_ptr[r];
        return r;
      }
    return -1;
  }
  void drop_slot_regions(int slot) {
    for (size_t i = 0; i < blocks.size();) {
      if (blocks[i].slot == slot) {
        cudaIpcCloseMemHandle(blocks[i].va);
        blocks.erase(blocks.begin() + (long)i);
      } else {
        ++i;
      }
    }
    for (int r = 0; r < kMaxRegions; ++r) peer_region_va[slot][r] = 0;
  }

  // enqueue a collective with `tag`; returns its control block or nullptr when full
  HostCtl* push(uint64_t tag) {
    if (q_count == kQueue) return nullptr;
    const int slot = (q_head + q_count) % kQueue;
    HostCtl* h = ctl_hs + slot;
    h->abort_tag = 0;
    h->started = 0;
    h->progress = 0;
    h->done = 0;
    h->detail = -1;
    h->available = -1;
    h->epoch = gen;
    q_tag[slot] = tag;
    ++q_count;
    ctl_h = h;
    ctl_d = ctl_ds + slot;
    cur_tag = tag;
    return h;
  }
  void pop_last() {  // undo a push whose launch failed
    --q_count;
  }
  bool all_done() const {
    for (int i = 0; i < q_count; ++i) {
      const int slot = (q_head + i) % kQueue;
      if (flag_tag(ctl_hs[slot].done) != q_tag[slot]) return false;
    }
    return true;
  }
};

struct PullArgs {
  PullSrcs src;
  int64_t want;
  char* dp;
  uint64_t pb;
  char* dm;
  uint64_t mb;
  int bulk;
};

struct ftar_snap {
  int device = 0;
  char* arena = nullptr;
  uint64_t cap = 0;
  HostCtl* ctl_h = nullptr;
  HostCtl* ctl_d = nullptr;
  PullArgs last{};  // the pull in flight (ftar_snap_pull_boost relaunches it)
  cudaEvent_t reset_done = nullptr;  // the pull's counters are reset (a boost grid waits for it)
  char* peer[kMaxSlots] = {};
  cudaIpcMemHandle_t peer_handle[kMaxSlots] = {};
  uint64_t seq = 0;
  uint64_t cur_tag = 0;
  bool inflight = false;
};

namespace {

template <int N, class In>
cudaError_t launch_n(const LaunchParams& p, dim3 grid, cudaStream_t st, bool coop, bool pdl) {
  auto fn = allreduce_kernel<N, In>;
  size_t dyn = 0;
  if (p.tma_stages) {
    dyn = (size_t)tma_smem_bytes(N, In::kBytes, p.tma_stages);
    static bool attr_set[64] = {};  // per template instance and device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmemMax);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
  }
  if (coop) {
    void* args[] = {const_cast<LaunchParams*>(&p)};
    return cudaLaunchCooperativeKernel((const void*)fn, grid, dim3(kThreads), args, dyn, st);
  }
  if (pdl) {
    // programmatic dependent launch: when the previous kernel on the stream
    // is one of ours, this call's entry overlaps that kernel's tail
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = dyn;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, p);
  }
  fn<<<grid, kThreads, dyn, st>>>(p);
  return cudaGetLastError();
}

template <int N, class In>
cudaError_t launch_small_n(const LaunchParams& p, dim3 grid, cudaStream_t st, bool coop, bool pdl) {
  auto fn = small_allreduce_kernel<N, In>;
  if (coop) {
    void* args[] = {const_cast<LaunchParams*>(&p)};
    return cudaLaunchCooperativeKernel((const void*)fn, grid, dim3(kThreads), args, 0, st);
  }
  if (pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, p);
  }
  fn<<<grid, kThreads, 0, st>>>(p);
  return cudaGetLastError();
}

template <int N, class In>
cudaError_t launch_intra_n(const LaunchParams& p, dim3 grid, cudaStream_t st, bool coop, bool pdl) {
  auto fn = intra_kernel<N, In>;
  if (coop) {
    void* args[] = {const_cast<LaunchParams*>(&p)};
    return cudaLaunchCooperativeKernel((const void*)fn, grid, dim3(kThreads), args, 0, st);
  }
  if (pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kThreads);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, p);
  }
  fn<<<grid, kThreads, 0, st>>>(p);
  return cudaGetLastError();
}

template <class In>
cudaError_t launch_intra(int n, const LaunchParams& p, dim3 grid, cudaStream_t st, bool coop, bool pdl = false) {
  switch (n) {
    case 1: return launch_intra_n<1, In>(p, grid, st, coop, pdl);
    case 2: return launch_intra_n<2, In>(p, grid, st, coop, pdl);
    case 3: return launch_intra_n<3, In>(p, grid, st, coop, pdl);
    case 4: return launch_intra_n<4, In>(p, grid, st, coop, pdl);
    case 5: return launch_intra_n<5, In>(p, grid, st, coop, pdl);
    case 6: return launch_intra_n<6, In>(p, grid, st, coop, pdl);
    case 7: return launch_intra_n<7, In>(p, grid, st, coop, pdl);
    case 8: return launch_intra_n<8, In>(p, grid, st, coop, pdl);
  }
  return cudaErrorInvalidValue;
}

template <class In>
cudaError_t launch_small(int n, const LaunchParams& p, dim3 grid, cudaStream_t st, bool coop, bool pdl = false) {
  switch (n) {
    case 2: return launch_small_n<2, In>(p, grid, st, coop, pdl);
    case 3: return launch_small_n<3, In>(p, grid, st, coop, pdl);
    case 4: return launch_small_n<4, In>(p, grid, st, coop, pdl);
    case 5: return launch_small_n<5, In>(p, grid, st, coop, pdl);
    case 6: return launch_small_n<6, In>(p, grid, st, coop, pdl);
    case 7: return launch_small_n<7, In>(p, grid, st, coop, pdl);
    case 8: return launch_small_n<8, In>(p, grid, st, coop, pdl);
  }
  return cudaErrorInvalidValue;
}

template <class In>
cudaError_t launch_dispatch(int n, const LaunchParams& p, dim3 grid, cudaStream_t st, bool coop, bool pdl = false) {
  switch (n) {
    case 1: return launch_n<1, In>(p, grid, st, coop, pdl);
    case 2: return launch_n<2, In>(p, grid, st, coop, pdl);
    case 3: return launch_n<3, In>(p, grid, st, coop, pdl);
    case 4: return launch_n<4, In>(p, grid, st, coop, pdl);
    case 5: return launch_n<5, In>(p, grid, st, coop, pdl);
    case 6: return launch_n<6, In>(p, grid, st, coop, pdl);
    case 7: return launch_n<7, In>(p, grid, st, coop, pdl);
    case 8: return launch_n<8, In>(p, grid, st, coop, pdl);
  }
  return cudaErrorInvalidValue;
}

// CUDA loads kernels lazily, at their first launch (or attribute query).
// Loading a module while other kernels run can stall the launching thread
// for milliseconds to hundreds of ms, and a collective's first launch of a
// kernel instance (a replica joining a new ring size, a recovering replica's
// first catch-up pull) is exactly when that hurts: the other members wait at
// the entry barrier.  So the instances a ring of size n will use are loaded
// when its membership is installed, and the catch-up kernels when a
// snapshot store is created.
template <class In>
void warm_ring_kernels(int n) {
  cudaFuncAttributes a;
  switch (n) {
#define CASE(K)                                                     \
  case K:                                                           \
    cudaFuncGetAttributes(&a, allreduce_kernel<K, In>);             \
    cudaFuncGetAttributes(&a, intra_kernel<K, In>);                 \
    if (K > 1) cudaFuncGetAttributes(&a, small_allreduce_kernel<(K > 1 ? K : 2), In>); \
    break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  cudaGetLastError();
}

template <class In>
int max_coop_blocks_per_sm(int n) {
  int nb = 0;
  cudaError_t e = cudaErrorInvalidValue;
  switch (n) {
#define CASE(K) case K: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, allreduce_kernel<K, In>, kThreads, 0); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  return e == cudaSuccess ? nb : 0;
}

template <class In>
cudaError_t oneshot_dispatch(int n, const LocalParams& lp, dim3 grid, cudaStream_t st) {
  void* args[] = {const_cast<LocalParams*>(&lp)};
  const void* fn = nullptr;
  switch (n) {
#define CASE(K) case K: fn = (const void*)local_oneshot_kernel<K, In>; break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
  // the staged (in-place) mode needs its grid barrier; direct mode does not
  if (lp.stage == nullptr) return cudaLaunchKernel(fn, grid, dim3(kThreads), args, 0, st);
  return cudaLaunchCooperativeKernel(fn, grid, dim3(kThreads), args, 0, st);
}

template <int N, class In>
cudaError_t local_bulk_launch_n(const LocalParams& lp, dim3 grid, cudaStream_t st) {
  auto fn = local_bulk_kernel<N, In>;
  static bool attr_set[64] = {};  // per template instance and device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTmaSmemMax);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  const size_t dyn = (size_t)(tma_stage_off() + (uint64_t)lp.stages * lb_stage_bytes(N, In::kBytes));
  fn<<<grid, kThreads, dyn, st>>>(lp);
  return cudaGetLastError();
}

template <class In>
cudaError_t local_bulk_dispatch(int n, const LocalParams& lp, dim3 grid, cudaStream_t st) {
  switch (n) {
#define CASE(K) case K: return local_bulk_launch_n<K, In>(lp, grid, st);
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default: return cudaErrorInvalidValue;
  }
}

template <class In>
int oneshot_blocks_per_sm(int n) {
  int nb = 0;
  cudaError_t e = cudaErrorInvalidValue;
  switch (n) {
#define CASE(K) case K: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, local_oneshot_kernel<K, In>, kThreads, 0); break;
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
  }
  return e == cudaSuccess ? nb : 0;
}

// Reference geometry (elements; ELEM = 4 bytes of the fp32 view), built on
// the whole bucket (`total`); this call covers [ebase, ebase + E).
void fill_geometry(LaunchParams& p, uint64_t E, uint64_t chunk_bytes, int C, int n, uint64_t ebase = 0,
                   uint64_t total = ~0ull) {
  if (total == ~0ull) total = E;
  uint64_t cap = (chunk_bytes * (uint64_t)C * (uint64_t)n) / 4;
  if (cap < 1) cap = 1;
  p.cap = cap;
  p.ebase = ebase;
  p.total = total;
  if (total == 0) {
    p.p_base = 1;
    p.p_rem = 0;
  } else {
    const uint64_t nparts = (total + cap - 1) / cap;
    p.p_base = total / nparts;
    p.p_rem = total % nparts;
  }
  const uint64_t per = (E + (uint64_t)n - 1) / (uint64_t)n;
  p.slice = (per + 7) & ~7ull;
  if (p.slice == 0) p.slice = 8;
}

uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// Workers = the contributors (every member if none): the reduce-scatter
// slices are split among them only, so a behind replica does no RS work.
void set_workers(LaunchParams& p, int n, uint64_t E) {
  const uint32_t all = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
  p.workers = (p.contrib & all) ? (p.contrib & all) : all;
  const uint64_t h = (uint64_t)__builtin_popcount(p.workers);
  const uint64_t per = (E + h - 1) / h;
  p.slice = (per + 7) & ~7ull;
  if (p.slice == 0) p.slice = 8;
}

int validate_common(int in_dtype, int n, uint64_t chunk_bytes, int max_in_flight) {
  if (in_dtype != FTAR_DT_F32 && in_dtype != FTAR_DT_BF16)
    return fail(FTAR_ST_INVARIANT, "all-reduce input must be float32 or bfloat16");
  if (n < 1 || n > kMaxMembers) return fail(FTAR_ST_INVARIANT, "ring size out of range 1..8");
  if (chunk_bytes < 4) return fail(FTAR_ST_INVARIANT, "chunk_bytes must be >= 4");
  if (max_in_flight < 1) return fail(FTAR_ST_INVARIANT, "max_in_flight must be >= 1");
  return FTAR_OK;
}

void reset_ctl(HostCtl* c) {
  c->abort_tag = 0;
  c->started = 0;
  c->progress = 0;
  c->done = 0;
  c->detail = -1;
  c->available = -1;
}

}  // namespace

extern "C" {

const char* ftar_last_error(void) { return g_err.c_str(); }
#ifdef FTAR_DIAGNOSTICS
const char* ftar_version(void) { return "ftar_b200 2.0 sm_100a DIAGNOSTIC VARIANT (FTAR_DIAG honoured)"; }
#else
const char* ftar_version(void) { return "ftar_b200 2.0 sm_100a (two-shot NVLink, TMA bulk-copy reduce-scatter, fp32 fold)"; }
#endif

int ftar_set_tuning(int ctas, int local_ctas) {
  g_ctas = ctas;
  g_local_ctas = local_ctas;
  return FTAR_OK;
}

int ftar_ctx_create(int device, uint64_t max_bucket_bytes, uint64_t pool_bytes, int exportable,
                    ftar_ctx** out) {
  if (!out) return fail(FTAR_ST_INVARIANT, "null out");
  DeviceGuard g(device);
  ftar_ctx* c = new ftar_ctx();
  c->device = device;
  c->exportable = exportable != 0;
  c->max_bucket_bytes = align_up(std::max<uint64_t>(max_bucket_bytes, 256), 256);
  c->res_off = kRecvOff + kRecvBytes;
  // result region: the fp32 image of a whole bucket (E <= max_bucket_bytes/2
  // for bf16 -> 2x bytes); the protocol kernel uses my slice of it, the
  // in-process one-shot kernel stages the whole fp32 sum in member 0's.
  const uint64_t res_bytes = align_up(2 * c->max_bucket_bytes + 64, 4096);
  c->stage_off[0] = c->res_off + res_bytes;
  c->stage_off[1] = c->stage_off[0] + c->max_bucket_bytes;
  c->pool_off = c->stage_off[1] + c->max_bucket_bytes;
  c->pool_bytes = align_up(pool_bytes, 4096);
  c->arena_bytes = c->pool_off + c->pool_bytes;
  cudaError_t e = cudaMalloc(&c->arena, c->arena_bytes);
  if (e != cudaSuccess) {
    delete c;
    return cuda_fail(e, "cudaMalloc(arena)");
  }
  cudaMemset(c->arena, 0, kHdrBytes);
  ArenaHdr init{};
  init.err_peer = -1;
  cudaMemcpy(c->arena, &init, sizeof(init), cudaMemcpyHostToDevice);
  e = cudaHostAlloc(&c->ctl_hs, kQueue * sizeof(HostCtl), cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) {
    cudaFree(c->arena);
    delete c;
    return cuda_fail(e, "cudaHostAlloc(ctl)");
  }
  std::memset((void*)c->ctl_hs, 0, kQueue * sizeof(HostCtl));
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->ctl_ds), (void*)c->ctl_hs, 0);
  for (int i = 0; i < kQueue; ++i) {
    reset_ctl(c->ctl_hs + i);
    c->ctl_hs[i].live_mask = 1;
    c->ctl_hs[i].contrib_mask = 1;
  }
  c->ctl_h = c->ctl_hs;
  c->ctl_d = c->ctl_ds;
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_fail(e, "ctx init");
  c->ring_slots[0] = -1;
  *out = c;
  return FTAR_OK;
}

int ftar_ctx_destroy(ftar_ctx* c) {
  if (!c) return FTAR_OK;
  DeviceGuard g(c->device);
  // queued collectives waiting on a peer that is gone would otherwise hold the
  // synchronize below until the device hard timeout: abort them first
  for (int i = 0; i < c->q_count; ++i) {
    const int slot = (c->q_head + i) % kQueue;
    c->ctl_hs[slot].abort_tag = c->q_tag[slot];
  }
  cudaDeviceSynchronize();
  for (auto& b : c->blocks) cudaIpcCloseMemHandle(b.va);
  c->blocks.clear();
  for (int s = 0; s < kMaxSlots; ++s)
    if (c->peer[s] && !c->peer_local[s]) cudaIpcCloseMemHandle(c->peer[s]);
  cudaFree(c->arena);
  cudaFreeHost((void*)c->ctl_hs);
  delete c;
  return FTAR_OK;
}

int ftar_ctx_pool(ftar_ctx* c, uint64_t* dev_ptr, uint64_t* bytes) {
  if (!c) return fail(FTAR_ST_INVARIANT, "null ctx");
  if (dev_ptr) *dev_ptr = reinterpret_cast<uint64_t>(c->arena + c->pool_off);
  if (bytes) *bytes = c->pool_bytes;
  return FTAR_OK;
}

int ftar_ctx_export(ftar_ctx* c, void* buf, size_t buflen, size_t* written) {
  if (!c || !buf || buflen < sizeof(cudaIpcMemHandle_t)) return fail(FTAR_ST_INVARIANT, "bad export args");
  DeviceGuard g(c->device);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, c->arena));
  std::memcpy(buf, &h, sizeof(h));
  if (written) *written = sizeof(h);
  return FTAR_OK;
}

int ftar_ctx_import(ftar_ctx* c, int slot, const void* handle, size_t len, uint64_t arena_bytes) {
  if (!c || slot < 0 || slot >= kMaxSlots || !handle || len < sizeof(cudaIpcMemHandle_t))
    return fail(FTAR_ST_INVARIANT, "bad import args");
  DeviceGuard g(c->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  if (c->peer[slot]) {
    // cached mapping of the SAME arena only: a slot still holding another
    // member's (or a dead incarnation's) arena must be unmapped first, never
    // silently reused for a different handle
    if (!c->peer_local[slot] && std::memcmp(&c->peer_handle[slot], &h, sizeof(h)) == 0) return FTAR_OK;
    return fail(FTAR_ST_INVARIANT, "slot " + std::to_string(slot) + " maps a different arena (unmap it first)");
  }
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    g_err = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
    return FTAR_ST_PEER_DOWN;
  }
  c->peer[slot] = static_cast<char*>(p);
  c->peer_handle[slot] = h;
  c->peer_bytes[slot] = arena_bytes;
  return FTAR_OK;
}

int ftar_ctx_link_local(ftar_ctx* c, int slot, ftar_ctx* other) {
  // Single-process multi-GPU: map member `other` (another device of this
  // process) as `slot` through peer access instead of CUDA IPC.
  if (!c || !other || slot < 0 || slot >= kMaxSlots) return fail(FTAR_ST_INVARIANT, "bad link args");
  if (c->peer[slot] && c->peer[slot] != other->arena) return fail(FTAR_ST_INVARIANT, "slot in use");
  if (c->device != other->device) {
    DeviceGuard g(c->device);
    cudaError_t e = cudaDeviceEnablePeerAccess(other->device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_fail(e, "enable peer access");
    cudaGetLastError();
  }
  c->peer[slot] = other->arena;
  c->peer_local[slot] = true;
  return FTAR_OK;
}

int ftar_ctx_unmap(ftar_ctx* c, int slot) {
  if (!c || slot < 0 || slot >= kMaxSlots) return fail(FTAR_ST_INVARIANT, "bad unmap args");
  for (int i = 0; i < c->n; ++i)
    if (i != c->self && c->ring_slots[i] == slot)
      return fail(FTAR_ST_INVARIANT, "slot " + std::to_string(slot) + " belongs to the current ring");
  DeviceGuard g(c->device);
  c->drop_slot_regions(slot);
  if (c->peer[slot]) {
    if (!c->peer_local[slot]) cudaIpcCloseMemHandle(c->peer[slot]);
    c->peer[slot] = nullptr;
    c->peer_local[slot] = false;
    std::memset(&c->peer_handle[slot], 0, sizeof(cudaIpcMemHandle_t));
  }
  return FTAR_OK;
}

int ftar_region_register(ftar_ctx* c, const void* ptr, uint64_t bytes, int* rid_out, void* handle,
                         size_t buflen, uint64_t* offset_out) {
  // Export the allocation block holding [ptr, ptr+bytes) (any caching-
  // allocator tensor): its IPC handle and ptr's offset inside it.  The
  // region id names the buffer in entry records.
  if (!c || !ptr || !bytes || !rid_out || !handle || buflen < sizeof(cudaIpcMemHandle_t) || !offset_out)
    return fail(FTAR_ST_INVARIANT, "bad register args");
  DeviceGuard g(c->device);
  uint64_t off = 0;
  int rid = c->find_region(ptr, bytes, &off);
  if (rid < 0) {
    for (int r = 0; r < kMaxRegions && rid < 0; ++r)
      if (!c->my_region_bytes[r]) rid = r;
    if (rid < 0) return fail(FTAR_ST_INVARIANT, "all 16 region ids in use (unregister one first)");
    c->my_region_ptr[rid] = reinterpret_cast<uint64_t>(ptr);
    c->my_region_bytes[rid] = bytes;
    off = 0;
  }
  using GetRange = int (*)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
    if (!fn) return fail(FTAR_ST_CUDA, "cuMemGetAddressRange unavailable");
    get_range = reinterpret_cast<GetRange>(fn);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0 || !base)
    return fail(FTAR_ST_INVARIANT, "pointer is not inside a device allocation");
  if (reinterpret_cast<uint64_t>(ptr) + bytes > base + size) return fail(FTAR_ST_INVARIANT, "region spans allocations");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle, &h, sizeof(h));
  *rid_out = rid;
  *offset_out = c->my_region_ptr[rid] - base;  // the region's start inside the block
  (void)off;
  return FTAR_OK;
}

int ftar_region_unregister(ftar_ctx* c, int rid) {
  if (!c || rid < 0 || rid >= kMaxRegions) return fail(FTAR_ST_INVARIANT, "bad region id");
  if (c->q_count && !c->all_done()) return fail(FTAR_ST_INVARIANT, "unregister with a collective in flight");
  c->my_region_ptr[rid] = c->my_region_bytes[rid] = 0;
  return FTAR_OK;
}

int ftar_region_import(ftar_ctx* c, int slot, int rid, const void* handle, size_t len, uint64_t offset,
                       uint64_t bytes) {
  // Map peer `slot`'s registered region `rid` (its block's IPC handle + the
  // region's offset in it); one mapping per peer block, shared by regions.
  if (!c || slot < 0 || slot >= kMaxSlots || rid < 0 || rid >= kMaxRegions || !handle ||
      len < sizeof(cudaIpcMemHandle_t))
    return fail(FTAR_ST_INVARIANT, "bad region import args");
  (void)bytes;
  DeviceGuard g(c->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  char* va = nullptr;
  for (auto& b : c->blocks)
    if (b.slot == slot && std::memcmp(&b.h, &h, sizeof(h)) == 0) va = b.va;
  if (!va) {
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      g_err = std::string("cudaIpcOpenMemHandle(region): ") + cudaGetErrorString(e);
      return FTAR_ST_PEER_DOWN;
    }
    va = static_cast<char*>(p);
    c->blocks.push_back({h, va, slot});
  }
  c->peer_region_va[slot][rid] = reinterpret_cast<uint64_t>(va) + offset;
  return FTAR_OK;
}

int ftar_set_membership(ftar_ctx* c, const int* ring_slots, int n, int self_index,
                        uint32_t contrib_mask, uint64_t generation) {
  if (!c || n < 1 || n > kMaxMembers || self_index < 0 || self_index >= n)
    return fail(FTAR_ST_INVARIANT, "bad membership");
  if (generation > 0xffffffull) return fail(FTAR_ST_INVARIANT, "generation exceeds 24 bits");
  if (c->q_count) {
    if (!c->all_done()) return fail(FTAR_ST_INVARIANT, "membership change with an all-reduce in flight");
    c->q_head = (c->q_head + c->q_count) % kQueue;  // statuses of finished, unwaited ops are dropped
    c->q_count = 0;
  }
  for (int i = 0; i < n; ++i) {
    if (i == self_index) {
      c->ring_slots[i] = -1;
      continue;
    }
    const int s = ring_slots ? ring_slots[i] : -1;
    if (s < 0 || s >= kMaxSlots || !c->peer[s]) return fail(FTAR_ST_INVARIANT, "ring member not mapped");
    c->ring_slots[i] = s;
  }
  // publish the installed generation in my arena (the zombie guard of
  // senders that push into it); no kernel of mine is running here
  {
    DeviceGuard g(c->device);
    CK(cudaMemcpy(c->arena + offsetof(ArenaHdr, gen_word), &generation, sizeof(uint64_t), cudaMemcpyHostToDevice));
  }
  if (n != c->n || !c->warmed) {  // load this ring size's kernel instances now, not mid-collective
    DeviceGuard g(c->device);
    warm_ring_kernels<F32In>(n);
    warm_ring_kernels<BF16In>(n);
    c->warmed = true;
  }
  c->n = n;
  c->self = self_index;
  c->contrib = contrib_mask & ((n >= 32) ? 0xffffffffu : ((1u << n) - 1u));
  c->gen = generation;
  c->seq = 0;
  for (int i = 0; i < kQueue; ++i) {
    c->ctl_hs[i].live_mask = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
    c->ctl_hs[i].contrib_mask = c->contrib;
    c->ctl_hs[i].epoch = generation;
  }
  return FTAR_OK;
}

int ftar_geometry(uint64_t n_elems, int n, uint64_t* slice_elems, int* ctas, int* threads) {
  if (n < 1 || n > kMaxMembers) return fail(FTAR_ST_INVARIANT, "ring size out of range 1..8");
  LaunchParams p{};
  fill_geometry(p, n_elems, 4, 1, n);
  if (slice_elems) *slice_elems = p.slice;
  if (ctas) *ctas = real_ctas();
  if (threads) *threads = kThreads;
  return FTAR_OK;
}

int ftar_inflight_bound(int n, uint64_t n_elems, int in_dtype, uint64_t chunk_bytes, int max_in_flight, int push,
                        uint64_t* bytes_per_link, int* ctas, int* path) {
  // The InflightMeter's figure (ftar.py:141-159): the most bytes one peer
  // link can have outstanding for this call, on the path launch_real picks.
  //   small push one-shot: the whole input, posted to each peer;
  //   bulk-copy reduce-scatter: G CTAs x (S-1) stages x one tile per peer;
  //   register path: G CTAs x 512 threads x U vectors of 4 elements per peer.
  if (n < 1 || n > kMaxMembers) return fail(FTAR_ST_INVARIANT, "ring size out of range");
  int v = validate_common(in_dtype, n, chunk_bytes, max_in_flight);
  if (v) return v;
  const uint64_t esz = in_dtype == FTAR_DT_BF16 ? 2 : 4;
  const uint64_t in_bytes = n_elems * esz;
  LaunchParams p{};
  fill_geometry(p, n_elems, chunk_bytes, max_in_flight, n);
  p.nelems = n_elems;
  const bool small = n >= 2 && in_bytes > 0 && in_bytes <= small_bytes();
  PathChoice pc{kPathNone, 0, 0};
  uint64_t bound = 0;
  if (n >= 2 && in_bytes > 0) {
    pc = choose_path(n, p, esz, small, false, push != 0);
    if (pc.kind == kPathSmall) {
      bound = in_bytes;
    } else if (pc.kind == kPathBulk) {
      bound = (uint64_t)pc.ctas * (pc.stages - 1) * tma_tile(n, (int)esz) * esz;
    } else {
      const int N = n;
      const int budget = (N >= 6 && esz == 2) ? 8 : (N >= 5 ? 12 : 16);  // Unroll<N, In>
      const int u0 = (budget * 16 / (int)(esz * 4)) / N;
      const int umax = N <= 2 ? 16 : (N == 3 ? 6 : 8);
      const int U = u0 < 1 ? 1 : (u0 > umax ? umax : u0);
      bound = (uint64_t)pc.ctas * kThreads * (uint64_t)U * 4 * esz;
    }
  }
  if (bytes_per_link) *bytes_per_link = bound;
  if (ctas) *ctas = pc.ctas;
  if (path) *path = pc.kind;
  return FTAR_OK;
}

struct SgdArgs {
  const float* p = nullptr;
  const float* m = nullptr;
  float* po = nullptr;
  float* mo = nullptr;
  float lr = 0.f, beta = 0.f;
};

static int launch_real(ftar_ctx* c, const void* in, int in_dtype, float* out, uint64_t n_elems,
                       uint64_t base_elem, uint64_t total_elems, uint64_t chunk_bytes, int max_in_flight,
                       float scale, uint32_t flags, void* stream, const SgdArgs* sgd);

int ftar_allreduce_launch_range(ftar_ctx* c, const void* in, int in_dtype, float* out, uint64_t n_elems,
                                uint64_t base_elem, uint64_t total_elems, uint64_t chunk_bytes,
                                int max_in_flight, float scale, uint32_t flags, void* stream) {
  return launch_real(c, in, in_dtype, out, n_elems, base_elem, total_elems, chunk_bytes, max_in_flight, scale,
                     flags, stream, nullptr);
}

int ftar_allreduce_sgd_launch(ftar_ctx* c, const void* in, int in_dtype, float* grad_out, uint64_t n_elems,
                              uint64_t chunk_bytes, int max_in_flight, float scale, uint32_t flags,
                              const float* params, const float* momentum, float* params_out, float* momentum_out,
                              float lr, float beta, void* stream) {
  if (!params || !momentum || !params_out || !momentum_out) return fail(FTAR_ST_INVARIANT, "null optimizer state");
  SgdArgs a;
  a.p = params;
  a.m = momentum;
  a.po = params_out;
  a.mo = momentum_out;
  a.lr = lr;
  a.beta = beta;
  return launch_real(c, in, in_dtype, grad_out, n_elems, 0, n_elems, chunk_bytes, max_in_flight, scale, flags,
                     stream, &a);
}

static int launch_real(ftar_ctx* c, const void* in, int in_dtype, float* out, uint64_t n_elems,
                       uint64_t base_elem, uint64_t total_elems, uint64_t chunk_bytes, int max_in_flight,
                       float scale, uint32_t flags, void* stream, const SgdArgs* sgd) {
  if (base_elem + n_elems > total_elems) return fail(FTAR_ST_INVARIANT, "range exceeds the bucket");
  if (!c) return fail(FTAR_ST_INVARIANT, "null ctx");
  int v = validate_common(in_dtype, c->n, chunk_bytes, max_in_flight);
  if (v) return v;
  if (c->q_count == kQueue) return fail(FTAR_ST_INVARIANT, "all-reduce queue full: wait for the oldest first");
  const uint64_t esz = in_dtype == FTAR_DT_BF16 ? 2 : 4;
  const uint64_t in_bytes = n_elems * esz;
  if (in_bytes > c->max_bucket_bytes || n_elems * 4 > 2 * c->max_bucket_bytes)
    return fail(FTAR_ST_INVARIANT, "bucket exceeds the ring group's arena capacity");
  if (n_elems && (!in || (!out && !sgd))) return fail(FTAR_ST_INVARIANT, "null buffer");
  DeviceGuard g(c->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  c->seq += 1;
  const uint64_t tag = mk_tag(c->gen, c->seq);
  const char* inp = static_cast<const char*>(in);
  uint64_t in_off;
  const bool registered = inp >= c->arena + c->pool_off && inp + in_bytes <= c->arena + c->arena_bytes;
  const bool small = c->n >= 2 && !sgd && in_bytes > 0 && in_bytes <= small_bytes();
  uint64_t roff = 0;
  const int rid = (!registered && c->n >= 2 && !small) ? c->find_region(inp, in_bytes, &roff) : -1;
  uint64_t my_in_va = reinterpret_cast<uint64_t>(inp);
  if (registered || c->n == 1 || small) {  // small buckets: peers never read my input
    in_off = (uint64_t)(inp - c->arena);
  } else if (rid >= 0) {
    // a registered user buffer: peers read it in place through their mapping
    in_off = region_ref((uint32_t)rid, roff);
  } else {
    // Unregistered bucket: peers can only read the arena, so stage it (double
    // buffered by call parity: peers finished reading this half two calls ago).
    const uint64_t so = c->stage_off[c->seq & 1];
    if (in_bytes) CK(cudaMemcpyAsync(c->arena + so, in, in_bytes, cudaMemcpyDeviceToDevice, st));
    in_off = so;
    my_in_va = reinterpret_cast<uint64_t>(c->arena + so);
  }
  LaunchParams p{};
  fill_geometry(p, n_elems, chunk_bytes, max_in_flight, c->n, base_elem, total_elems);
  for (int i = 0; i < c->n; ++i) p.base[i] = (i == c->self) ? c->arena : c->peer[c->ring_slots[i]];
  p.my_in_va = my_in_va;
  for (int i = 0; i < c->n; ++i)
    if (i != c->self)
      for (int r = 0; r < kMaxRegions; ++r) p.region_va[i][r] = c->peer_region_va[c->ring_slots[i]][r];
  c->push(tag);
  p.ctl[c->self] = c->ctl_d;
  p.out[c->self] = out;
  p.in_off[c->self] = in_off;
  p.res_off[c->self] = c->res_off;
  p.tag = tag;
  p.nelems = n_elems;
  p.hard_timeout_ns = c->hard_timeout_ns;
  p.scale = scale;
  p.flags = flags & 0xffu;
  {
    // out-of-place: the reduce-scatter also writes my slice of `out` (peers
    // still pull from the library-owned result region, so `out` is free for
    // the caller as soon as the call returns)
    const uint64_t o0 = reinterpret_cast<uint64_t>(out), i0 = reinterpret_cast<uint64_t>(in);
    const bool alias = o0 < i0 + in_bytes && i0 < o0 + n_elems * 4;
    if (out && !alias && n_elems && !env_int("FTAR_NO_DIRECT", 0)) p.flags |= kFlagDirect;
    if (sgd) {
      p.flags |= kFlagSGD;
      p.sgd_p[c->self] = sgd->p;
      p.sgd_m[c->self] = sgd->m;
      p.sgd_po[c->self] = sgd->po;
      p.sgd_mo[c->self] = sgd->mo;
      p.sgd_lr = sgd->lr;
      p.sgd_beta = sgd->beta;
    }
    // push mode needs `out` addressable by the peers: in my exported arena
    // or a registered buffer (peers write into it)
    const char* op = reinterpret_cast<const char*>(out);
    const bool out_pool = op >= c->arena + c->pool_off && op + n_elems * 4 <= c->arena + c->arena_bytes;
    uint64_t ooff = 0;
    const int orid = out_pool ? -1 : c->find_region(op, n_elems * 4, &ooff);
    if (!sgd && (p.flags & kFlagDirect) && (out_pool || orid >= 0) && !env_int("FTAR_NO_PUSH", 0)) {
      p.flags |= kFlagPush;
      p.out_off[c->self] = out_pool ? (uint64_t)(op - c->arena) : region_ref((uint32_t)orid, ooff);
    }
  }
  p.contrib = c->contrib;
  set_workers(p, c->n, n_elems);
  p.dtype = (uint32_t)in_dtype;
  p.self = c->self;
  p.emulated = 0;
  p.fault_member = -1;
  p.fault_after_tiles = 0;
  p.rs_layout = rs_layout();
  p.diag = diag_mode();
  p.rs_ctas = rs_ctas_knob();
  const PathChoice pc = choose_path(c->n, p, esz, small, sgd != nullptr, (p.flags & kFlagPush) != 0);
  if (small) {
    if (p.flags & kFlagDirect) p.flags |= kFlagSmallDirect;
    p.flags &= ~(kFlagPush | kFlagDirect);
  }
  p.tma_stages = pc.stages;
  {
    // Early PDL trigger (FTAR_PDL_EARLY: 0 off, 1 register-path calls, 2
    // every call).  N=4 f32, queue depth 3 (tools/tune_tma.py --early,
    // profiles/r02/tune/pdl_early_n4.jsonl): +8-15% from 2 to 16 MiB, but
    // -2..-5% on the bulk-copy path (64 MiB and up), also when only CTA 0
    // triggers early, so the bulk path keeps the end-of-call trigger.
    const int early = env_int("FTAR_PDL_EARLY", 1);
    p.early_trigger = (pdl_on() && (early >= 2 || (early == 1 && pc.kind != kPathBulk))) ? 1u : 0u;
  }
  p.entry_fence = env_int("FTAR_ENTRY_FENCE", 0) != 0 ? 1u : 0u;
  const dim3 grid(pc.ctas, 1);
  cudaError_t e = small ? (in_dtype == FTAR_DT_BF16 ? launch_small<BF16In>(c->n, p, grid, st, false, pdl_on())
                                                    : launch_small<F32In>(c->n, p, grid, st, false, pdl_on()))
                        : (in_dtype == FTAR_DT_BF16 ? launch_dispatch<BF16In>(c->n, p, grid, st, false, pdl_on())
                                                    : launch_dispatch<F32In>(c->n, p, grid, st, false, pdl_on()));
  if (e != cudaSuccess) {
    c->pop_last();
    return cuda_fail(e, "allreduce launch");
  }
  return FTAR_OK;
}

static int launch_local(ftar_ctx** ctxs, int n, const void* const* ins, int in_dtype, float* const* outs,
                        uint64_t n_elems, uint64_t base_elem, uint64_t total_elems, uint64_t chunk_bytes,
                        int max_in_flight, float scale, uint32_t flags, uint32_t contrib_mask, int fault_member,
                        int fault_after_tiles, void* stream, const float* const* sgd_p, const float* const* sgd_m,
                        float* const* sgd_po, float* const* sgd_mo, float lr, float beta);

int ftar_local_allreduce_launch_range(ftar_ctx** ctxs, int n, const void* const* ins, int in_dtype,
                                      float* const* outs, uint64_t n_elems, uint64_t base_elem,
                                      uint64_t total_elems, uint64_t chunk_bytes, int max_in_flight,
                                      float scale, uint32_t flags, uint32_t contrib_mask, int fault_member,
                                      int fault_after_tiles, void* stream) {
  return launch_local(ctxs, n, ins, in_dtype, outs, n_elems, base_elem, total_elems, chunk_bytes, max_in_flight,
                      scale, flags, contrib_mask, fault_member, fault_after_tiles, stream, nullptr, nullptr, nullptr,
                      nullptr, 0.f, 0.f);
}

int ftar_local_allreduce_sgd_launch(ftar_ctx** ctxs, int n, const void* const* ins, int in_dtype,
                                    float* const* grad_outs, uint64_t n_elems, uint64_t chunk_bytes,
                                    int max_in_flight, float scale, uint32_t flags, uint32_t contrib_mask,
                                    const float* const* params, const float* const* momentum,
                                    float* const* params_out, float* const* momentum_out, float lr, float beta,
                                    void* stream) {
  if (!params || !momentum || !params_out || !momentum_out) return fail(FTAR_ST_INVARIANT, "null optimizer state");
  return launch_local(ctxs, n, ins, in_dtype, grad_outs, n_elems, 0, n_elems, chunk_bytes, max_in_flight, scale,
                      flags | FTAR_F_PROTOCOL, contrib_mask, -1, 0, stream, params, momentum, params_out,
                      momentum_out, lr, beta);
}

static int launch_local(ftar_ctx** ctxs, int n, const void* const* ins, int in_dtype, float* const* outs,
                        uint64_t n_elems, uint64_t base_elem, uint64_t total_elems, uint64_t chunk_bytes,
                        int max_in_flight, float scale, uint32_t flags, uint32_t contrib_mask, int fault_member,
                        int fault_after_tiles, void* stream, const float* const* sgd_p, const float* const* sgd_m,
                        float* const* sgd_po, float* const* sgd_mo, float lr, float beta) {
  if (base_elem + n_elems > total_elems) return fail(FTAR_ST_INVARIANT, "range exceeds the bucket");
  int v = validate_common(in_dtype, n, chunk_bytes, max_in_flight);
  if (v) return v;
  if (!ctxs || !ins || !outs) return fail(FTAR_ST_INVARIANT, "null arrays");
  const int dev = ctxs[0]->device;
  for (int i = 0; i < n; ++i) {
    ftar_ctx* c = ctxs[i];
    if (!c || c->device != dev) return fail(FTAR_ST_INVARIANT, "in-process ring members must share a device");
    // queued launches run back to back on the stream; ftar_wait_local
    // collects each member's oldest (FIFO), like ftar_wait
    if (c->q_count == kQueue) return fail(FTAR_ST_INVARIANT, "queue full: wait for the oldest first");
    if (n_elems * 4 > 2 * c->max_bucket_bytes)
      return fail(FTAR_ST_INVARIANT, "bucket exceeds the ring group's arena capacity");
    if (c->gen != ctxs[0]->gen || c->seq != ctxs[0]->seq)
      return fail(FTAR_ST_PROTOCOL, "ring members disagree on (generation, call sequence)");
  }
  DeviceGuard g(dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LaunchParams p{};
  fill_geometry(p, n_elems, chunk_bytes, max_in_flight, n, base_elem, total_elems);
  uint64_t tag = 0;
  for (int i = 0; i < n; ++i) {
    ftar_ctx* c = ctxs[i];
    c->seq += 1;
    tag = mk_tag(c->gen, c->seq);
    c->push(tag);
    p.base[i] = c->arena;
    p.ctl[i] = c->ctl_d;
    p.out[i] = outs[i];
    p.in_off[i] = (uint64_t)(static_cast<const char*>(ins[i]) - c->arena);
    p.res_off[i] = c->res_off;
  }
  p.tag = tag;
  p.nelems = n_elems;
  p.hard_timeout_ns = ctxs[0]->hard_timeout_ns;
  p.scale = scale;
  p.flags = flags & 0xffu;
  {
    const uint64_t ib = n_elems * (in_dtype == FTAR_DT_BF16 ? 2 : 4), ob = n_elems * 4;
    bool alias = false, null_out = false;
    for (int i = 0; i < n && !alias; ++i) {
      null_out |= outs[i] == nullptr;
      for (int j = 0; j < n && !alias; ++j) {
        const uint64_t o0 = reinterpret_cast<uint64_t>(outs[i]), i0 = reinterpret_cast<uint64_t>(ins[j]);
        alias = o0 < i0 + ib && i0 < o0 + ob;
      }
    }
    if (!alias && !null_out && n_elems) p.flags |= kFlagDirect;
    if (sgd_p) {
      p.flags |= kFlagSGD;
      for (int i = 0; i < n; ++i) {
        p.sgd_p[i] = sgd_p[i];
        p.sgd_m[i] = sgd_m[i];
        p.sgd_po[i] = sgd_po[i];
        p.sgd_mo[i] = sgd_mo[i];
      }
      p.sgd_lr = lr;
      p.sgd_beta = beta;
    }
    if (!sgd_p && (p.flags & kFlagDirect) && !env_int("FTAR_NO_PUSH", 0)) {
      p.flags |= kFlagPush;  // in-process: every member's out is addressable
      for (int i = 0; i < n; ++i)
        p.out_off[i] = (uint64_t)(reinterpret_cast<const char*>(outs[i]) - ctxs[i]->arena);
    }
  }
  p.contrib = contrib_mask & ((1u << n) - 1u);
  set_workers(p, n, n_elems);
  p.dtype = (uint32_t)in_dtype;
  p.self = 0;
  p.emulated = 1;
  p.fault_member = fault_member;
  p.fault_after_tiles = fault_after_tiles;
  p.rs_layout = rs_layout();
  p.diag = diag_mode();
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (!(flags & FTAR_F_PROTOCOL) && fault_member < 0) {
    LocalParams lp{};
    for (int i = 0; i < n; ++i) {
      lp.in[i] = ins[i];
      lp.out[i] = outs[i];
      lp.ctl[i] = ctxs[i]->ctl_d;
      lp.tag[i] = ctxs[i]->cur_tag;
    }
    ArenaHdr* h0 = reinterpret_cast<ArenaHdr*>(ctxs[0]->arena);
    // direct mode unless some output overlaps some input (in-place calls):
    // then stage so that a non-finite sum leaves every buffer untouched
    const uint64_t ib = n_elems * (in_dtype == FTAR_DT_BF16 ? 2 : 4), ob = n_elems * 4;
    bool alias = false;
    for (int i = 0; i < n && !alias; ++i)
      for (int j = 0; j < n && !alias; ++j) {
        const uint64_t o0 = reinterpret_cast<uint64_t>(outs[i]), i0 = reinterpret_cast<uint64_t>(ins[j]);
        alias = o0 < i0 + ib && i0 < o0 + ob;
      }
    lp.stage = alias ? reinterpret_cast<float*>(ctxs[0]->arena + ctxs[0]->res_off) : nullptr;
    lp.flags = &h0->nonfinite;
    lp.arrive = &h0->done_arrive;
    lp.nelems = n_elems;
    lp.p_base = p.p_base;
    lp.p_rem = p.p_rem;
    lp.ebase = p.ebase;
    lp.scale = scale;
    lp.flags_in = flags;
    lp.contrib = p.contrib;
    const int esz = in_dtype == FTAR_DT_BF16 ? 2 : 4;
    uint64_t orbits = 0;
    for (int i = 0; i < n; ++i) orbits |= reinterpret_cast<uint64_t>(ins[i]) | reinterpret_cast<uint64_t>(outs[i]);
    // the bulk-copy form: direct mode, 16-byte aligned buffers, every
    // segment at least one tile (at most one owner change per tile)
    const bool bulk = !alias && (orbits & 15u) == 0 && tma_on() && env_int("FTAR_LOCAL_BULK", 1) != 0 &&
                      n_elems >= 8 && p.p_base / (uint64_t)n >= lb_tile(n, esz);
    cudaError_t e;
    if (bulk) {
      lp.stages = lb_stages_for(n, esz);
      const dim3 grid(std::max(1, env_int("FTAR_LOCAL_BULK_CTAS", sms)));
      e = in_dtype == FTAR_DT_BF16 ? local_bulk_dispatch<BF16In>(n, lp, grid, st)
                                   : local_bulk_dispatch<F32In>(n, lp, grid, st);
    } else {
      const int bps = in_dtype == FTAR_DT_BF16 ? oneshot_blocks_per_sm<BF16In>(n) : oneshot_blocks_per_sm<F32In>(n);
      const dim3 grid(std::max(1, sms * std::max(bps, 1)));
      e = in_dtype == FTAR_DT_BF16 ? oneshot_dispatch<BF16In>(n, lp, grid, st)
                                   : oneshot_dispatch<F32In>(n, lp, grid, st);
    }
    if (e != cudaSuccess) {
      for (int i = 0; i < n; ++i) ctxs[i]->pop_last();
      return cuda_fail(e, "local one-shot cooperative launch");
    }
    return FTAR_OK;
  }
  const int per_sm = in_dtype == FTAR_DT_BF16 ? max_coop_blocks_per_sm<BF16In>(n) : max_coop_blocks_per_sm<F32In>(n);
  int G = std::max(1, (sms * std::max(per_sm, 1)) / n);
  const int want = g_local_ctas > 0 ? g_local_ctas : env_int("FTAR_LOCAL_CTAS", 32);
  G = std::min(G, want);
  const uint64_t in_bytes_l = n_elems * (in_dtype == FTAR_DT_BF16 ? 2 : 4);
  const bool small = n >= 2 && !sgd_p && fault_member < 0 && in_bytes_l > 0 && in_bytes_l <= small_bytes();
  if (small) {
    if (p.flags & kFlagDirect) p.flags |= kFlagSmallDirect;
    p.flags &= ~(kFlagPush | kFlagDirect);
    G = std::min(G, small_ctas(in_bytes_l));
    const dim3 sgrid(G, n);
    cudaError_t e = in_dtype == FTAR_DT_BF16 ? launch_small<BF16In>(n, p, sgrid, st, true)
                                              : launch_small<F32In>(n, p, sgrid, st, true);
    if (e != cudaSuccess) {
      for (int i = 0; i < n; ++i) ctxs[i]->pop_last();
      return cuda_fail(e, "local small-bucket cooperative launch");
    }
    return FTAR_OK;
  }
  if (!sgd_p && n >= 2 && tma_on() && p.p_base / (uint64_t)n >= tma_tile(n, in_dtype == FTAR_DT_BF16 ? 2 : 4)) {
    p.tma_stages = tma_stages_for(n, in_dtype == FTAR_DT_BF16 ? 2 : 4);
    if (g_local_ctas <= 0) G = std::min(G, tma_ctas(n, p.slice * (in_dtype == FTAR_DT_BF16 ? 2 : 4)));
  }
  const dim3 grid(G, n);
  cudaError_t e = in_dtype == FTAR_DT_BF16 ? launch_dispatch<BF16In>(n, p, grid, st, true)
                                            : launch_dispatch<F32In>(n, p, grid, st, true);
  if (e != cudaSuccess) {
    for (int i = 0; i < n; ++i) ctxs[i]->pop_last();
    return cuda_fail(e, "local allreduce cooperative launch");
  }
  return FTAR_OK;
}

int ftar_allreduce_launch(ftar_ctx* c, const void* in, int in_dtype, float* out, uint64_t n_elems,
                          uint64_t chunk_bytes, int max_in_flight, float scale, uint32_t flags,
                          void* stream) {
  return ftar_allreduce_launch_range(c, in, in_dtype, out, n_elems, 0, n_elems, chunk_bytes, max_in_flight,
                                     scale, flags, stream);
}

int ftar_local_allreduce_launch(ftar_ctx** ctxs, int n, const void* const* ins, int in_dtype,
                                float* const* outs, uint64_t n_elems, uint64_t chunk_bytes,
                                int max_in_flight, float scale, uint32_t flags, uint32_t contrib_mask,
                                int fault_member, int fault_after_tiles, void* stream) {
  return ftar_local_allreduce_launch_range(ctxs, n, ins, in_dtype, outs, n_elems, 0, n_elems, chunk_bytes,
                                           max_in_flight, scale, flags, contrib_mask, fault_member,
                                           fault_after_tiles, stream);
}

int ftar_poll(ftar_ctx* c, int* status, uint64_t* progress) {
  if (!c) return fail(FTAR_ST_INVARIANT, "null ctx");
  if (!c->q_count) {
    if (status) *status = FTAR_OK;
    if (progress) *progress = c->ctl_h->progress;
    return FTAR_OK;
  }
  const HostCtl* h = c->ctl_hs + c->q_head;
  const uint64_t d = h->done;
  if (progress) *progress = h->progress;
  if (status) *status = flag_tag(d) == c->q_tag[c->q_head] ? (int)(d & 0xff) : FTAR_ST_PENDING;
  return FTAR_OK;
}

// ---- intra-replica collectives (§8f rank 2) -------------------------------
static int intra_check(int op, int in_dtype, int n, uint64_t total, const uint64_t* offs, const uint64_t* lens) {
  if (op != (int)kIntraRS && op != (int)kIntraAG) return fail(FTAR_ST_INVARIANT, "op must be 1 (RS) or 2 (AG)");
  if (in_dtype != FTAR_DT_F32 && in_dtype != FTAR_DT_BF16) return fail(FTAR_ST_INVARIANT, "dtype must be f32 or bf16");
  if (op == (int)kIntraAG && in_dtype != FTAR_DT_F32) return fail(FTAR_ST_INVARIANT, "all-gather shards are fp32");
  if (n < 1 || n > kMaxMembers) return fail(FTAR_ST_INVARIANT, "1..8 ranks");
  if (!offs || !lens) return fail(FTAR_ST_INVARIANT, "null bounds");
  for (int k = 0; k < n; ++k)
    if (offs[k] > total || lens[k] > total - offs[k]) return fail(FTAR_ST_INVARIANT, "shard bounds exceed the vector");
  return FTAR_OK;
}

static void intra_grid_params(LaunchParams& p, int op, int in_dtype, uint64_t total, const uint64_t* offs,
                              const uint64_t* lens, int n) {
  p.intra_op = (uint32_t)op;
  p.nelems = total;
  p.total = total;
  p.cap = 0;
  p.ebase = 0;
  p.dtype = (uint32_t)in_dtype;
  p.contrib = (n >= 32) ? 0xffffffffu : ((1u << n) - 1u);
  for (int k = 0; k < n; ++k) {
    p.seg_off[k] = offs[k];
    p.seg_len[k] = lens[k];
  }
}

static int intra_ctas(int op, int in_dtype, uint64_t total, const uint64_t* lens, int self, int n) {
  // ~64 KB of my work per CTA, like the all-reduce grid sizing
  uint64_t work = op == (int)kIntraRS ? lens[self] * (in_dtype == FTAR_DT_BF16 ? 2 : 4) : total * 4 / (uint64_t)n;
  const uint64_t per = (uint64_t)env_int("FTAR_BYTES_PER_CTA", 64 << 10);
  const int cap = g_ctas > 0 ? g_ctas : 64;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)cap, (work + per - 1) / per));
}

int ftar_intra_launch(ftar_ctx* c, int op, const void* in, int in_dtype, float* out, uint64_t total,
                      const uint64_t* offs, const uint64_t* lens, void* stream) {
  if (!c) return fail(FTAR_ST_INVARIANT, "null ctx");
  int v = intra_check(op, in_dtype, c->n, total, offs, lens);
  if (v) return v;
  if (c->q_count == kQueue) return fail(FTAR_ST_INVARIANT, "queue full: wait for the oldest first");
  const uint64_t esz = in_dtype == FTAR_DT_BF16 ? 2 : 4;
  const uint64_t in_bytes = op == (int)kIntraRS ? total * esz : lens[c->self] * 4;
  if (in_bytes > c->max_bucket_bytes) return fail(FTAR_ST_INVARIANT, "input exceeds the group's staging capacity");
  const uint64_t out_elems = op == (int)kIntraRS ? lens[c->self] : total;
  if ((in_bytes && !in) || (out_elems && !out)) return fail(FTAR_ST_INVARIANT, "null buffer");
  DeviceGuard g(c->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  c->seq += 1;
  const uint64_t tag = mk_tag(c->gen, c->seq);
  const char* inp = static_cast<const char*>(in);
  uint64_t in_off;
  const bool registered = inp >= c->arena + c->pool_off && inp + in_bytes <= c->arena + c->arena_bytes;
  if (registered || c->n == 1) {
    in_off = (uint64_t)(inp - c->arena);
  } else {
    // peers can only address my arena: stage the input there (the closing
    // barrier keeps it alive until every peer has read it)
    const uint64_t so = c->stage_off[c->seq & 1];
    if (in_bytes) CK(cudaMemcpyAsync(c->arena + so, in, in_bytes, cudaMemcpyDeviceToDevice, st));
    in_off = so;
  }
  LaunchParams p{};
  intra_grid_params(p, op, in_dtype, total, offs, lens, c->n);
  for (int i = 0; i < c->n; ++i) p.base[i] = (i == c->self) ? c->arena : c->peer[c->ring_slots[i]];
  c->push(tag);
  p.ctl[c->self] = c->ctl_d;
  p.out[c->self] = out;
  p.in_off[c->self] = in_off;
  p.tag = tag;
  p.hard_timeout_ns = c->hard_timeout_ns;
  p.self = c->self;
  p.emulated = 0;
  p.fault_member = -1;
  const dim3 grid(intra_ctas(op, in_dtype, total, lens, c->self, c->n), 1);
  // staged inputs are written by a copy on this stream, which keeps the full
  // dependency; PDL only relaxes kernel-after-kernel
  cudaError_t e = in_dtype == FTAR_DT_BF16 ? launch_intra<BF16In>(c->n, p, grid, st, false, pdl_on())
                                            : launch_intra<F32In>(c->n, p, grid, st, false, pdl_on());
  if (e != cudaSuccess) {
    c->pop_last();
    return cuda_fail(e, "intra-replica collective launch");
  }
  return FTAR_OK;
}

int ftar_local_intra_launch(ftar_ctx** ctxs, int n, int op, const void* const* ins, int in_dtype, float* const* outs,
                            uint64_t total, const uint64_t* offs, const uint64_t* lens, void* stream) {
  int v = intra_check(op, in_dtype, n, total, offs, lens);
  if (v) return v;
  if (!ctxs || !ins || !outs) return fail(FTAR_ST_INVARIANT, "null arrays");
  const int dev = ctxs[0]->device;
  for (int i = 0; i < n; ++i) {
    ftar_ctx* c = ctxs[i];
    if (!c || c->device != dev) return fail(FTAR_ST_INVARIANT, "in-process ranks must share a device");
    if (c->q_count) return fail(FTAR_ST_INVARIANT, "in-process groups run one collective at a time");
    if (c->gen != ctxs[0]->gen || c->seq != ctxs[0]->seq)
      return fail(FTAR_ST_PROTOCOL, "ranks disagree on (generation, call sequence)");
    const uint64_t in_elems = op == (int)kIntraRS ? total : lens[i], out_elems = op == (int)kIntraRS ? lens[i] : total;
    if ((!ins[i] && in_elems) || (!outs[i] && out_elems)) return fail(FTAR_ST_INVARIANT, "null buffer");
  }
  DeviceGuard g(dev);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  LaunchParams p{};
  intra_grid_params(p, op, in_dtype, total, offs, lens, n);
  uint64_t tag = 0;
  for (int i = 0; i < n; ++i) {
    ftar_ctx* c = ctxs[i];
    c->seq += 1;
    tag = mk_tag(c->gen, c->seq);
    c->push(tag);
    p.base[i] = c->arena;
    p.ctl[i] = c->ctl_d;
    p.out[i] = outs[i];
    p.in_off[i] = (uint64_t)(static_cast<const char*>(ins[i]) - c->arena);  // same process: any address
  }
  p.tag = tag;
  p.hard_timeout_ns = ctxs[0]->hard_timeout_ns;
  p.self = 0;
  p.emulated = 1;
  p.fault_member = -1;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int G = intra_ctas(op, in_dtype, total, lens, 0, n);
  G = std::max(1, std::min(G, std::max(1, sms / n)));  // cooperative: every rank's CTAs co-resident
  const dim3 grid(G, n);
  cudaError_t e = in_dtype == FTAR_DT_BF16 ? launch_intra<BF16In>(n, p, grid, st, true)
                                            : launch_intra<F32In>(n, p, grid, st, true);
  if (e != cudaSuccess) {
    for (int i = 0; i < n; ++i) ctxs[i]->pop_last();
    return cuda_fail(e, "in-process intra-replica cooperative launch");
  }
  return FTAR_OK;
}

int ftar_abort(ftar_ctx* c) {
  if (!c) return fail(FTAR_ST_INVARIANT, "null ctx");
  for (int i = 0; i < c->q_count; ++i) {
    const int slot = (c->q_head + i) % kQueue;
    c->ctl_hs[slot].abort_tag = c->q_tag[slot];
  }
  return FTAR_OK;
}

int ftar_inflight(ftar_ctx* c) { return c ? c->q_count : 0; }

int ftar_wait(ftar_ctx* c, double progress_timeout_s, int* detail) {
  // Waits for the OLDEST queued collective (FIFO).  Its per-chunk deadline
  // starts when its kernel starts (queued work behind earlier buckets does
  // not count); no progress for progress_timeout_s -> abort word -> drain.
  if (!c) return fail(FTAR_ST_INVARIANT, "null ctx");
  if (detail) *detail = -1;
  if (!c->q_count) return FTAR_OK;
  const int slot = c->q_head;
  HostCtl* h = c->ctl_hs + slot;
  const uint64_t tag = c->q_tag[slot];
  uint64_t last_prog = ~0ull;
  double last_change = now_s();
  const double t_begin = last_change;
  bool aborted = false;
  double abort_t = 0;
  for (uint64_t it = 0;; ++it) {
    const uint64_t d = h->done;
    if (flag_tag(d) == tag) {
      c->q_head = (c->q_head + 1) % kQueue;
      --c->q_count;
      // the device writes `detail` (then fences) only for a failed call
      if (detail) *detail = (d & 0xff) ? (int)h->detail : -1;
      return (int)(d & 0xff);
    }
    const double t = now_s();
    if (h->started == tag) {
      const uint64_t pr = h->progress;
      if (pr != last_prog) {
        last_prog = pr;
        last_change = t;
      } else if (!aborted && t - last_change > progress_timeout_s) {
        // per-chunk deadline expired: drain this and every queued collective
        for (int i = 0; i < c->q_count; ++i) {
          const int sl = (c->q_head + i) % kQueue;
          c->ctl_hs[sl].abort_tag = c->q_tag[sl];
        }
        aborted = true;
        abort_t = t;
      }
    } else {
      last_change = t;  // still queued behind earlier stream work
    }
    if (aborted && t - abort_t > 60.0) {
      return fail(FTAR_ST_TIMEOUT, "kernel did not drain after abort");
    }
    host_backoff(it, t - t_begin);
  }
}

int ftar_wait_local(ftar_ctx** ctxs, int n, double progress_timeout_s, int* statuses, int* details) {
  // One watcher for all members of an in-process ring: every member's
  // progress word is tracked; a member whose progress stalls is aborted.
  if (!ctxs || n < 1) return fail(FTAR_ST_INVARIANT, "bad wait_local args");
  uint64_t last_prog[kMaxMembers];
  double last_change[kMaxMembers];
  bool aborted[kMaxMembers] = {};
  bool fin[kMaxMembers] = {};
  double t0 = now_s();
  const double t_begin = t0;
  for (int i = 0; i < n; ++i) {
    last_prog[i] = ~0ull;
    last_change[i] = t0;
    statuses[i] = FTAR_OK;
    if (details) details[i] = -1;
    fin[i] = ctxs[i]->q_count == 0;
  }
  double abort_t = 0;
  for (uint64_t it = 0;; ++it) {
    int left = 0;
    const double t = now_s();
    for (int i = 0; i < n; ++i) {
      if (fin[i]) continue;
      ftar_ctx* c = ctxs[i];
      const int slot = c->q_head;
      HostCtl* h = c->ctl_hs + slot;
      const uint64_t tag = c->q_tag[slot];
      const uint64_t d = h->done;
      if (flag_tag(d) == tag) {
        fin[i] = true;
        c->q_head = (c->q_head + 1) % kQueue;
        --c->q_count;
        statuses[i] = (int)(d & 0xff);
        if (details) details[i] = (d & 0xff) ? (int)h->detail : -1;
        continue;
      }
      ++left;
      if (h->started == tag) {
        const uint64_t pr = h->progress;
        if (pr != last_prog[i]) {
          last_prog[i] = pr;
          last_change[i] = t;
        } else if (!aborted[i] && t - last_change[i] > progress_timeout_s) {
          h->abort_tag = tag;
          aborted[i] = true;
          if (abort_t == 0) abort_t = t;
        }
      } else {
        last_change[i] = t;
      }
    }
    if (!left) return FTAR_OK;
    if (abort_t > 0 && t - abort_t > 60.0) return fail(FTAR_ST_TIMEOUT, "kernel did not drain after abort");
    host_backoff(it, t - t_begin);
  }
}

int ftar_phase_times(ftar_ctx* c, uint64_t* out, int n) {
  // the last completed call's %globaltimer stamps, kept in the arena header
  // (the kernels spend no PCIe writes on them); synchronises the device
  if (!c || !out) return fail(FTAR_ST_INVARIANT, "bad args");
  DeviceGuard g(c->device);
  uint64_t t[6];
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(t, c->arena + offsetof(ArenaHdr, tph), sizeof(t), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < 6; ++i) out[i] = t[i];
  return FTAR_OK;
}

int ftar_probe_pattern(float* c, const float* a, const float* b, uint64_t n, int mode, int layout, int unroll,
                       int ctas, int device, void* stream) {
  DeviceGuard dg(device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int g = std::max(1, ctas);
  switch (unroll) {
    case 1: probe_pattern_kernel<1><<<g, kThreads, 0, st>>>(c, a, b, n, mode, layout); break;
    case 2: probe_pattern_kernel<2><<<g, kThreads, 0, st>>>(c, a, b, n, mode, layout); break;
    case 4: probe_pattern_kernel<4><<<g, kThreads, 0, st>>>(c, a, b, n, mode, layout); break;
    case 8: probe_pattern_kernel<8><<<g, kThreads, 0, st>>>(c, a, b, n, mode, layout); break;
    default: return fail(FTAR_ST_INVARIANT, "unroll must be 1, 2, 4 or 8");
  }
  CK(cudaGetLastError());
  return FTAR_OK;
}

int ftar_debug_trace(ftar_ctx* c, uint64_t* out, int n) {
  // the diagnostic build's per-tile pipeline stamps of CTA 0 (last call)
  if (!c || !out) return fail(FTAR_ST_INVARIANT, "bad args");
  DeviceGuard g(c->device);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, c->arena + offsetof(ArenaHdr, dbg_trace), sizeof(uint64_t) * std::min(n, 512),
                cudaMemcpyDeviceToHost));
  return FTAR_OK;
}

int ftar_debug_cta_times(ftar_ctx* c, uint64_t* rs_end, uint64_t* ag_end, int n) {
  if (!c) return fail(FTAR_ST_INVARIANT, "null ctx");
  DeviceGuard g(c->device);
  ArenaHdr h;
  CK(cudaMemcpy(&h, c->arena, sizeof(h), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < 256; ++i) {
    rs_end[i] = h.dbg_rs_end[i];
    ag_end[i] = h.dbg_ag_end[i];
  }
  if (n >= 260) {  // caller wants the fence stamps too (rs_end[256..259])
    for (int i = 0; i < 4; ++i) rs_end[256 + i] = h.dbg_fence[i];
  }
  return FTAR_OK;
}

// Clock pairing for cross-GPU timelines (diagnostic): a one-thread kernel
// writes %globaltimer into pinned host memory while the host spins on it and
// stamps CLOCK_MONOTONIC the moment it appears.  host - gpu, minimised over
// `reps`, is this GPU's timer offset to the host clock that every process on
// the box shares (error ~ one PCIe write latency).
__global__ void probe_clock_kernel(volatile uint64_t* slot) { *slot = globaltimer_ns(); }

int ftar_probe_clock(int device, int reps, int64_t* offset_ns) {
  if (!offset_ns || reps < 1) return fail(FTAR_ST_INVARIANT, "bad args");
  DeviceGuard g(device);
  uint64_t* h = nullptr;
  CK(cudaHostAlloc(reinterpret_cast<void**>(&h), sizeof(uint64_t), cudaHostAllocMapped));
  uint64_t* d = nullptr;
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), h, 0);
  int64_t best = INT64_MAX;
  for (int r = 0; r < reps; ++r) {
    *reinterpret_cast<volatile uint64_t*>(h) = 0;
    probe_clock_kernel<<<1, 1>>>(d);
    uint64_t v;
    while ((v = *reinterpret_cast<volatile uint64_t*>(h)) == 0) {
    }
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    const int64_t host = (int64_t)ts.tv_sec * 1000000000ll + ts.tv_nsec;
    best = std::min(best, host - (int64_t)v);
    cudaDeviceSynchronize();
  }
  cudaFreeHost(h);
  *offset_ns = best;
  return FTAR_OK;
}

int ftar_probe_fence(float* c, const float* a, const float* b, uint64_t n, int kind, int ctas, uint64_t* stamps,
                     int device, void* stream) {
  DeviceGuard dg(device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int g = std::max(1, ctas);
  if (kind == 0) probe_fence_kernel<0><<<g, kThreads, 0, st>>>(c, a, b, n, stamps);
  else if (kind == 1) probe_fence_kernel<1><<<g, kThreads, 0, st>>>(c, a, b, n, stamps);
  else probe_fence_kernel<2><<<g, kThreads, 0, st>>>(c, a, b, n, stamps);
  CK(cudaGetLastError());
  return FTAR_OK;
}

int ftar_probe_copy(void* dst, const void* src, uint64_t bytes, int ctas, void* stream) {
  probe_copy_kernel<<<std::max(1, ctas), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<char*>(dst), static_cast<const char*>(src), bytes);
  CK(cudaGetLastError());
  return FTAR_OK;
}

int ftar_probe_bulk(void* dst, const void* src, uint64_t bytes, int ctas, int tile, int stages, void* stream) {
  if (tile < 16 || (tile & 15) || stages < 2 || (uint64_t)tile * stages + 1024 > 227 * 1024)
    return fail(FTAR_ST_INVARIANT, "bad bulk probe shape");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t sm = 1024 + (size_t)tile * stages;
  const int g = std::max(1, ctas);
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
#define BULK_CASE(K)                                                                           \
  case K:                                                                                      \
    CK(cudaFuncSetAttribute(probe_bulk_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                            (int)sm));                                                         \
    probe_bulk_kernel<K><<<g, 32, sm, st>>>(d, s, bytes, (uint32_t)tile);                      \
    break;
  switch (stages) {
    BULK_CASE(2) BULK_CASE(4) BULK_CASE(6) BULK_CASE(8) BULK_CASE(12) BULK_CASE(16)
    default: return fail(FTAR_ST_INVARIANT, "stages must be 2, 4, 6, 8, 12 or 16");
  }
#undef BULK_CASE
  CK(cudaGetLastError());
  return FTAR_OK;
}

int ftar_peer_enable(int device, int peer) {
  DeviceGuard g(device);
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return FTAR_OK;
  }
  CK(e);
  return FTAR_OK;
}

// ------------------------------------------------------------------ operators
int ftar_accumulate(float* dst, const void* src, int src_dtype, uint64_t n, void* stream) {
  if (!n) return FTAR_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = (int)std::min<uint64_t>((n + 255) / 256, 148ull * 8);
  if (src_dtype == FTAR_DT_BF16)
    accumulate_kernel<BF16In><<<blocks, 256, 0, st>>>(dst, static_cast<const __nv_bfloat16*>(src), n);
  else if (src_dtype == FTAR_DT_F32)
    accumulate_kernel<F32In><<<blocks, 256, 0, st>>>(dst, static_cast<const float*>(src), n);
  else
    return fail(FTAR_ST_INVARIANT, "bad dtype");
  CK(cudaGetLastError());
  return FTAR_OK;
}

int ftar_copy_into(float* dst, const void* src, int src_dtype, uint64_t n, void* stream) {
  if (!n) return FTAR_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int blocks = (int)std::min<uint64_t>((n + 255) / 256, 148ull * 8);
  if (src_dtype == FTAR_DT_BF16)
    copy_into_kernel<BF16In><<<blocks, 256, 0, st>>>(dst, static_cast<const __nv_bfloat16*>(src), n);
  else if (src_dtype == FTAR_DT_F32)
    copy_into_kernel<F32In><<<blocks, 256, 0, st>>>(dst, static_cast<const float*>(src), n);
  else
    return fail(FTAR_ST_INVARIANT, "bad dtype");
  CK(cudaGetLastError());
  return FTAR_OK;
}

// ------------------------------------------------------------------ catch-up
int ftar_snap_create(int device, uint64_t capacity_bytes, int exportable, ftar_snap** out) {
  (void)exportable;
  if (!out) return fail(FTAR_ST_INVARIANT, "null out");
  DeviceGuard g(device);
  ftar_snap* s = new ftar_snap();
  s->device = device;
  s->cap = align_up(std::max<uint64_t>(capacity_bytes, 16), 256);
  cudaError_t e = cudaMalloc(&s->arena, kSnapHdrBytes + s->cap);
  if (e != cudaSuccess) {
    delete s;
    return cuda_fail(e, "cudaMalloc(snapshot)");
  }
  snap_init_kernel<<<1, 1>>>(reinterpret_cast<SnapHdr*>(s->arena));
  {  // load the catch-up kernels now (see warm_ring_kernels): a recovering
     // replica's first pull must not load modules while the ring runs
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, snap_pull_kernel);
    cudaFuncGetAttributes(&a, snap_pull_reset_kernel);
    cudaFuncGetAttributes(&a, snap_copy_kernel);
    cudaFuncGetAttributes(&a, snap_mark_kernel);
    cudaFuncSetAttribute(snap_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPullSmem);
    cudaGetLastError();
  }
  e = cudaHostAlloc(&s->ctl_h, sizeof(HostCtl), cudaHostAllocMapped | cudaHostAllocPortable);
  if (e != cudaSuccess) return cuda_fail(e, "cudaHostAlloc(snap ctl)");
  std::memset((void*)s->ctl_h, 0, sizeof(HostCtl));
  reset_ctl(s->ctl_h);
  cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->ctl_d), (void*)s->ctl_h, 0);
  CK(cudaDeviceSynchronize());
  *out = s;
  return FTAR_OK;
}

int ftar_snap_destroy(ftar_snap* s) {
  if (!s) return FTAR_OK;
  DeviceGuard g(s->device);
  cudaDeviceSynchronize();
  for (int i = 0; i < kMaxSlots; ++i)
    if (s->peer[i]) cudaIpcCloseMemHandle(s->peer[i]);
  if (s->reset_done) cudaEventDestroy(s->reset_done);
  cudaFree(s->arena);
  cudaFreeHost((void*)s->ctl_h);
  delete s;
  return FTAR_OK;
}

int ftar_snap_export(ftar_snap* s, void* buf, size_t buflen, size_t* written) {
  if (!s || !buf || buflen < sizeof(cudaIpcMemHandle_t)) return fail(FTAR_ST_INVARIANT, "bad export args");
  DeviceGuard g(s->device);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, s->arena));
  std::memcpy(buf, &h, sizeof(h));
  if (written) *written = sizeof(h);
  return FTAR_OK;
}

int ftar_snap_capture(ftar_snap* s, uint64_t step, const void* params, uint64_t pbytes,
                      const void* momentum, uint64_t mbytes, void* stream) {
  if (!s) return fail(FTAR_ST_INVARIANT, "null snapshot");
  if (pbytes + mbytes > s->cap) return fail(FTAR_ST_INVARIANT, "snapshot exceeds capacity");
  DeviceGuard g(s->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SnapHdr* h = reinterpret_cast<SnapHdr*>(s->arena);
  snap_mark_kernel<<<1, 1, 0, st>>>(h, (int64_t)step, pbytes, mbytes, 1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
  const uint64_t total = pbytes + mbytes;
  const int blocks = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * 2, (total + 65535) / 65536));
  if (total)
    snap_copy_kernel<<<blocks, kThreads, 0, st>>>(s->arena + kSnapHdrBytes, static_cast<const char*>(params),
                                                  pbytes, static_cast<const char*>(momentum), mbytes);
  snap_mark_kernel<<<1, 1, 0, st>>>(h, (int64_t)step, pbytes, mbytes, 0);
  CK(cudaGetLastError());
  return FTAR_OK;
}

int ftar_snap_info(ftar_snap* s, int64_t* step, uint64_t* pbytes, uint64_t* mbytes) {
  if (!s) return fail(FTAR_ST_INVARIANT, "null snapshot");
  DeviceGuard g(s->device);
  SnapHdr h;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, s->arena, sizeof(h), cudaMemcpyDeviceToHost));
  if (step) *step = (h.seq & 1u) ? -1 : h.step;
  if (pbytes) *pbytes = h.pbytes;
  if (mbytes) *mbytes = h.mbytes;
  return FTAR_OK;
}

int ftar_snap_region(ftar_snap* s, void** params, void** momentum, uint64_t* pbytes, uint64_t* mbytes,
                     uint64_t* seq, int64_t* step) {
  // §8f rank 4: where the retention-1 snapshot lives, and its seqlock word,
  // for a host-side writer streaming it to storage.  A writer reads `seq`
  // before and after copying: an odd or changed value means a capture ran in
  // between and the copy is torn.  Synchronises the device.
  if (!s) return fail(FTAR_ST_INVARIANT, "null snapshot");
  DeviceGuard g(s->device);
  SnapHdr h;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(&h, s->arena, sizeof(h), cudaMemcpyDeviceToHost));
  if (params) *params = s->arena + kSnapHdrBytes;
  if (momentum) *momentum = s->arena + kSnapHdrBytes + h.pbytes;
  if (pbytes) *pbytes = h.pbytes;
  if (mbytes) *mbytes = h.mbytes;
  if (seq) *seq = h.seq;
  if (step) *step = (h.seq & 1u) ? -1 : h.step;
  return FTAR_OK;
}

int ftar_snap_import(ftar_snap* s, int slot, const void* handle, size_t len, uint64_t capacity_bytes) {
  (void)capacity_bytes;
  if (!s || slot < 0 || slot >= kMaxSlots || !handle || len < sizeof(cudaIpcMemHandle_t))
    return fail(FTAR_ST_INVARIANT, "bad import args");
  DeviceGuard g(s->device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  if (s->peer[slot]) {
    if (std::memcmp(&s->peer_handle[slot], &h, sizeof(h)) == 0) return FTAR_OK;
    return fail(FTAR_ST_INVARIANT, "snapshot slot " + std::to_string(slot) + " maps a different donor (unmap it first)");
  }
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    g_err = std::string("cudaIpcOpenMemHandle(snapshot): ") + cudaGetErrorString(e);
    return FTAR_ST_PEER_DOWN;
  }
  s->peer[slot] = static_cast<char*>(p);
  s->peer_handle[slot] = h;
  return FTAR_OK;
}

int ftar_snap_unmap(ftar_snap* s, int slot) {
  if (!s || slot < 0 || slot >= kMaxSlots) return fail(FTAR_ST_INVARIANT, "bad unmap args");
  if (s->inflight && flag_tag(s->ctl_h->done) != s->cur_tag)
    return fail(FTAR_ST_INVARIANT, "unmap with a pull in flight");
  DeviceGuard g(s->device);
  if (s->peer[slot]) {
    cudaIpcCloseMemHandle(s->peer[slot]);
    s->peer[slot] = nullptr;
    std::memset(&s->peer_handle[slot], 0, sizeof(cudaIpcMemHandle_t));
  }
  return FTAR_OK;
}

int ftar_snap_peer_info(ftar_snap* s, int slot, int64_t* step, uint64_t* pbytes, uint64_t* mbytes) {
  // the donor's snapshot header read over NVLink (a 32-byte peer copy): what
  // step it holds (-1: nothing, or a capture in progress) and its lengths
  if (!s || slot < 0 || slot >= kMaxSlots || !s->peer[slot]) return fail(FTAR_ST_INVARIANT, "donor not mapped");
  DeviceGuard g(s->device);
  SnapHdr h;
  CK(cudaMemcpy(&h, s->peer[slot], 32, cudaMemcpyDefault));
  if (step) *step = (h.seq & 1u) ? -1 : h.step;
  if (pbytes) *pbytes = h.pbytes;
  if (mbytes) *mbytes = h.mbytes;
  return FTAR_OK;
}

int ftar_snap_pull_multi_launch(ftar_snap* local, const int* slots, int nslots, const ftar_snap* src_local,
                                uint64_t want_step, void* dst_params, uint64_t pbytes, void* dst_momentum,
                                uint64_t mbytes, int ctas, void* stream) {
  if (!local) return fail(FTAR_ST_INVARIANT, "null snapshot");
  if (local->inflight && flag_tag(local->ctl_h->done) != local->cur_tag)
    return fail(FTAR_ST_INVARIANT, "one pull in flight per snapshot context");
  PullSrcs src{};
  if (nslots > 0) {
    if (nslots > kMaxMembers) return fail(FTAR_ST_INVARIANT, "too many donors");
    for (int i = 0; i < nslots; ++i) {
      const int slot = slots[i];
      if (slot < 0 || slot >= kMaxSlots || !local->peer[slot]) return fail(FTAR_ST_INVARIANT, "donor not mapped");
      src.arena[i] = local->peer[slot];
    }
    src.n = nslots;
  } else {
    if (!src_local) return fail(FTAR_ST_INVARIANT, "no donor");
    src.arena[0] = src_local->arena;
    src.n = 1;
  }
  DeviceGuard g(local->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  local->seq += 1;
  const uint64_t tag = mk_tag(0, local->seq);
  reset_ctl(local->ctl_h);
  local->cur_tag = tag;
  local->inflight = true;
  const int G = std::max(1, ctas);
  snap_pull_reset_kernel<<<1, 1, 0, st>>>(reinterpret_cast<SnapHdr*>(local->arena));
  if (!local->reset_done) CK(cudaEventCreateWithFlags(&local->reset_done, cudaEventDisableTiming));
  CK(cudaEventRecord(local->reset_done, st));
  // the bulk-copy pull when every region is 16-byte aligned (FTAR_TMA=0: register copy)
  const int bulk = tma_on() && (pbytes % 16 == 0) && (mbytes % 16 == 0) &&
                   ((reinterpret_cast<uint64_t>(dst_params) | reinterpret_cast<uint64_t>(dst_momentum)) % 16 == 0);
  if (bulk) {
    static bool attr_set[64] = {};
    const int dev = local->device;
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      CK(cudaFuncSetAttribute(snap_pull_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPullSmem));
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
  }
  snap_pull_kernel<<<G, kThreads, bulk ? kPullSmem : 0, st>>>(
      src, reinterpret_cast<SnapHdr*>(local->arena), local->ctl_d, tag, (int64_t)want_step,
      static_cast<char*>(dst_params), pbytes, static_cast<char*>(dst_momentum), mbytes, bulk);
  local->last = {src, (int64_t)want_step, static_cast<char*>(dst_params), pbytes, static_cast<char*>(dst_momentum),
                 mbytes, bulk};
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    local->inflight = false;
    return cuda_fail(e, "snapshot pull launch");
  }
  return FTAR_OK;
}

int ftar_snap_pull_boost(ftar_snap* local, int ctas, void* stream) {
  // A second grid for the pull in flight, on another stream: its CTAs claim
  // chunks from the same counter, so the remaining transfer widens at once.
  // A no-op when the pull already finished.
  if (!local) return fail(FTAR_ST_INVARIANT, "null snapshot");
  if (!local->inflight || flag_tag(local->ctl_h->done) == local->cur_tag) return FTAR_OK;
  DeviceGuard g(local->device);
  const PullArgs& a = local->last;
  CK(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), local->reset_done, 0));  // not on the first grid
  snap_pull_kernel<<<std::max(1, ctas), kThreads, a.bulk ? kPullSmem : 0, static_cast<cudaStream_t>(stream)>>>(
      a.src, reinterpret_cast<SnapHdr*>(local->arena), local->ctl_d, local->cur_tag, a.want, a.dp, a.pb, a.dm, a.mb,
      a.bulk);
  CK(cudaGetLastError());
  return FTAR_OK;
}

int ftar_snap_pull_launch(ftar_snap* local, int slot, const ftar_snap* src_local, uint64_t want_step,
                          void* dst_params, uint64_t pbytes, void* dst_momentum, uint64_t mbytes, int ctas,
                          void* stream) {
  return ftar_snap_pull_multi_launch(local, &slot, slot >= 0 ? 1 : 0, src_local, want_step, dst_params, pbytes,
                                     dst_momentum, mbytes, ctas, stream);
}

int ftar_snap_poll(ftar_snap* s, int* status, uint64_t* progress, int64_t* available) {
  if (!s) return fail(FTAR_ST_INVARIANT, "null snapshot");
  const uint64_t d = s->ctl_h->done;
  if (progress) *progress = s->ctl_h->progress;
  if (available) *available = s->ctl_h->available;
  if (status) *status = (s->inflight && flag_tag(d) == s->cur_tag) ? (int)(d & 0xff)
                       : (s->inflight ? FTAR_ST_PENDING : FTAR_OK);
  return FTAR_OK;
}

int ftar_snap_abort(ftar_snap* s) {
  if (!s) return fail(FTAR_ST_INVARIANT, "null snapshot");
  s->ctl_h->abort_tag = s->cur_tag;
  return FTAR_OK;
}

int ftar_snap_wait(ftar_snap* s, double progress_timeout_s, int64_t* available) {
  if (!s) return fail(FTAR_ST_INVARIANT, "null snapshot");
  if (!s->inflight) return FTAR_OK;
  HostCtl* h = s->ctl_h;
  const uint64_t tag = s->cur_tag;
  uint64_t last = ~0ull;
  double last_change = now_s();
  const double t_begin = last_change;
  bool aborted = false;
  double abort_t = 0;
  for (uint64_t it = 0;; ++it) {
    const uint64_t d = h->done;
    if (flag_tag(d) == tag) {
      s->inflight = false;
      if (available) *available = h->available;
      return (int)(d & 0xff);
    }
    const double t = now_s();
    if (h->started == tag) {
      const uint64_t pr = h->progress;
      if (pr != last) {
        last = pr;
        last_change = t;
      } else if (!aborted && t - last_change > progress_timeout_s) {
        h->abort_tag = tag;
        aborted = true;
        abort_t = t;
      }
    } else {
      last_change = t;
    }
    if (aborted && t - abort_t > 60.0) return fail(FTAR_ST_TIMEOUT, "pull did not drain after abort");
    host_backoff(it, t - t_begin);
  }
}

}  // extern "C"
