// Device-side data structures and primitives of the B200 NVRAR all-reduce.
//
// Transport model (replaces the reference's one-sided Ctx, transport.hpp:137-202):
//  * every rank owns ONE symmetric region (same layout on all ranks, mapped
//    into each peer process through CUDA IPC) — the analogue of
//    Ctx::alloc_region's symmetric regions;
//  * slots are arrays of 16-byte cells. A cell is EMPTY when all its bits are
//    ones; the region starts empty and every reader re-empties what it read,
//    so the invariant holds between calls whatever protocol used the slot;
//  * two wire protocols, both self-validating (arrival of data is arrival of
//    its signal — no fence, no per-pair ordering assumption; NVLink does not
//    order weak stores to different addresses, unlike the reference
//    transport, transport.hpp:9-11):
//      LL      — the reference's fused word (transport.hpp:81-87, fused.hpp:4-8):
//                8 bytes = 4-byte payload (low) + 4-byte sequence flag (high);
//                eta = 2. Used for int32 (no spare bit pattern) and on request.
//      Lamport — raw payload (eta = 1); the all-ones pattern (a NaN in fp32
//                and bf16) means "not arrived", writers map that one NaN
//                pattern to another NaN. Default for fp32 / bf16.
//    Both are double-buffered by call parity (nvrar.hpp:107-109,124-126).
//  * sequence/length words (seq<<32 | len) published into the peer's counter
//    array stand in for Ctx::publish_counter (transport.hpp:161-164), and the
//    wait on them is the reference's peer-only sync (nvrar.hpp:163-171).
#pragma once

#include <cstdint>

namespace nvrar {

constexpr int kMaxRanks = 64;   // NVRAR_MAX_RANKS
constexpr int kCtrlWords = 3 * kMaxRanks;  // counters, diag (+pad), done
constexpr int kMaxLocal = 32;   // NVRAR_MAX_LOCAL (virtual ranks per launch)
constexpr int kThreads = 512;   // threads per CTA
constexpr int kDirectThreads = 256;  // direct schedule (no waits; several CTAs per SM)

enum Status : uint32_t {
  kOk = 0,
  kInternal = 1,
  kInvalidArgument = 2,
  kInvalidTopology = 3,
  kProtocolFault = 4,
  kDeadlock = 5,
};

enum WaitKind : int32_t { kFlagWait = 0, kSeqWait = 1, kLenMismatch = 2, kStaleFlag = 3 };

// Byte offsets inside the symmetric region; identical on every rank.
struct Layout {
  uint64_t ctrl_off;  // control words, kCtrlWords u64: counters[kMaxRanks] ((seq<<32)|len
                      // from rank p), the ping-pong diag word, done[kMaxRanks]
  uint64_t a_off;     // A slots: [2 parity][P src][a_src words]  (RS / one-shot inputs)
  uint64_t a_src;     // words (8 B) per source slot
  uint64_t b_off;     // B slots: [2][P][b_src]                    (all-gather)
  uint64_t b_src;
  uint64_t c_off;     // C slots: [2][steps][c_step]               (recursive doubling)
  uint64_t c_step;
  uint64_t bytes;     // total
};

struct ErrRec {
  uint32_t code;      // Status
  int32_t kind;       // WaitKind
  int32_t peer;       // global rank awaited
  uint32_t expected;  // awaited sequence number
  uint64_t word;      // unit index inside the awaited slot (FlagWait)
  uint64_t observed;  // what was seen instead
  int32_t phase;      // kernel phase of the wait (2 RS/push, 3 sync, 4 reduce/RD, 5 AG)
  int32_t cta;        // CTA that recorded it
};

// Private (not shared) per-rank state. seq is the NvrarAllreduce::seq_ analogue
// (nvrar.hpp:248): the kernel reads seq+1 as its call number and stores it
// back on exit, so the counter stays on the device and a CUDA graph of
// back-to-back calls needs no host involvement.
constexpr int kSeqSlots = 512;  // >= co-resident CTAs of one launch
constexpr int kPhases = 8;

// seq is replicated in kSeqSlots slots: CTA b reads slot b at entry and, on
// exit, writes slots b, b+grid, b+2*grid, ... — so every slot advances on every
// call whatever the grid size, without atomics or a grid-wide barrier.
struct RankState {
  uint32_t seq[kSeqSlots];
  ErrRec err;
  uint32_t arrive;  // CTAs of the current registered-buffer launch that finished reading
  uint64_t ts[kSeqSlots][kPhases];  // per-CTA phase timestamps, thread 0 (profiling)
};

struct RankDesc {
  uint8_t* base[kMaxRanks];  // every rank's symmetric region, as mapped here
  RankState* state;          // own
  Layout lay;
  int rank, world, nodes, gpus, steps, node, local;
  int profile;
  uint32_t poll_ns;  // back-off between unsatisfied polls (0 = spin)
  uint64_t timeout_ns;
  // NVLS multicast A area (one-shot over multicast): the multicast mapping
  // (stores reach every rank's copy) and this rank's own copy; same
  // [2 parity][P src][a_src words] shape as the region's A slots. Null when
  // multicast is not set up.
  uint8_t* mc;
  uint8_t* mc_local;
  // Delay injection (nvrar_set_jitter; the GPU counterpart of the reference's
  // RunOptions::delay_max_us, concurrent_transport.hpp:393-419): when
  // jitter_ns > 0 every CTA warp sleeps a seeded pseudo-random 0..jitter_ns ns
  // before its remote stores and between unsatisfied polls. 0 = off.
  uint32_t jitter_ns;
  uint32_t jitter_seed;
};

// One rank per launch (the real multi-GPU path) passes its descriptor BY VALUE
// (__grid_constant__ param space: no dependent global loads in the prologue);
// virtual ranks sharing a device (EMU) go through the pointer table.
struct LaunchParams {
  RankDesc d0;
  const RankDesc* desc[kMaxLocal];
  const void* send[kMaxLocal];
  void* recv[kMaxLocal];
  uint64_t count;
  int oneshot;  // flat kernel: 1 = one-shot ownership, 0 = two-shot
  int nlocal;
  int order;    // flat kernel: reduction order, kOrderNvrar / kOrderRing / kOrderTree
  uint8_t perm[64];  // ring order: global rank at ring position p (ring.hpp:27-30)
  // fused residual epilogue (nvrar_allreduce_residual): recv = resid + sum,
  // with the element type's own add (bf16: fp32 add of the rounded sum, one
  // RNE) — bit-identical to the all-reduce followed by `resid + out`
  const void* resid[kMaxLocal];
  int mc;  // flat one-shot: push each unit once through the multicast mapping
  // Window of a longer vector (the pipelined host-buffer path): this launch
  // reduces elements [e_off, e_off + count) of a vector of n_order elements, so
  // the reduction ORDER (shard index c = e / ceil(n/G)) follows the whole
  // vector and the bits equal one all-reduce of all n_order elements.
  // n_order = 0: the launch is the whole vector. Flat and direct kernels only.
  uint64_t e_off;
  uint64_t n_order;
  // Schedule variants (bit flags, kFlag*): where the call counter is written
  // back and where the flat schedules check the peers' lengths.
  int flags;
};

// kFlagEarlySeq: each CTA writes its call-counter slots right after reading
//   its own (nothing in this launch reads them again; the next launch reads
//   them after griddepcontrol.wait), taking those stores off the kernel tail.
// kFlagLazyLen: the flat schedules (one rank per launch) do not wait for the
//   peers' (seq, len) words before reducing; the length check runs at the end
//   of the call — before it completes, so a mismatch still faults the call
//   (sticky: later launches return at entry) — and a wait on a shorter peer's
//   missing data is diagnosed as the length mismatch it is.
// kFlagL2Fetch256: the direct schedule's input loads carry the .L2::256B
//   prefetch-size hint (set for pinned host inputs read over PCIe).
// kFlagSeqBarrier: thread 0 alone reads the call number and a __syncthreads
//   broadcasts it (the round-1 prologue; default: every thread reads it).
// kFlagDirectStream: the direct schedule stores its outputs evict-first
//   (st.global.cs) — an A/B knob.
enum : int {
  kFlagEarlySeq = 1,
  kFlagLazyLen = 2,
  kFlagL2Fetch256 = 4,
  kFlagSeqBarrier = 8,
  kFlagDirectStream = 16
};

// Reduction orders the flat kernel evaluates (the reference's three collectives):
//   NVRAR — ring fold of the node's ranks per G-chunk, pairwise tree over nodes;
//   RING  — ring fold of ALL ranks in ring positions per P-chunk (ring.hpp);
//   TREE  — chain fold in[0] + (in[1] + (... + in[G-1])) per node, pairwise
//           tree over nodes (tree.hpp:10-12).
enum : int { kOrderNvrar = 0, kOrderRing = 1, kOrderTree = 2 };

// ---------------------------------------------------------------------------
// PTX primitives

// Branch-layout hints: the hot path of a call (aligned full units, no residual,
// no injected delay, no fault) is laid out contiguously, the rare cases out of
// the way — the instruction fetch at the start of every call is part of the
// small-message latency (profiles/r02_summary.md §3).
#define NVRAR_LIKELY(x) __builtin_expect(!!(x), 1)
#define NVRAR_UNLIKELY(x) __builtin_expect(!!(x), 0)

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Data-path accesses carry no "memory" clobber: cells are self-validating, so
// no ordering against unrelated loads/stores is needed, and leaving the
// compiler free to hoist the next unit's input loads above this unit's remote
// stores is what keeps several HBM loads in flight per thread. (asm volatile
// statements still keep their order among themselves: read-then-empty of a
// cell stays in program order. pdl_wait keeps its clobber.)
#ifndef NVRAR_POLL_LD
#define NVRAR_POLL_LD "ld.volatile.global.v4.u32"
#endif
__device__ __forceinline__ uint4 ld_volatile16(const void* p) {
  uint4 v;
  asm volatile(NVRAR_POLL_LD " {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

#ifndef NVRAR_PUT_ST
#define NVRAR_PUT_ST "st.volatile.global.v4.u32"
#endif
// One 16-byte store to a multicast (NVLS) address: the NVSwitch replicates it
// into every member GPU's copy of the line. The payload is raw bits.
__device__ __forceinline__ void st_mc16(void* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p),
               "f"(__uint_as_float(a)), "f"(__uint_as_float(b)), "f"(__uint_as_float(c)),
               "f"(__uint_as_float(d))
               : "memory");
}

__device__ __forceinline__ void st_volatile16(void* p, uint32_t a, uint32_t b, uint32_t c,
                                              uint32_t d) {
  asm volatile(NVRAR_PUT_ST " [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d));
}

// 16-byte read-only load with a 256-byte L2 fetch-size hint (aligned unit)
__device__ __forceinline__ uint4 ld_l2_256(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint64_t ld_volatile64(const void* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void st_volatile64(void* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}

__device__ __forceinline__ uint32_t ld_volatile32(const void* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// ---------------------------------------------------------------------------
// Per-thread wait control: watchdog (DeadlockError analogue, errors.hpp:61-85)
// and fault recording. Once a thread aborts it keeps walking the same control
// flow (so every __syncthreads is still reached) but stops waiting.

struct Ctl {
  RankState* st;
  uint64_t timeout_ns;
  uint32_t poll_ns;
  uint32_t jitter_ns, jitter_seed;
  uint32_t seq;
  uint32_t spins;
  uint64_t t0;
  bool aborted;
  int phase;
  bool last_chance;
  // kFlagLazyLen: this rank's counters (peer p's (seq<<32)|len at [p]) and
  // the call's length, consulted when a data wait stalls
  const uint64_t* len_words;
  uint32_t len;
};

// The fault and watchdog paths are out of line (__noinline__): they are cold,
// and inlined at every poll site they made the kernels several times larger —
// the hot path then spread over more instruction-cache lines (no_instruction
// stalls dominated the one-shot's profile, profiles/r02_ncu_nvlink_p2.json).
// Poll sites holding a large register tile (16 sources) keep them inline
// (kOutline = false): a call there makes the caller save the tile.
__device__ __forceinline__ void record_fault_body(RankState* st, uint32_t code, int kind, int peer,
                                                  uint32_t seq, uint64_t word, uint64_t observed,
                                                  int phase) {
  ErrRec* e = &st->err;
  if (atomicCAS(&e->code, 0u, 0xFFFFFFFFu) == 0u) {
    e->kind = kind;
    e->peer = peer;
    e->expected = seq;
    e->word = word;
    e->observed = observed;
    e->phase = phase;
    e->cta = static_cast<int32_t>(blockIdx.x);
    __threadfence();
    atomicExch(&e->code, code);
  }
}
static __device__ __noinline__ void record_fault_at(RankState* st, uint32_t code, int kind,
                                                    int peer, uint32_t seq, uint64_t word,
                                                    uint64_t observed, int phase) {
  record_fault_body(st, code, kind, peer, seq, word, observed, phase);
}

template <bool kOutline = true>
__device__ __forceinline__ void record_fault(Ctl& c, uint32_t code, int kind, int peer,
                                             uint64_t word, uint64_t observed) {
  if constexpr (kOutline) {
    record_fault_at(c.st, code, kind, peer, c.seq, word, observed, c.phase);
  } else {
    record_fault_body(c.st, code, kind, peer, c.seq, word, observed, c.phase);
  }
  c.aborted = true;
}

// The watchdog's periodic check: 0 = keep waiting, 1 = give up (a fault is
// recorded, here or by another thread), 2 = the deadline passed once (poll one
// more full round before declaring a deadlock: a thread can be descheduled
// between its poll and this check).
__device__ __forceinline__ int wait_check_body(RankState* st, uint64_t t0, uint64_t timeout_ns,
                                               int last_chance, const uint64_t* len_words,
                                               uint32_t len, uint32_t spins, uint32_t seq,
                                               int phase, int kind, int peer, uint64_t word,
                                               uint64_t observed) {
  if (ld_volatile32(&st->err.code) != 0u) return 1;
  if (len_words != nullptr && kind == kFlagWait && peer >= 0 && (spins & 4095u) == 0u) {
    // a data wait that lasts: is the peer in this call with another length?
    const uint64_t v = ld_volatile64(len_words + peer);
    if (static_cast<uint32_t>(v >> 32) == seq && static_cast<uint32_t>(v) != len) {
      record_fault_body(st, kProtocolFault, kLenMismatch, peer, seq, 0, v, phase);
      return 1;
    }
  }
  if (globaltimer() - t0 > timeout_ns) {
    if (!last_chance) return 2;
    record_fault_body(st, kDeadlock, kind, peer, seq, word, observed, phase);
    return 1;
  }
  return 0;
}
static __device__ __noinline__ int wait_check(RankState* st, uint64_t t0, uint64_t timeout_ns,
                                              int last_chance, const uint64_t* len_words,
                                              uint32_t len, uint32_t spins, uint32_t seq,
                                              int phase, int kind, int peer, uint64_t word,
                                              uint64_t observed) {
  return wait_check_body(st, t0, timeout_ns, last_chance, len_words, len, spins, seq, phase, kind,
                         peer, word, observed);
}

// Called while a wait is unsatisfied. Returns true when the thread must give up.
template <bool kOutline = true>
__device__ __forceinline__ bool wait_tick(Ctl& c, int kind, int peer, uint64_t word,
                                          uint64_t observed) {
  if (NVRAR_UNLIKELY(c.aborted)) return true;
  if (NVRAR_LIKELY((++c.spins & 127u) != 0u)) return false;
  int r;
  if constexpr (kOutline) {
    r = wait_check(c.st, c.t0, c.timeout_ns, c.last_chance ? 1 : 0, c.len_words, c.len, c.spins,
                   c.seq, c.phase, kind, peer, word, observed);
  } else {
    r = wait_check_body(c.st, c.t0, c.timeout_ns, c.last_chance ? 1 : 0, c.len_words, c.len,
                        c.spins, c.seq, c.phase, kind, peer, word, observed);
  }
  if (r == 1) {
    c.aborted = true;
    return true;
  }
  if (r == 2) {
    c.last_chance = true;
    c.spins |= 127u;
  }
  return false;
}

// Back-off between unsatisfied polling rounds. It is also the yield point that
// lets the other diverged lane groups of the warp run: a tight spin without it
// was observed to starve lanes whose data had already arrived (independent
// thread scheduling does not rotate diverged groups often enough).
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}

static __device__ __noinline__ void jitter_sleep(uint32_t seed, uint32_t key, uint32_t max_ns) {
  __nanosleep(mix32(seed ^ mix32(key)) % max_ns);
}

template <bool kOutline = true>
__device__ __forceinline__ void poll_pause(const Ctl& c) {
  __nanosleep(c.poll_ns ? c.poll_ns : 32u);
  if (NVRAR_UNLIKELY(c.jitter_ns != 0)) {
    const uint32_t key = c.spins * 0x9E3779B9u ^ threadIdx.x ^ (blockIdx.x << 16);
    if constexpr (kOutline) {
      jitter_sleep(c.jitter_seed, key, c.jitter_ns);
    } else {
      __nanosleep(mix32(c.jitter_seed ^ mix32(key)) % c.jitter_ns);
    }
  }
}

// Injected delay at a program point (`site`) of call `seq`: the same for a
// whole warp (per CTA, warp, unit group and site), different per seed.
__device__ __forceinline__ void jitter(const Ctl& c, uint32_t site) {
  if (NVRAR_LIKELY(c.jitter_ns == 0)) return;
  jitter_sleep(c.jitter_seed,
               c.seq * 0x9E3779B9u ^ (blockIdx.x << 20) ^ (blockIdx.y << 26) ^
                   ((threadIdx.x >> 5) << 8) ^ site,
               c.jitter_ns);
}

// flag observed in a slot for call `seq`: equal = arrived; behind = not yet
// (an empty cell reads 0xFFFFFFFF); ahead = a peer ran more calls than this
// rank (ProtocolFaultError).
__device__ __forceinline__ bool flag_ahead(uint32_t flag, uint32_t seq) {
  return flag != 0xFFFFFFFFu && static_cast<int32_t>(flag - seq) > 0;
}

// ---------------------------------------------------------------------------
// Wire protocols over 16-byte cells. A unit carries W payload dwords in
// cells<W>() cells; within each group of 32 units, cell h of all 32 units is
// contiguous, so one warp-wide store writes 512 contiguous bytes.

__device__ __forceinline__ uint64_t cell_index(uint64_t u, int cells, int h) {
  return (((u >> 5) * static_cast<uint64_t>(cells) + static_cast<uint64_t>(h)) << 5) + (u & 31);
}

struct LL {
  static constexpr bool kLamport = false;
  template <int W>
  static constexpr int cells() {
    return W / 2;
  }
  template <int W>
  __device__ static __forceinline__ void put(uint4* slot, uint64_t u, const uint32_t (&d)[W],
                                             uint32_t seq) {
#pragma unroll
    for (int h = 0; h < W / 2; ++h) {
      st_volatile16(slot + cell_index(u, W / 2, h), d[2 * h], seq, d[2 * h + 1], seq);
    }
  }
  template <int W>
  __device__ static __forceinline__ void put_mc(uint4* slot, uint64_t u, const uint32_t (&d)[W],
                                                uint32_t seq) {
#pragma unroll
    for (int h = 0; h < W / 2; ++h) {
      st_mc16(slot + cell_index(u, W / 2, h), d[2 * h], seq, d[2 * h + 1], seq);
    }
  }
  template <int W>
  __device__ static __forceinline__ bool try_get(const uint4* slot, uint64_t u, uint32_t seq,
                                                 uint32_t (&d)[W], uint32_t& bad) {
    bool ok = true;
#pragma unroll
    for (int h = 0; h < W / 2; ++h) {
      const uint4 v = ld_volatile16(slot + cell_index(u, W / 2, h));
      d[2 * h] = v.x;
      d[2 * h + 1] = v.z;
      if (v.y != seq) {
        ok = false;
        bad = v.y;
      }
      if (v.w != seq) {
        ok = false;
        bad = v.w;
      }
    }
    return ok;
  }
  template <int W>
  __device__ static __forceinline__ void clear(uint4* slot, uint64_t u) {
#pragma unroll
    for (int h = 0; h < W / 2; ++h) {
      st_volatile16(slot + cell_index(u, W / 2, h), ~0u, ~0u, ~0u, ~0u);
    }
  }
};

// EB = element width in bytes for the sentinel test (2 = bf16, 4 = fp32).
template <int EB>
struct Lamport {
  static constexpr bool kLamport = true;
  template <int W>
  static constexpr int cells() {
    return W / 4;
  }
  // An all-ones element is the only pattern a writer may never send.
  __device__ static __forceinline__ uint32_t canon(uint32_t x) {
    if constexpr (EB == 4) {
      return x == 0xFFFFFFFFu ? 0x7FFFFFFFu : x;
    } else {
      const uint32_t m = __vcmpeq2(x, 0xFFFFFFFFu);  // 0xFFFF per all-ones half
      return x ^ (m & 0x80008000u);                  // -> 0x7FFF (another NaN)
    }
  }
  __device__ static __forceinline__ bool empty(uint32_t x) {
    if constexpr (EB == 4) {
      return x == 0xFFFFFFFFu;
    } else {
      return __vcmpeq2(x, 0xFFFFFFFFu) != 0u;
    }
  }
  template <int W>
  __device__ static __forceinline__ void put(uint4* slot, uint64_t u, const uint32_t (&d)[W],
                                             uint32_t) {
#pragma unroll
    for (int h = 0; h < W / 4; ++h) {
      st_volatile16(slot + cell_index(u, W / 4, h), canon(d[4 * h]), canon(d[4 * h + 1]),
                    canon(d[4 * h + 2]), canon(d[4 * h + 3]));
    }
  }
  template <int W>
  __device__ static __forceinline__ void put_mc(uint4* slot, uint64_t u, const uint32_t (&d)[W],
                                                uint32_t) {
#pragma unroll
    for (int h = 0; h < W / 4; ++h) {
      st_mc16(slot + cell_index(u, W / 4, h), canon(d[4 * h]), canon(d[4 * h + 1]),
              canon(d[4 * h + 2]), canon(d[4 * h + 3]));
    }
  }
  template <int W>
  __device__ static __forceinline__ bool try_get(const uint4* slot, uint64_t u, uint32_t,
                                                 uint32_t (&d)[W], uint32_t& bad) {
    bool ok = true;
#pragma unroll
    for (int h = 0; h < W / 4; ++h) {
      const uint4 v = ld_volatile16(slot + cell_index(u, W / 4, h));
      d[4 * h] = v.x;
      d[4 * h + 1] = v.y;
      d[4 * h + 2] = v.z;
      d[4 * h + 3] = v.w;
      if (empty(v.x) || empty(v.y) || empty(v.z) || empty(v.w)) ok = false;
    }
    bad = 0xFFFFFFFFu;
    return ok;
  }
  template <int W>
  __device__ static __forceinline__ void clear(uint4* slot, uint64_t u) {
#pragma unroll
    for (int h = 0; h < W / 4; ++h) {
      st_volatile16(slot + cell_index(u, W / 4, h), ~0u, ~0u, ~0u, ~0u);
    }
  }
};

// Blocking receive of unit u with watchdog; the cells are re-emptied after the
// read. `peer` labels the diagnosis.
template <class Pr, int W>
__device__ __forceinline__ void recv_unit(Ctl& c, uint4* slot, uint64_t u, uint32_t (&d)[W],
                                          int peer) {
  uint32_t bad = 0;
  while (!Pr::template try_get<W>(slot, u, c.seq, d, bad)) {
    if (!Pr::kLamport && flag_ahead(bad, c.seq)) {
      record_fault(c, kProtocolFault, kStaleFlag, peer, u, bad);
      return;
    }
    if (wait_tick(c, kFlagWait, peer, u, bad)) return;
    poll_pause(c);
  }
  Pr::template clear<W>(slot, u);
}

// Receive K cells at once: every round issues one load per still-pending cell
// (bit k of `pending`), so detection costs one L2 round trip after the LAST
// arrival instead of one round trip per source. Arrived cells are re-emptied.
template <class Pr, int W, int K>
__device__ __forceinline__ void recv_all(Ctl& c, uint4* const (&slot)[K], const uint64_t (&u)[K],
                                         uint32_t (&d)[K][W], uint32_t pending,
                                         const int (&peer)[K]) {
  while (pending) {
    uint32_t bad = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if ((pending >> k) & 1u) {
        if (Pr::template try_get<W>(slot[k], u[k], c.seq, d[k], bad)) {
          Pr::template clear<W>(slot[k], u[k]);
          pending &= ~(1u << k);
        } else if (!Pr::kLamport && flag_ahead(bad, c.seq)) {
          record_fault<(K <= 8)>(c, kProtocolFault, kStaleFlag, peer[k], u[k], bad);
          return;
        }
      }
    }
    if (pending) {
      const int k0 = __ffs(pending) - 1;
      int pk = peer[0];
      uint64_t uk = u[0];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (k == k0) {
          pk = peer[k];
          uk = u[k];
        }
      }
      if (wait_tick<(K <= 8)>(c, kFlagWait, pk, uk, bad)) return;
      poll_pause<(K <= 8)>(c);
    }
  }
}

// Same, for an [NN][MM] grid of source cells of one unit u (bit nn*MM + m).
template <class Pr, int W, int NN, int MM>
__device__ __forceinline__ void recv_grid(Ctl& c, uint4* const (&slot)[NN][MM], uint64_t u,
                                          uint32_t (&d)[NN][MM][W], uint32_t pending,
                                          const int (&peer)[NN][MM]) {
  while (pending) {
    uint32_t bad = 0;
#pragma unroll
    for (int a = 0; a < NN; ++a) {
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const uint32_t bit = 1u << (a * MM + m);
        if (pending & bit) {
          if (Pr::template try_get<W>(slot[a][m], u, c.seq, d[a][m], bad)) {
            Pr::template clear<W>(slot[a][m], u);
            pending &= ~bit;
          } else if (!Pr::kLamport && flag_ahead(bad, c.seq)) {
            record_fault<(NN * MM <= 8)>(c, kProtocolFault, kStaleFlag, peer[a][m], u, bad);
            return;
          }
        }
      }
    }
    if (pending) {
      const int k0 = __ffs(pending) - 1;
      int pk = 0;
#pragma unroll
      for (int a = 0; a < NN; ++a) {
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          if (a * MM + m == k0) pk = peer[a][m];
        }
      }
      if (wait_tick<(NN * MM <= 8)>(c, kFlagWait, pk, u, bad)) return;
      poll_pause<(NN * MM <= 8)>(c);
    }
  }
}

// Same, for NN rows of MM source cells where row a is unit u[a] (bit a*MM + m).
template <class Pr, int W, int NN, int MM>
__device__ __forceinline__ void recv_rows(Ctl& c, uint4* const (&slot)[NN][MM],
                                          const uint64_t (&u)[NN], uint32_t (&d)[NN][MM][W],
                                          uint32_t pending, const int (&peer)[NN][MM]) {
  constexpr bool kOutline = NN * MM <= 8;
  while (pending) {
    uint32_t bad = 0;
#pragma unroll
    for (int a = 0; a < NN; ++a) {
#pragma unroll
      for (int m = 0; m < MM; ++m) {
        const uint32_t bit = 1u << (a * MM + m);
        if (pending & bit) {
          if (Pr::template try_get<W>(slot[a][m], u[a], c.seq, d[a][m], bad)) {
            Pr::template clear<W>(slot[a][m], u[a]);
            pending &= ~bit;
          } else if (!Pr::kLamport && flag_ahead(bad, c.seq)) {
            record_fault<kOutline>(c, kProtocolFault, kStaleFlag, peer[a][m], u[a], bad);
            return;
          }
        }
      }
    }
    if (pending) {
      const int k0 = __ffs(pending) - 1;
      int pk = 0;
      uint64_t uk = 0;
#pragma unroll
      for (int a = 0; a < NN; ++a) {
#pragma unroll
        for (int m = 0; m < MM; ++m) {
          if (a * MM + m == k0) {
            pk = peer[a][m];
            uk = u[a];
          }
        }
      }
      if (wait_tick<kOutline>(c, kFlagWait, pk, uk, bad)) return;
      poll_pause<kOutline>(c);
    }
  }
}

// ---------------------------------------------------------------------------
// Element traits. RAW is the caller dtype's bits, ACC the arithmetic type
// (fp32 for float/bf16, wrapping uint32 for int32).

struct F32 {
  using acc = float;
  static constexpr int kBytes = 4;
};
struct I32 {
  using acc = uint32_t;
  static constexpr int kBytes = 4;
};
struct BF16 {
  using acc = float;
  static constexpr int kBytes = 2;
};

__device__ __forceinline__ float acc_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ uint32_t acc_add(uint32_t a, uint32_t b) { return a + b; }

__device__ __forceinline__ uint32_t f32_to_bf16_rne(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (u >> 16) | 0x40u;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return u >> 16;
}

// raw dwords (UE elements) <-> UE accumulators
template <int UE>
__device__ __forceinline__ void raw_to_acc(F32, const uint32_t (&d)[UE], float (&a)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) a[k] = __uint_as_float(d[k]);
}
template <int UE>
__device__ __forceinline__ void raw_to_acc(I32, const uint32_t (&d)[UE], uint32_t (&a)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) a[k] = d[k];
}
template <int UE>
__device__ __forceinline__ void raw_to_acc(BF16, const uint32_t (&d)[UE / 2], float (&a)[UE]) {
#pragma unroll
  for (int k = 0; k < UE / 2; ++k) {
    a[2 * k] = __uint_as_float(d[k] << 16);
    a[2 * k + 1] = __uint_as_float(d[k] & 0xFFFF0000u);
  }
}
template <int UE>
__device__ __forceinline__ void acc_to_raw(F32, const float (&a)[UE], uint32_t (&d)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) d[k] = __float_as_uint(a[k]);
}
template <int UE>
__device__ __forceinline__ void acc_to_raw(I32, const uint32_t (&a)[UE], uint32_t (&d)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) d[k] = a[k];
}
template <int UE>
__device__ __forceinline__ void acc_to_raw(BF16, const float (&a)[UE], uint32_t (&d)[UE / 2]) {
#pragma unroll
  for (int k = 0; k < UE / 2; ++k) {
    d[k] = f32_to_bf16_rne(a[2 * k]) | (f32_to_bf16_rne(a[2 * k + 1]) << 16);
  }
}

// accumulators <-> payload dwords (recursive-doubling partials)
template <int UE>
__device__ __forceinline__ void acc_bits(const float (&a)[UE], uint32_t (&d)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) d[k] = __float_as_uint(a[k]);
}
template <int UE>
__device__ __forceinline__ void acc_bits(const uint32_t (&a)[UE], uint32_t (&d)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) d[k] = a[k];
}
template <int UE>
__device__ __forceinline__ void bits_acc(const uint32_t (&d)[UE], float (&a)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) a[k] = __uint_as_float(d[k]);
}
template <int UE>
__device__ __forceinline__ void bits_acc(const uint32_t (&d)[UE], uint32_t (&a)[UE]) {
#pragma unroll
  for (int k = 0; k < UE; ++k) a[k] = d[k];
}

// Load UE raw elements starting at element index e of `p`, `valid` of them real
// (the rest are the reference's zero padding, nvrar.hpp:99-104). RDW dwords.
template <class E, int UE>
__device__ __forceinline__ void load_raw(const void* p, uint64_t e, int valid,
                                         uint32_t (&d)[UE * E::kBytes / 4]) {
  constexpr int RDW = UE * E::kBytes / 4;
  if constexpr (E::kBytes == 4) {
    const uint32_t* q = static_cast<const uint32_t*>(p) + e;
    if (NVRAR_LIKELY(valid == UE && (reinterpret_cast<uintptr_t>(q) & 15u) == 0)) {
#pragma unroll
      for (int h = 0; h < RDW / 4; ++h) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(q) + h);
        d[4 * h] = v.x;
        d[4 * h + 1] = v.y;
        d[4 * h + 2] = v.z;
        d[4 * h + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < UE; ++k) d[k] = k < valid ? __ldg(q + k) : 0u;
    }
  } else {
    const uint16_t* q = static_cast<const uint16_t*>(p) + e;
    if constexpr (RDW == 4) {
      if (NVRAR_LIKELY(valid == UE && (reinterpret_cast<uintptr_t>(q) & 15u) == 0)) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(q));
        d[0] = v.x;
        d[1] = v.y;
        d[2] = v.z;
        d[3] = v.w;
        return;
      }
    } else {
      if (NVRAR_LIKELY(valid == UE && (reinterpret_cast<uintptr_t>(q) & 7u) == 0)) {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(q));
        d[0] = v.x;
        d[1] = v.y;
        return;
      }
    }
#pragma unroll
    for (int k = 0; k < RDW; ++k) {
      const uint32_t lo = 2 * k < valid ? static_cast<uint32_t>(__ldg(q + 2 * k)) : 0u;
      const uint32_t hi = 2 * k + 1 < valid ? static_cast<uint32_t>(__ldg(q + 2 * k + 1)) : 0u;
      d[k] = lo | (hi << 16);
    }
  }
}

template <class E, int UE>
__device__ __forceinline__ void store_raw(void* p, uint64_t e, int valid,
                                          const uint32_t (&d)[UE * E::kBytes / 4]) {
  constexpr int RDW = UE * E::kBytes / 4;
  if constexpr (E::kBytes == 4) {
    uint32_t* q = static_cast<uint32_t*>(p) + e;
    if (NVRAR_LIKELY(valid == UE && (reinterpret_cast<uintptr_t>(q) & 15u) == 0)) {
#pragma unroll
      for (int h = 0; h < RDW / 4; ++h) {
        reinterpret_cast<uint4*>(q)[h] = make_uint4(d[4 * h], d[4 * h + 1], d[4 * h + 2], d[4 * h + 3]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < UE; ++k)
        if (k < valid) q[k] = d[k];
    }
  } else {
    uint16_t* q = static_cast<uint16_t*>(p) + e;
    if constexpr (RDW == 4) {
      if (NVRAR_LIKELY(valid == UE && (reinterpret_cast<uintptr_t>(q) & 15u) == 0)) {
        *reinterpret_cast<uint4*>(q) = make_uint4(d[0], d[1], d[2], d[3]);
        return;
      }
    } else {
      if (NVRAR_LIKELY(valid == UE && (reinterpret_cast<uintptr_t>(q) & 7u) == 0)) {
        *reinterpret_cast<uint2*>(q) = make_uint2(d[0], d[1]);
        return;
      }
    }
#pragma unroll
    for (int k = 0; k < RDW; ++k) {
      if (2 * k < valid) q[2 * k] = static_cast<uint16_t>(d[k] & 0xFFFFu);
      if (2 * k + 1 < valid) q[2 * k + 1] = static_cast<uint16_t>(d[k] >> 16);
    }
  }
}

template <int UE>
__device__ __forceinline__ int clamp_valid(int64_t v) {
  return v < 0 ? 0 : (v > UE ? UE : static_cast<int>(v));
}

// Symmetric-region slot addressing.
__device__ __forceinline__ uint4* slot_a(const RankDesc& d, int rank, uint32_t parity, int src) {
  return reinterpret_cast<uint4*>(d.base[rank] + d.lay.a_off +
                                  ((static_cast<uint64_t>(parity) * d.world + src) * d.lay.a_src) * 8);
}
__device__ __forceinline__ uint4* slot_b(const RankDesc& d, int rank, uint32_t parity, int src) {
  return reinterpret_cast<uint4*>(d.base[rank] + d.lay.b_off +
                                  ((static_cast<uint64_t>(parity) * d.world + src) * d.lay.b_src) * 8);
}
__device__ __forceinline__ uint4* slot_c(const RankDesc& d, int rank, uint32_t parity, int step) {
  return reinterpret_cast<uint4*>(d.base[rank] + d.lay.c_off +
                                  ((static_cast<uint64_t>(parity) * d.steps + step) * d.lay.c_step) * 8);
}
__device__ __forceinline__ uint64_t* counters(const RankDesc& d, int rank) {
  return reinterpret_cast<uint64_t*>(d.base[rank] + d.lay.ctrl_off);
}
// ping-pong word (signal-latency probe), right after the counters
__device__ __forceinline__ uint64_t* diag_word(const RankDesc& d, int rank) {
  return counters(d, rank) + kMaxRanks;
}
// 16-byte cell of the word-atomicity canary (nvrar_debug_canary), in the diag block
__device__ __forceinline__ uint4* canary_cell(const RankDesc& d, int rank) {
  return reinterpret_cast<uint4*>(counters(d, rank) + kMaxRanks + 2);
}
// done[p] = (seq<<32)|len from rank p: p finished reading this rank's
// registered buffer for call seq (nvrar_allreduce_registered)
__device__ __forceinline__ uint64_t* done_words(const RankDesc& d, int rank) {
  return counters(d, rank) + 2 * kMaxRanks;
}

// Programmatic dependent launch: everything before pdl_wait() may overlap the
// previous kernel on the stream; nothing it wrote may be touched before.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void stamp(const RankDesc& d, int k) {
  if (d.profile && threadIdx.x == 0) d.state->ts[blockIdx.x][k] = globaltimer();
}

// Pull the residual unit of element e into L2 while the unit's data is still
// in flight (no registers held; emit's load then hits L2).
template <class E>
__device__ __forceinline__ void prefetch_resid(const void* resid, uint64_t e) {
  if (NVRAR_UNLIKELY(resid != nullptr)) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const char*>(resid) + e * E::kBytes));
  }
}

// Final store of an output unit: plain, or fused with the residual add.
template <class E, int UE>
__device__ __forceinline__ void emit(void* recv, const void* resid, uint64_t e, int valid,
                                     const uint32_t (&o)[UE * E::kBytes / 4]) {
  if (NVRAR_LIKELY(resid == nullptr)) {
    store_raw<E, UE>(recv, e, valid, o);
    return;
  }
  using A = typename E::acc;
  uint32_t x[UE * E::kBytes / 4];
  load_raw<E, UE>(resid, e, valid, x);
  A xa[UE], oa[UE];
  raw_to_acc<UE>(E{}, x, xa);
  raw_to_acc<UE>(E{}, o, oa);
#pragma unroll
  for (int q = 0; q < UE; ++q) xa[q] = acc_add(xa[q], oa[q]);
  uint32_t r[UE * E::kBytes / 4];
  acc_to_raw<UE>(E{}, xa, r);
  store_raw<E, UE>(recv, e, valid, r);
}

}  // namespace nvrar
