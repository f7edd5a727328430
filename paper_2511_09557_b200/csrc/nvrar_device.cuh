// Device-side data structures and primitives of the B200 NVRAR all-reduce.
//
// Transport model (replaces the reference's one-sided Ctx, transport.hpp:137-202):
//  * every rank owns ONE symmetric region (same layout on all ranks, zeroed at
//    creation, mapped into each peer process through CUDA IPC) — the analogue
//    of Ctx::alloc_region's symmetric, zero-filled regions;
//  * data moves as LL ("low-latency") words: 8 bytes = 4-byte payload (low) +
//    4-byte sequence flag (high), i.e. the reference's fused word
//    (transport.hpp:81-87, fused.hpp:4-8). A thread stores two words with one
//    16-byte st.volatile over NVLink and the receiver polls the words
//    themselves, so arrival of data is arrival of its signal — no fence and no
//    per-pair ordering assumption (NVLink does not order weak stores to
//    different addresses, unlike the reference transport, transport.hpp:9-11);
//  * sequence/length words (seq<<32 | len) published into the peer's counter
//    array stand in for Ctx::publish_counter (transport.hpp:161-164), and the
//    wait on them is the reference's peer-only sync (nvrar.hpp:163-171).
#pragma once

#include <cstdint>

namespace nvrar {

constexpr int kMaxRanks = 64;   // NVRAR_MAX_RANKS
constexpr int kMaxLocal = 32;   // NVRAR_MAX_LOCAL (virtual ranks per launch)
constexpr int kThreads = 512;   // threads per CTA
constexpr int kUnit = 4;        // elements per unit (one thread's work item)

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
  uint64_t ctrl_off;  // u64 counters[kMaxRanks]: counters[p] = (seq<<32)|len from rank p
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
  uint64_t word;      // word index inside the awaited slot (FlagWait)
  uint64_t observed;  // what was seen instead
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
  uint64_t ts[kPhases];  // phase timestamps of CTA 0, thread 0 (profiling)
};

struct RankDesc {
  uint8_t* base[kMaxRanks];  // every rank's symmetric region, as mapped here
  RankState* state;          // own
  Layout lay;
  int rank, world, nodes, gpus, steps, node, local;
  int profile;
  uint64_t timeout_ns;
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
};

// ---------------------------------------------------------------------------
// PTX primitives

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint4 ld_volatile16(const void* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile16(void* p, uint32_t a, uint32_t b, uint32_t c,
                                              uint32_t d) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b),
               "r"(c), "r"(d)
               : "memory");
}

__device__ __forceinline__ uint64_t ld_volatile64(const void* p) {
  uint64_t v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_volatile64(void* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_volatile32(const void* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// Per-thread wait control: watchdog (DeadlockError analogue, errors.hpp:61-85)
// and fault recording. Once a thread aborts it keeps walking the same control
// flow (so every __syncthreads is still reached) but stops waiting.

struct Ctl {
  RankState* st;
  uint64_t timeout_ns;
  uint32_t seq;
  uint32_t spins;
  uint64_t t0;
  bool aborted;
};

__device__ __forceinline__ void record_fault(Ctl& c, uint32_t code, int kind, int peer,
                                             uint64_t word, uint64_t observed) {
  ErrRec* e = &c.st->err;
  if (atomicCAS(&e->code, 0u, 0xFFFFFFFFu) == 0u) {
    e->kind = kind;
    e->peer = peer;
    e->expected = c.seq;
    e->word = word;
    e->observed = observed;
    __threadfence();
    atomicExch(&e->code, code);
  }
  c.aborted = true;
}

// Called while a wait is unsatisfied. Returns true when the thread must give up.
__device__ __forceinline__ bool wait_tick(Ctl& c, int kind, int peer, uint64_t word,
                                          uint64_t observed) {
  if (c.aborted) return true;
  if ((++c.spins & 127u) != 0u) return false;
  if (ld_volatile32(&c.st->err.code) != 0u) {
    c.aborted = true;
    return true;
  }
  const uint64_t now = globaltimer();
  if (now - c.t0 > c.timeout_ns) {
    record_fault(c, kDeadlock, kind, peer, word, observed);
    return true;
  }
  return false;
}

// flag observed in a slot for call `seq`: equal = arrived; behind = not yet;
// ahead = a peer ran more calls than this rank (ProtocolFaultError).
__device__ __forceinline__ bool flag_ahead(uint32_t flag, uint32_t seq) {
  return static_cast<int32_t>(flag - seq) > 0;
}

// ---------------------------------------------------------------------------
// LL slots. A unit carries DW payload dwords as DW LL words (DW/2 16-byte
// stores). Within each group of 32 units, part h of all 32 units is
// contiguous, so one warp-wide store writes 512 contiguous bytes.

template <int DW>
__device__ __forceinline__ uint64_t ll_off16(uint64_t u, int h) {
  return (((u >> 5) * (DW / 2) + static_cast<uint64_t>(h)) << 5) + (u & 31);
}

template <int DW>
__device__ __forceinline__ void ll_store(uint4* slot, uint64_t u, const uint32_t (&d)[DW],
                                         uint32_t seq) {
#pragma unroll
  for (int h = 0; h < DW / 2; ++h) {
    st_volatile16(slot + ll_off16<DW>(u, h), d[2 * h], seq, d[2 * h + 1], seq);
  }
}

// One non-blocking attempt: fills d and returns true when every word carries
// `seq`.
template <int DW>
__device__ __forceinline__ bool ll_try(const uint4* slot, uint64_t u, uint32_t seq,
                                       uint32_t (&d)[DW], uint32_t& bad_flag) {
  bool ok = true;
#pragma unroll
  for (int h = 0; h < DW / 2; ++h) {
    const uint4 v = ld_volatile16(slot + ll_off16<DW>(u, h));
    d[2 * h] = v.x;
    d[2 * h + 1] = v.z;
    if (v.y != seq) {
      ok = false;
      bad_flag = v.y;
    }
    if (v.w != seq) {
      ok = false;
      bad_flag = v.w;
    }
  }
  return ok;
}

// Blocking poll with watchdog. `peer` labels the diagnosis.
template <int DW>
__device__ __forceinline__ void ll_wait(Ctl& c, const uint4* slot, uint64_t u,
                                        uint32_t (&d)[DW], int peer) {
  uint32_t bad = 0;
  while (!ll_try<DW>(slot, u, c.seq, d, bad)) {
    if (flag_ahead(bad, c.seq)) {
      record_fault(c, kProtocolFault, kStaleFlag, peer, u * DW, bad);
      return;
    }
    if (wait_tick(c, kFlagWait, peer, u * DW, bad)) return;
  }
}

// ---------------------------------------------------------------------------
// Element traits. A unit is kUnit=4 elements; RAW is the caller dtype's bits,
// ACC the arithmetic type (fp32 for float/bf16, wrapping uint32 for int32).

struct F32 {
  using acc = float;
  static constexpr int DW = 4;  // payload dwords per unit of raw elements
  static constexpr int kBytes = 4;
};
struct I32 {
  using acc = uint32_t;
  static constexpr int DW = 4;
  static constexpr int kBytes = 4;
};
struct BF16 {
  using acc = float;
  static constexpr int DW = 2;
  static constexpr int kBytes = 2;
};

__device__ __forceinline__ float acc_add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ uint32_t acc_add(uint32_t a, uint32_t b) { return a + b; }

// raw dwords <-> 4 accumulators
__device__ __forceinline__ void raw_to_acc(F32, const uint32_t (&d)[4], float (&a)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = __uint_as_float(d[k]);
}
__device__ __forceinline__ void raw_to_acc(I32, const uint32_t (&d)[4], uint32_t (&a)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = d[k];
}
__device__ __forceinline__ void raw_to_acc(BF16, const uint32_t (&d)[2], float (&a)[4]) {
  a[0] = __uint_as_float(d[0] << 16);
  a[1] = __uint_as_float(d[0] & 0xFFFF0000u);
  a[2] = __uint_as_float(d[1] << 16);
  a[3] = __uint_as_float(d[1] & 0xFFFF0000u);
}

__device__ __forceinline__ uint32_t f32_to_bf16_rne(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (u >> 16) | 0x40u;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return u >> 16;
}

__device__ __forceinline__ void acc_to_raw(F32, const float (&a)[4], uint32_t (&d)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k] = __float_as_uint(a[k]);
}
__device__ __forceinline__ void acc_to_raw(I32, const uint32_t (&a)[4], uint32_t (&d)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k] = a[k];
}
__device__ __forceinline__ void acc_to_raw(BF16, const float (&a)[4], uint32_t (&d)[2]) {
  d[0] = f32_to_bf16_rne(a[0]) | (f32_to_bf16_rne(a[1]) << 16);
  d[1] = f32_to_bf16_rne(a[2]) | (f32_to_bf16_rne(a[3]) << 16);
}

// acc <-> 4 payload dwords (recursive-doubling partials always travel as 4 dwords)
__device__ __forceinline__ void acc_bits(const float (&a)[4], uint32_t (&d)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k] = __float_as_uint(a[k]);
}
__device__ __forceinline__ void acc_bits(const uint32_t (&a)[4], uint32_t (&d)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k] = a[k];
}
__device__ __forceinline__ void bits_acc(const uint32_t (&d)[4], float (&a)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = __uint_as_float(d[k]);
}
__device__ __forceinline__ void bits_acc(const uint32_t (&d)[4], uint32_t (&a)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) a[k] = d[k];
}

// Load 4 raw elements starting at element index e of `p`, `valid` of them real
// (the rest are the reference's zero padding, nvrar.hpp:99-104).
template <class E>
__device__ __forceinline__ void load_raw(const void* p, uint64_t e, int valid,
                                         uint32_t (&d)[E::DW]) {
  if constexpr (E::kBytes == 4) {
    const uint32_t* q = static_cast<const uint32_t*>(p) + e;
    if (valid == 4 && (reinterpret_cast<uintptr_t>(q) & 15u) == 0) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(q));
      d[0] = v.x;
      d[1] = v.y;
      d[2] = v.z;
      d[3] = v.w;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) d[k] = k < valid ? __ldg(q + k) : 0u;
    }
  } else {
    const uint16_t* q = static_cast<const uint16_t*>(p) + e;
    if (valid == 4 && (reinterpret_cast<uintptr_t>(q) & 7u) == 0) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(q));
      d[0] = v.x;
      d[1] = v.y;
    } else {
      uint32_t h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = k < valid ? static_cast<uint32_t>(__ldg(q + k)) : 0u;
      d[0] = h[0] | (h[1] << 16);
      d[1] = h[2] | (h[3] << 16);
    }
  }
}

template <class E>
__device__ __forceinline__ void store_raw(void* p, uint64_t e, int valid,
                                          const uint32_t (&d)[E::DW]) {
  if constexpr (E::kBytes == 4) {
    uint32_t* q = static_cast<uint32_t*>(p) + e;
    if (valid == 4 && (reinterpret_cast<uintptr_t>(q) & 15u) == 0) {
      *reinterpret_cast<uint4*>(q) = make_uint4(d[0], d[1], d[2], d[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < valid) q[k] = d[k];
    }
  } else {
    uint16_t* q = static_cast<uint16_t*>(p) + e;
    if (valid == 4 && (reinterpret_cast<uintptr_t>(q) & 7u) == 0) {
      *reinterpret_cast<uint2*>(q) = make_uint2(d[0], d[1]);
    } else {
      const uint32_t h[4] = {d[0] & 0xFFFFu, d[0] >> 16, d[1] & 0xFFFFu, d[1] >> 16};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k < valid) q[k] = static_cast<uint16_t>(h[k]);
    }
  }
}

__device__ __forceinline__ int clamp_valid(int64_t v) {
  return v < 0 ? 0 : (v > 4 ? 4 : static_cast<int>(v));
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

// Programmatic dependent launch: everything before pdl_wait() may overlap the
// previous kernel on the stream; nothing it wrote may be touched before.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void stamp(const RankDesc& d, int k) {
  if (d.profile && blockIdx.x == 0 && threadIdx.x == 0) d.state->ts[k] = globaltimer();
}

}  // namespace nvrar
