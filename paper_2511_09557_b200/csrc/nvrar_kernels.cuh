// B200 (sm_100a) kernels of the NVRAR all-reduce (templates; instantiated per
// dtype in nvrar_inst_*.cu so the build compiles them in parallel).
//
// One persistent launch per call runs every phase of the schedule; no host
// round trip, no NCCL. Two kernel families compute the SAME bits — the
// reference's reduction order for hierarchy nodes x gpus_per_node:
//
//   element e, shard S = ceil(n/G), c = e / S:
//     node partial = x[(c+1)%G] + x[(c+2)%G] + ... + x[c]   (ring_schedule.hpp:12-15,
//                                                             oracles.hpp:49-61)
//     result       = pairwise tree over nodes in node order  (nvrar.hpp:207-219;
//                    i.e. v = partner + own per XOR step       oracles.hpp:122-130)
//
// hier_kernel — the paper's three phases (nvrar.hpp:84-129):
//   1. intra-group reduce-scatter: every rank pushes chunk c of its input to
//      group member c over NVLink; member c folds its chunk in the pinned
//      order with its own copy last;
//   2. inter-group recursive doubling on the shard (nvrar.hpp:197-220): per
//      unit, the running fp32/int32 partial goes to the XOR peer's per-step
//      receive slot, the partner's arrives in ours, v = partner + own, and the
//      unit is forwarded to the next step at once (the reference's chunk
//      pipeline at the granularity of one thread's unit);
//   3. intra-group all-gather fused with the final cast (fp32 -> bf16 RNE):
//      the finished shard is written to the caller's output and pushed to the
//      group members.
//   Before the first inter-group send each rank publishes (seq<<32 | len) to
//   its log2(N) XOR peers and waits for theirs — the reference's peer-only
//   sync with its length check (nvrar.hpp:163-171, ring.hpp:86-98).
//
// flat_kernel — the same order on a flat schedule (B200-first: every peer is
//   one NVSwitch hop away, so the hierarchy only has to fix the ORDER):
//   two-shot = flat reduce-scatter (rank p owns elements [p*SP, (p+1)*SP)) +
//   flat all-gather; one-shot = every rank receives every input (optionally
//   pushed once through an NVSwitch multicast mapping). It also evaluates the
//   reference's ring and tree orders (LaunchParams.order) and windows of a
//   longer vector (LaunchParams.e_off / n_order, the host-buffer pipeline).
//
// direct_kernel — virtual ranks sharing one GPU, all in one launch: each unit
//   is folded once from every rank's input and written to every output.
//
// Every kernel's final store can fuse the residual add (nvrar_allreduce_residual)
// and hier_kernel<..., MODE> also runs one phase on its own (phase-only entry
// points). Kernels are specialised on the node count and on the group size.
//
// Reuse safety without any barrier: every slot set is double-buffered by call
// parity (nvrar.hpp:107-109,124-126) and re-emptied by its reader. A rank can
// only write parity p again in call k+2 after finishing call k+1, which needed
// data the reader sent only after it had finished call k (reads and re-empty
// stores included) — so a slot is never overwritten before it is read.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "nvrar_device.cuh"

namespace nvrar {

// Protocol configuration per dtype: LL (fused words, 4 elements per unit) or
// Lamport (raw payload, 16 bytes of elements per unit). RD partials are fp32 /
// int32 accumulators and travel with the matching 4-byte protocol.
template <class E, bool LAMPORT>
struct Cfg {
  using Raw = std::conditional_t<LAMPORT, Lamport<E::kBytes>, LL>;
  using Part = std::conditional_t<LAMPORT, Lamport<4>, LL>;
  static constexpr int UE = LAMPORT ? 16 / E::kBytes : 4;  // elements per unit
  static constexpr int RDW = UE * E::kBytes / 4;           // raw dwords per unit
};

template <bool EMU>
__device__ __forceinline__ const RankDesc& rank_desc(const LaunchParams& lp) {
  if constexpr (EMU) {
    return *lp.desc[blockIdx.y];
  } else {
    return lp.d0;
  }
}

// Prologue, part 1: wait for the previous kernel on the stream (the previous
// call, or the producer of our input) and let the next launch start early.
__device__ __forceinline__ void begin_wait(const RankDesc& d) {
  stamp(d, 0);
  pdl_wait();
  pdl_launch_dependents();
  stamp(d, 7);
}

// The call number and the sticky fault word of this CTA. Only this GPU's
// kernels write them (a gpu-scope load measured no faster). Every thread loads
// them itself (the same two words per CTA: warp-broadcast loads), so no thread
// waits at a barrier for thread 0's load — the barrier stalls dominated the
// prologue (profiles/r02_summary.md §3). kFlagSeqBarrier (and kFlagEarlySeq,
// whose early write-back must follow every warp's read) keep the round-1 form:
// thread 0 loads, a __syncthreads broadcasts.
struct SeqWords {
  uint32_t err, seq;
};
__device__ __forceinline__ bool seq_per_thread(int flags) {
  return (flags & (kFlagSeqBarrier | kFlagEarlySeq)) == 0;
}
__device__ __forceinline__ SeqWords seq_issue(const RankDesc& d, int flags = 0) {
  SeqWords w{0u, 0u};
#ifdef NVRAR_ABL_NO_SEQ  // experiment builds only (tools/ablate.sh): no call-number read
  return w;
#endif
  if (seq_per_thread(flags) || threadIdx.x == 0) {
    w.err = ld_volatile32(&d.state->err.code);
    w.seq = ld_volatile32(&d.state->seq[blockIdx.x]);
  }
  return w;
}

// Prologue, part 2 (after the caller has issued its first input loads, which
// do not depend on the call number). Returns false on a sticky fault.
__device__ __forceinline__ bool begin_seq(const RankDesc& d, Ctl& c, SeqWords w, int flags = 0) {
  if (!seq_per_thread(flags)) {
    __shared__ uint32_t s_seq, s_err;
    if (threadIdx.x == 0) {
      s_err = w.err;
      s_seq = w.seq;
    }
    __syncthreads();
    w.err = s_err;
    w.seq = s_seq;
  }
  c.st = d.state;
  c.timeout_ns = d.timeout_ns;
  c.poll_ns = d.poll_ns;
  c.jitter_ns = d.jitter_ns;
  c.jitter_seed = d.jitter_seed;
  c.spins = 0;
  c.aborted = false;
  c.last_chance = false;
  c.len_words = nullptr;
  c.len = 0;
  c.t0 = globaltimer();
  c.seq = w.seq + 1u;
  c.phase = 2;
  stamp(d, 1);
  return w.err == 0u;
}
__device__ __forceinline__ bool begin_seq(const RankDesc& d, Ctl& c, int flags = 0) {
  return begin_seq(d, c, seq_issue(d, flags), flags);
}

// CTA b owns slots b, b + grid, ...; warp 0 writes them (small grids own many).
// The caller guarantees every warp of the CTA has read slot b already.
__device__ __forceinline__ void write_seq_slots(const RankDesc& d, uint32_t seq) {
#ifdef NVRAR_ABL_NO_END  // experiment builds only (tools/ablate.sh): no counter write-back
  return;
#endif
  if (threadIdx.x < 32) {
    for (int i = blockIdx.x + static_cast<int>(threadIdx.x) * gridDim.x; i < kSeqSlots;
         i += 32 * gridDim.x) {
      d.state->seq[i] = seq;
    }
  }
}

__device__ __forceinline__ void end_call(const RankDesc& d, uint32_t seq) {
  // every warp of the CTA has read slot b (seq_issue) before it is rewritten
  __syncthreads();
  write_seq_slots(d, seq);
  stamp(d, 6);
}

__device__ __forceinline__ void publish_seq_len(const RankDesc& d, int peer, uint32_t seq,
                                                uint64_t n) {
  st_volatile64(counters(d, peer) + d.rank,
                (static_cast<uint64_t>(seq) << 32) | (n & 0xFFFFFFFFull));
}

// wait_counter_ge(counters[peer], seq<<32) + check_peer_length
// (transport.hpp:227-237, ring.hpp:90-98).
__device__ __forceinline__ void wait_seq_len(Ctl& c, const RankDesc& d, int peer, uint64_t n) {
  const uint64_t* p = counters(d, d.rank) + peer;
  while (true) {
    const uint64_t v = ld_volatile64(p);
    const uint32_t s = static_cast<uint32_t>(v >> 32);
    if (s == c.seq) {
      if ((v & 0xFFFFFFFFull) != (n & 0xFFFFFFFFull)) {
        record_fault(c, kProtocolFault, kLenMismatch, peer, 0, v);
      }
      return;
    }
    if (flag_ahead(s, c.seq)) return;
    if (wait_tick(c, kSeqWait, peer, 0, v)) return;
    poll_pause(c);
  }
}

template <int N>
struct Log2 {
  static constexpr int value = N <= 1 ? 0 : 1 + Log2<N / 2>::value;
};
template <>
struct Log2<1> {
  static constexpr int value = 0;
};

// Real elements of unit u of the chunk starting at cbase with S elements: the
// chunk boundary (not only n) bounds it, since S need not be a multiple of UE.
template <int UE>
__device__ __forceinline__ int chunk_valid(uint64_t S, uint64_t u, uint64_t n, uint64_t cbase) {
  const int64_t in_chunk = static_cast<int64_t>(S) - static_cast<int64_t>(UE * u);
  const int64_t in_vec = static_cast<int64_t>(n) - static_cast<int64_t>(cbase + UE * u);
  return clamp_valid<UE>(in_chunk < in_vec ? in_chunk : in_vec);
}

constexpr int kHierMaxG = 8;
constexpr int kHierUpt = 2;  // units per thread carried through the RD steps together

// hier_kernel MODE: the full all-reduce, or one phase of it on its own (the
// reference's standalone phases: IntraReduceScatter / IntraAllGather,
// nvrar.hpp:254-373, and NvrarAllreduce::rd_inter, nvrar.hpp:133-155). The
// phase-only modes run the very same phase code as the all-reduce.
enum : int { kModeFull = 0, kModeRS = 1, kModeRD = 2, kModeAG = 3 };

// Group members' length guard for the intra-only modes: publish (seq<<32|len)
// to every other member and wait for theirs (the reference guard,
// nvrar.hpp:324-336, checks the ring neighbour; every member is stricter).
__device__ __forceinline__ void group_guard(Ctl& c, const RankDesc& d, uint64_t len) {
  const int G = d.gpus;
  if (G == 1) return;
  const int t = static_cast<int>(threadIdx.x);
  const int peer = d.node * G + (d.local + 1 + t) % G;
  if (blockIdx.x == 0 && t < G - 1) publish_seq_len(d, peer, c.seq, len);
  if (t < G - 1) wait_seq_len(c, d, peer, len);
  __syncthreads();
}

// ---------------------------------------------------------------------------
template <class E, bool LAMPORT, int N, bool EMU, int MODE = kModeFull, int MG = kHierMaxG>
__global__ void __launch_bounds__(kThreads, 1) hier_kernel(const __grid_constant__ LaunchParams lp) {
  using A = typename E::acc;
  using C = Cfg<E, LAMPORT>;
  using Raw = typename C::Raw;
  using Part = typename C::Part;
  constexpr int UE = C::UE;
  constexpr int RDW = C::RDW;
  constexpr bool kFull = MODE == kModeFull, kRS = MODE == kModeRS;
  constexpr bool kRD = MODE == kModeRD, kAG = MODE == kModeAG;
  constexpr bool kFold = kFull || kRS;    // phase 1 runs
  constexpr bool kGather = kFull || kAG;  // phase 3 runs
  constexpr int kSteps = (kFull || kRD) ? Log2<N>::value : 0;
  static_assert(!kRD || (E::kBytes == 4 && UE == 4), "rd_inter moves 4-byte elements");
  const RankDesc& d = rank_desc<EMU>(lp);
  const int G = d.gpus, me = d.rank, node = d.node, local = d.local;
  // full / RS: n = vector length, S = ceil(n/G); AG: count = shard, n = G * shard;
  // RD: count = shard words, the shard is the whole vector (no chunking)
  const uint64_t n = kAG ? lp.count * G : lp.count;
  const uint64_t S = (kAG || kRD) ? lp.count : (n + G - 1) / G;
  const uint64_t U = (S + UE - 1) / UE;
  const uint64_t ub = U * blockIdx.x / gridDim.x;
  const uint64_t ue = U * (blockIdx.x + 1) / gridDim.x;
  const void* send = EMU ? lp.send[blockIdx.y] : lp.send[0];
  void* recv = EMU ? lp.recv[blockIdx.y] : lp.recv[0];
  const void* resid = EMU ? lp.resid[blockIdx.y] : lp.resid[0];
  const uint64_t u_first = ub + threadIdx.x;
  // grp[j] = (local + j) % G for j < G, without a division per use
  int grp[MG];
#pragma unroll
  for (int j = 0; j < MG; ++j) grp[j] = local + j >= G ? local + j - G : local + j;

  begin_wait(d);
  const SeqWords sw = seq_issue(d, lp.flags);
  // Prefetch this thread's first unit of every chunk while the call number is
  // read (the loads do not depend on it): pre[j] = chunk (local + j) % G.
  uint32_t pre[MG][RDW];
  int pv[MG];
#pragma unroll
  for (int j = 0; j < MG; ++j) {
    pv[j] = 0;
    if (kFold && j < G && u_first < ue) {
      const uint64_t cbase = static_cast<uint64_t>(grp[j]) * S;
      pv[j] = chunk_valid<UE>(S, u_first, n, cbase);
      if (pv[j] > 0) load_raw<E, UE>(send, cbase + UE * u_first, pv[j], pre[j]);
    }
  }
  Ctl c;
  if (!begin_seq(d, c, sw, lp.flags)) return;  // sticky fault: comm is dead
  const uint32_t parity = c.seq & 1u;
  if (lp.flags & kFlagEarlySeq) end_call(d, c.seq);

  // Peer-only sync, publish half (nvrar.hpp:163-171).
  if (kSteps > 0 && blockIdx.x == 0 && threadIdx.x < kSteps) {
    publish_seq_len(d, ((node ^ (1 << threadIdx.x)) * G) + local, c.seq, n);
  }

  // Phase 1a: reduce-scatter pushes (ring_reduce_scatter_phase, ring_schedule.hpp:33-58).
  jitter(c, 1);
  if (kFold && G > 1) {
#pragma unroll
    for (int j = 1; j < MG; ++j) {
      if (j < G && pv[j] > 0) {
        Raw::template put<RDW>(slot_a(d, node * G + grp[j], parity, local), u_first,
                               pre[j], c.seq);
      }
    }
    for (int j = 1; j < G; ++j) {
      const int cc = (local + j) % G;
      uint4* slot = slot_a(d, node * G + cc, parity, local);
      const uint64_t cbase = static_cast<uint64_t>(cc) * S;
#pragma unroll 4
      for (uint64_t u = u_first + blockDim.x; u < ue; u += blockDim.x) {
        const int valid = chunk_valid<UE>(S, u, n, cbase);
        if (valid == 0) continue;  // pure padding: skipped identically by the reader
        uint32_t raw[RDW];
        load_raw<E, UE>(send, cbase + UE * u, valid, raw);
        Raw::template put<RDW>(slot, u, raw, c.seq);
      }
    }
  }
  stamp(d, 2);
  c.phase = 3;

  // Peer-only sync, wait half (nvrar.hpp:163-171): all log2(N) XOR peers'
  // (seq, len) words are checked before any RD RECEIVE — each thread checks
  // right after its first step-0 send, so the wait overlaps that send instead
  // of preceding it (the parity double-buffering, not this wait, is what makes
  // slot reuse safe; a length mismatch is still caught before any RD data is
  // consumed, and a stalled peer still shows up as a SeqWait).
  if constexpr (kRS || kAG) group_guard(c, d, lp.count);
  stamp(d, 3);
  c.phase = 4;

  // Phases 1b+2+3a: fold own chunk, recursive doubling, cast + all-gather push.
  const uint64_t mybase = kRD ? 0 : static_cast<uint64_t>(local) * S;
  bool xor_synced = false;
  for (uint64_t u0 = ub + threadIdx.x; u0 < ue; u0 += static_cast<uint64_t>(blockDim.x) * kHierUpt) {
    A f[kHierUpt][UE];
    int valid[kHierUpt];
    uint64_t uu[kHierUpt];
#pragma unroll
    for (int k = 0; k < kHierUpt; ++k) {
      uu[k] = u0 + static_cast<uint64_t>(k) * blockDim.x;
      valid[k] = uu[k] < ue ? chunk_valid<UE>(S, uu[k], n, mybase) : 0;
    }
#pragma unroll
    for (int k = 0; k < kHierUpt; ++k) {
      if (kFull && valid[k] > 0) prefetch_resid<E>(resid, mybase + UE * uu[k]);
    }
    if constexpr (kRD) {
      // rd_inter input: this rank's shard packed as LL words {data, seq}; every
      // flag must be this call's (nvrar.hpp:145-150); one node copies (:140-143)
#pragma unroll
      for (int k = 0; k < kHierUpt; ++k) {
        if (valid[k] == 0) continue;
        const uint64_t* in = static_cast<const uint64_t*>(send) + UE * uu[k];
        uint32_t b[UE];
#pragma unroll
        for (int q = 0; q < UE; ++q) {
          b[q] = 0u;
          if (q < valid[k]) {
            const uint64_t w = in[q];
            b[q] = static_cast<uint32_t>(w);
            if (N > 1 && static_cast<uint32_t>(w >> 32) != c.seq) {
              record_fault(c, kProtocolFault, kStaleFlag, me, UE * uu[k] + q, w);
            }
          }
        }
        bits_acc<UE>(b, f[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kHierUpt; ++k) {
      if (!kFold || valid[k] == 0) continue;
      uint32_t own[RDW];
      if (k == 0 && u0 == u_first) {
#pragma unroll
        for (int q = 0; q < RDW; ++q) own[q] = pre[0][q];
      } else {
        load_raw<E, UE>(send, mybase + UE * uu[k], valid[k], own);
      }
      if (G == 1) {
        raw_to_acc<UE>(E{}, own, f[k]);
        continue;
      }
      uint32_t r[1][MG - 1][RDW];
      uint4* slots[1][MG - 1];
      int peers[1][MG - 1];
      uint32_t pending = 0;
#pragma unroll
      for (int j = 1; j < MG; ++j) {
        slots[0][j - 1] = slot_a(d, me, parity, grp[j]);
        peers[0][j - 1] = node * G + grp[j];
        if (j < G) pending |= 1u << (j - 1);
      }
      recv_grid<Raw, RDW, 1, MG - 1>(c, slots, uu[k], r, pending, peers);
      // c owns in[c] + (in[c-1] + (... + (in[c+2] + in[c+1])))  (ring_schedule.hpp:12-15)
      raw_to_acc<UE>(E{}, r[0][0], f[k]);
#pragma unroll
      for (int j = 2; j < MG; ++j) {
        if (j < G) {
          A a[UE];
          raw_to_acc<UE>(E{}, r[0][j - 1], a);
#pragma unroll
          for (int q = 0; q < UE; ++q) f[k][q] = acc_add(f[k][q], a[q]);
        }
      }
      A a[UE];
      raw_to_acc<UE>(E{}, own, a);
#pragma unroll
      for (int q = 0; q < UE; ++q) f[k][q] = acc_add(f[k][q], a[q]);
    }

    // Recursive doubling (rd_block, nvrar.hpp:197-220): v = partner + own.
#pragma unroll
    for (int l = 0; l < kSteps; ++l) {
      const int partner = ((node ^ (1 << l)) * G) + local;
      uint4* dst = slot_c(d, partner, parity, l);
      jitter(c, 16 + l + static_cast<uint32_t>(u0 >> 5) * 64);
#pragma unroll
      for (int k = 0; k < kHierUpt; ++k) {
        if (valid[k] == 0) continue;
        uint32_t b[UE];
        acc_bits<UE>(f[k], b);
        Part::template put<UE>(dst, uu[k], b, c.seq);
      }
      if (l == 0 && !xor_synced) {
#pragma unroll
        for (int s2 = 0; s2 < kSteps; ++s2) wait_seq_len(c, d, ((node ^ (1 << s2)) * G) + local, n);
        xor_synced = true;
      }
      uint4* src = slot_c(d, me, parity, l);
      uint4* srcs[kHierUpt];
      int partners[kHierUpt];
      uint32_t b[kHierUpt][UE];
      uint32_t pending = 0;
#pragma unroll
      for (int k = 0; k < kHierUpt; ++k) {
        srcs[k] = src;
        partners[k] = partner;
        if (valid[k] > 0) pending |= 1u << k;
      }
      recv_all<Part, UE, kHierUpt>(c, srcs, uu, b, pending, partners);
#pragma unroll
      for (int k = 0; k < kHierUpt; ++k) {
        if (valid[k] == 0) continue;
        A p[UE];
        bits_acc<UE>(b[k], p);
#pragma unroll
        for (int q = 0; q < UE; ++q) f[k][q] = acc_add(p[q], f[k][q]);
      }
    }

    // Final cast, own output, all-gather push (ring_all_gather_phase, ring_schedule.hpp:62-83).
    jitter(c, 3 + static_cast<uint32_t>(u0 >> 5) * 64);
#pragma unroll
    for (int k = 0; k < kHierUpt; ++k) {
      if constexpr (kRS) {
        // the shard is the whole output (IntraReduceScatter::run's `out`),
        // padding past n included: zeros summed, i.e. +0 (nvrar.hpp:296-297)
        if (uu[k] >= ue) continue;
        uint32_t o[RDW];
#pragma unroll
        for (int q = 0; q < RDW; ++q) o[q] = 0u;
        if (valid[k] > 0) acc_to_raw<UE>(E{}, f[k], o);
        store_raw<E, UE>(recv, UE * uu[k], clamp_valid<UE>(static_cast<int64_t>(S) -
                                                            static_cast<int64_t>(UE * uu[k])), o);
        continue;
      }
      if (valid[k] == 0) continue;
      if constexpr (kRD) {
        // packed result, flag = this call (rd_inter's out, nvrar.hpp:153)
        uint32_t b[UE];
        acc_bits<UE>(f[k], b);
        uint64_t* out = static_cast<uint64_t*>(recv) + UE * uu[k];
        const uint64_t* in = static_cast<const uint64_t*>(send) + UE * uu[k];
#pragma unroll
        for (int q = 0; q < UE; ++q) {
          if (q < valid[k]) out[q] = N == 1 ? in[q] : (static_cast<uint64_t>(c.seq) << 32) | b[q];
        }
        continue;
      }
      uint32_t o[RDW];
      if constexpr (kAG) {
        load_raw<E, UE>(send, UE * uu[k], valid[k], o);  // the caller's shard
      } else {
        acc_to_raw<UE>(E{}, f[k], o);
      }
      emit<E, UE>(recv, resid, mybase + UE * uu[k], valid[k], o);
#pragma unroll
      for (int j = 1; j < MG; ++j) {
        if (j < G) {
          Raw::template put<RDW>(slot_b(d, node * G + grp[j], parity, local), uu[k], o, c.seq);
        }
      }
    }
  }
  stamp(d, 4);
  c.phase = 5;

  // Phase 3b: all-gather receive.
  if (kGather && G > 1) {
    for (uint64_t u = ub + threadIdx.x; u < ue; u += blockDim.x) {
      uint32_t r[1][MG - 1][RDW];
      uint4* slots[1][MG - 1];
      int peers[1][MG - 1];
      int valid[MG - 1];
      uint32_t pending = 0;
#pragma unroll
      for (int j = 1; j < MG; ++j) {
        const int s = grp[j];
        slots[0][j - 1] = slot_b(d, me, parity, s);
        peers[0][j - 1] = node * G + s;
        valid[j - 1] = 0;
        if (j < G) {
          valid[j - 1] = chunk_valid<UE>(S, u, n, static_cast<uint64_t>(s) * S);
          if (valid[j - 1] > 0) {
            pending |= 1u << (j - 1);
            prefetch_resid<E>(resid, static_cast<uint64_t>(s) * S + UE * u);
          }
        }
      }
      recv_grid<Raw, RDW, 1, MG - 1>(c, slots, u, r, pending, peers);
#pragma unroll
      for (int j = 1; j < MG; ++j) {
        if (j < G && valid[j - 1] > 0) {
          emit<E, UE>(recv, resid, static_cast<uint64_t>(grp[j]) * S + UE * u, valid[j - 1],
                      r[0][j - 1]);
        }
      }
    }
  }
  stamp(d, 5);
  if (!(lp.flags & kFlagEarlySeq)) end_call(d, c.seq);
}

// ---------------------------------------------------------------------------
// Flat schedules. MAXG bounds gpus_per_node so the N x MAXG source units live
// in statically indexed registers.

template <class E, int UE, int RDW, int N, int MAXG>
__device__ __forceinline__ typename E::acc pick(const uint32_t (&r)[N][MAXG][RDW], int nn,
                                                int idx, int k) {
  using A = typename E::acc;
  A v{};
#pragma unroll
  for (int t = 0; t < MAXG; ++t) {
    if (t == idx) {
      A a[UE];
      raw_to_acc<UE>(E{}, r[nn][t], a);
#pragma unroll
      for (int q = 0; q < UE; ++q)
        if (q == k) v = a[q];
    }
  }
  return v;
}

// SHOT = 0: schedule, order and multicast chosen at run time (LaunchParams);
// SHOT = 1: the small-message specialisation — one-shot, NVRAR order, unicast —
// with the two-shot, ring/tree and multicast code compiled out (a smaller
// kernel: fewer instruction-fetch stalls at the start of every call).
template <class E, bool LAMPORT, int N, int MAXG, bool EMU, int SHOT = 0>
__global__ void __launch_bounds__(kThreads, 1) flat_kernel(const __grid_constant__ LaunchParams lp) {
  using A = typename E::acc;
  using C = Cfg<E, LAMPORT>;
  using Raw = typename C::Raw;
  constexpr int UE = C::UE;
  constexpr int RDW = C::RDW;
  constexpr int kLevels = Log2<N>::value + 1;
  const RankDesc& d = rank_desc<EMU>(lp);
  const uint64_t n = lp.count;
  const int G = d.gpus, P = d.world, me = d.rank;
  const bool oneshot = SHOT == 1 ? true : lp.oneshot != 0;
  const int order = SHOT == 1 ? static_cast<int>(kOrderNvrar) : lp.order;
  // members of one fold: the node's G ranks, or (ring order) all P ranks
  const int OG = order == kOrderRing ? P : G;
  // 32-bit index math: the host rejects vectors of 2^31 or more elements
  // (64-bit divisions compile to an out-of-line routine on the prologue path)
  const uint32_t n_ord = static_cast<uint32_t>(lp.n_order ? lp.n_order : n);  // the whole vector
  const uint32_t SG = (n_ord + static_cast<uint32_t>(OG) - 1u) / static_cast<uint32_t>(OG);
  const uint32_t e_off = static_cast<uint32_t>(lp.e_off);
  constexpr uint32_t kAlign = UE;
  const uint32_t n32a = static_cast<uint32_t>(n);
  const uint32_t SP = oneshot ? ((n32a + kAlign - 1u) / kAlign) * kAlign
                              : ((((n32a + static_cast<uint32_t>(P) - 1u) / static_cast<uint32_t>(P)) +
                                  kAlign - 1u) / kAlign) * kAlign;
  const uint32_t U = SP / UE;
  // this CTA's units: an even split, the first U % grid CTAs one more
  const uint32_t uq = U / gridDim.x, ur = U % gridDim.x;
  const uint64_t ub = static_cast<uint64_t>(uq) * blockIdx.x + (blockIdx.x < ur ? blockIdx.x : ur);
  const uint64_t ue = ub + uq + (blockIdx.x < ur ? 1u : 0u);
  const void* send = EMU ? lp.send[blockIdx.y] : lp.send[0];
  void* recv = EMU ? lp.recv[blockIdx.y] : lp.recv[0];
  const void* resid = EMU ? lp.resid[blockIdx.y] : lp.resid[0];
  const uint64_t u_first = ub + threadIdx.x;

  begin_wait(d);
  // the call-number load first: its latency overlaps the input prefetch
  const SeqWords sw = seq_issue(d, lp.flags);
  // Prefetch this thread's first unit of every sub-shard (pre[j]: owner
  // (me + j) % P; j = 0 is our own) before the call number is read. One-shot
  // sends the same unit to everyone, so it loads once.
  constexpr int kPre = N * MAXG < 8 ? N * MAXG : 8;  // ranks <= N * MAXG
  uint32_t pre[kPre][RDW];
  int pv[kPre];
#pragma unroll
  for (int j = 0; j < kPre; ++j) {
    pv[j] = 0;
    if (j < P && u_first < ue && (!oneshot || j == 0)) {
      const uint64_t e = (oneshot ? 0 : static_cast<uint64_t>((me + j) % P) * SP) + UE * u_first;
      pv[j] = clamp_valid<UE>(static_cast<int64_t>(n) - static_cast<int64_t>(e));
      if (pv[j] > 0) load_raw<E, UE>(send, e, pv[j], pre[j]);
    }
  }
  Ctl c;
  if (!begin_seq(d, c, sw, lp.flags)) return;
  const uint32_t parity = c.seq & 1u;
  const bool lazy_len = !EMU && (lp.flags & kFlagLazyLen) != 0;
  if (lp.flags & kFlagEarlySeq) end_call(d, c.seq);
  if (lazy_len) {
    c.len_words = counters(d, me);
    c.len = static_cast<uint32_t>(n);
  }

  if (blockIdx.x == 0) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      if (p != me) publish_seq_len(d, p, c.seq, n);
    }
  }

  jitter(c, 1);
  // Reduce-scatter pushes: the owner q of each sub-shard receives our copy.
  // Multicast one-shot: ONE store per cell to the multicast mapping reaches
  // slot `me` of every rank's multicast A area (the NVSwitch replicates it).
  const bool mc = SHOT == 1 ? false : lp.mc != 0;
  uint4* const mc_slot = mc ? reinterpret_cast<uint4*>(
                                  d.mc + (static_cast<uint64_t>(parity) * d.world + me) * d.lay.a_src * 8)
                            : nullptr;
  if (mc) {
    if (pv[0] > 0) Raw::template put_mc<RDW>(mc_slot, u_first, pre[0], c.seq);
    for (uint64_t u = u_first + blockDim.x; u < ue; u += blockDim.x) {
      const int valid = clamp_valid<UE>(static_cast<int64_t>(n) - static_cast<int64_t>(UE * u));
      if (valid == 0) continue;
      uint32_t raw[RDW];
      load_raw<E, UE>(send, UE * u, valid, raw);
      Raw::template put_mc<RDW>(mc_slot, u, raw, c.seq);
    }
  }
#pragma unroll
  for (int j = 1; j < kPre; ++j) {
    if (j < P && !mc) {
      // compile-time indices only (a runtime index would put pre[] in local memory)
      if (oneshot) {
        if (pv[0] > 0) Raw::template put<RDW>(slot_a(d, (me + j) % P, parity, me), u_first, pre[0], c.seq);
      } else if (pv[j] > 0) {
        Raw::template put<RDW>(slot_a(d, (me + j) % P, parity, me), u_first, pre[j], c.seq);
      }
    }
  }
  if (oneshot && !mc) {
    // one-shot: the same unit goes to every peer — load it once, store P-1 times
    for (uint64_t u = u_first + blockDim.x; u < ue; u += blockDim.x) {
      const int valid = clamp_valid<UE>(static_cast<int64_t>(n) - static_cast<int64_t>(UE * u));
      if (valid == 0) continue;
      uint32_t raw[RDW];
      load_raw<E, UE>(send, UE * u, valid, raw);
      int q = me;
      for (int j = 1; j < P; ++j) {
        q = q + 1 == P ? 0 : q + 1;
        Raw::template put<RDW>(slot_a(d, q, parity, me), u, raw, c.seq);
      }
    }
    // peers beyond the prefetch loop's reach have not had the first unit yet
    for (int j = kPre; j < P; ++j) {
      if (pv[0] > 0) Raw::template put<RDW>(slot_a(d, (me + j) % P, parity, me), u_first, pre[0], c.seq);
    }
  }
  for (int j = 1; j < (mc || oneshot ? 1 : P); ++j) {
    const int q = (me + j) % P;
    const uint64_t qbase = oneshot ? 0 : static_cast<uint64_t>(q) * SP;
    uint4* slot = slot_a(d, q, parity, me);
#pragma unroll 4
    for (uint64_t u = (j < kPre ? u_first + blockDim.x : u_first); u < ue; u += blockDim.x) {
      const uint64_t e = qbase + UE * u;
      const int valid = clamp_valid<UE>(static_cast<int64_t>(n) - static_cast<int64_t>(e));
      if (valid == 0) continue;
      uint32_t raw[RDW];
      load_raw<E, UE>(send, e, valid, raw);
      Raw::template put<RDW>(slot, u, raw, c.seq);
    }
  }
  stamp(d, 2);
  c.phase = 3;

  // the counter write-back rides on this barrier when there is one: every warp
  // has read the call number before it, and the stores leave the kernel's tail
#ifdef NVRAR_ABL_NO_SYNC2
  const bool seq_mid = false;
#else
  const bool seq_mid = !lazy_len && !(lp.flags & kFlagEarlySeq);
#endif
  if (!lazy_len) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      if (p != me) wait_seq_len(c, d, p, n);
    }
#ifndef NVRAR_ABL_NO_SYNC2  // experiment builds only (tools/ablate.sh)
    __syncthreads();
#endif
    if (seq_mid) write_seq_slots(d, c.seq);
  }
  stamp(d, 3);
  c.phase = 4;

  // Index math in 32 bits (counts < 2^31 elements) and slot bases hoisted out
  // of the unit loop: per unit the kernel does one division (the shard of the
  // unit's first element) and walks the fold order incrementally.
  const uint32_t mybase = oneshot ? 0u : static_cast<uint32_t>(me * SP);
  const uint32_t n32 = static_cast<uint32_t>(n), SG32 = static_cast<uint32_t>(SG);
  uint8_t* const a_mine = (mc ? d.mc_local : d.base[me] + d.lay.a_off) +
                          static_cast<uint64_t>(parity) * d.world * d.lay.a_src * 8;
  const uint64_t a_stride = d.lay.a_src * 8;
  uint64_t len_seen = 0;
  // this rank's own unit of the NEXT iteration is loaded one iteration ahead,
  // so a thread with several units does not wait for an HBM load per unit
  // (small tiles only: with 16 sources the extra live registers spill)
  constexpr bool kOwnAhead = N * MAXG <= 8;
  uint32_t own_next[RDW];
#pragma unroll
  for (int q = 0; q < RDW; ++q) own_next[q] = pre[0][q];
  for (uint64_t u = ub + threadIdx.x; u < ue; u += blockDim.x) {
    const uint32_t e0 = mybase + UE * static_cast<uint32_t>(u);
    const int valid = clamp_valid<UE>(static_cast<int64_t>(n32) - static_cast<int64_t>(e0));
    uint32_t own[RDW];
    if constexpr (kOwnAhead) {
#pragma unroll
      for (int q = 0; q < RDW; ++q) own[q] = own_next[q];
      if (u + blockDim.x < ue) {
        const uint32_t e1 = e0 + UE * blockDim.x;
        const int v1 = clamp_valid<UE>(static_cast<int64_t>(n32) - static_cast<int64_t>(e1));
        if (v1 > 0) load_raw<E, UE>(send, e1, v1, own_next);
      }
    }
    if (valid == 0) continue;
    prefetch_resid<E>(resid, e0);
    const bool tree = order == kOrderTree;
    const uint32_t eg0 = e0 + e_off;  // index in the whole vector (the order's frame)
    // the tree chain does not depend on the chunk: one fixed order
    const int c0 = tree ? 0 : static_cast<int>(eg0 / SG32);
    const bool straddle = NVRAR_UNLIKELY(
        !tree && eg0 + static_cast<uint32_t>(valid) - 1u >= static_cast<uint32_t>(c0 + 1) * SG32);
    int l0 = tree ? OG - 1 : c0 + 1;
    if (l0 >= OG) l0 -= OG;

    // Every source's unit, in fold order: r[nn][j] is the copy of member
    // (c0+1+j) % OG of node nn (tree: member OG-1-j; ring: the rank at ring
    // position (c0+1+j) % P).
    uint32_t r[N][MAXG][RDW];
    uint4* slots[N][MAXG];
    int src[N][MAXG];
    uint32_t pending = 0;
#pragma unroll
    for (int nn = 0; nn < N; ++nn) {
      int l = l0;
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        src[nn][j] = order == kOrderRing ? static_cast<int>(lp.perm[l & 63]) : nn * G + l;
        slots[nn][j] = reinterpret_cast<uint4*>(a_mine + static_cast<uint64_t>(src[nn][j]) * a_stride);
        if (j < OG) {
          const int s = src[nn][j];
          if (s == me) {
            if constexpr (kOwnAhead) {
#pragma unroll
              for (int q = 0; q < RDW; ++q) r[nn][j][q] = own[q];
            } else if (u == u_first) {
#pragma unroll
              for (int q = 0; q < RDW; ++q) r[nn][j][q] = pre[0][q];
            } else {
              load_raw<E, UE>(send, e0, valid, r[nn][j]);
            }
          } else {
            pending |= 1u << (nn * MAXG + j);
          }
          l = tree ? l - 1 : (l + 1 == OG ? 0 : l + 1);
        }
      }
    }
    recv_grid<Raw, RDW, N, MAXG>(c, slots, u, r, pending, src);
    if (lazy_len && u == u_first && threadIdx.x < P) {
      // the peer's (seq, len) word, read now that its data is here; used at the end
      len_seen = ld_volatile64(counters(d, me) + threadIdx.x);
    }
    const int c3 = straddle ? c0 + 1 : c0;

    // Node partials, combined on the fly into the pairwise tree over nodes
    // (node order == the XOR-step adds): stack[k] holds a finished subtree of
    // 2^k nodes.
    A stack[kLevels][UE];
#pragma unroll
    for (int nn = 0; nn < N; ++nn) {
      A v[UE];
      if (NVRAR_LIKELY(c0 == c3)) {
        raw_to_acc<UE>(E{}, r[nn][0], v);
#pragma unroll
        for (int j = 1; j < MAXG; ++j) {
          if (j < OG) {
            A a[UE];
            raw_to_acc<UE>(E{}, r[nn][j], a);
#pragma unroll
            for (int q = 0; q < UE; ++q) v[q] = acc_add(v[q], a[q]);
          }
        }
      } else {
        // The unit straddles a shard boundary: per-element fold order.
#pragma unroll
        for (int q = 0; q < UE; ++q) {
          const int cq = q < valid ? static_cast<int>((eg0 + q) / SG32) : c0;
          const int rot = cq - c0;
          A x = pick<E, UE, RDW, N, MAXG>(r, nn, rot % OG, q);
#pragma unroll
          for (int j = 1; j < MAXG; ++j) {
            if (j < OG) x = acc_add(x, pick<E, UE, RDW, N, MAXG>(r, nn, (j + rot) % OG, q));
          }
          v[q] = x;
        }
      }
      int lvl = 0;
#pragma unroll
      for (int k = 0; k < kLevels - 1; ++k) {
        if (((nn >> k) & 1) && lvl == k) {
#pragma unroll
          for (int q = 0; q < UE; ++q) v[q] = acc_add(stack[k][q], v[q]);
          lvl = k + 1;
        }
      }
#pragma unroll
      for (int k = 0; k < kLevels; ++k) {
        if (k == lvl) {
#pragma unroll
          for (int q = 0; q < UE; ++q) stack[k][q] = v[q];
        }
      }
    }
    uint32_t o[RDW];
    acc_to_raw<UE>(E{}, stack[kLevels - 1], o);
    emit<E, UE>(recv, resid, e0, valid, o);
    if (!oneshot) {
      jitter(c, 3 + static_cast<uint32_t>(u >> 5) * 64);
      int q = me;
      for (int j = 1; j < P; ++j) {
        q = q + 1 == P ? 0 : q + 1;
        Raw::template put<RDW>(slot_b(d, q, parity, me), u, o, c.seq);
      }
    }
  }
  stamp(d, 4);
  c.phase = 5;

  if (!oneshot) {
    uint8_t* const b_mine = d.base[me] + d.lay.b_off + static_cast<uint64_t>(parity) * d.world * d.lay.b_src * 8;
    const uint64_t b_stride = d.lay.b_src * 8;
    // sources polled together (P <= N*MAXG ranks: at most N*MAXG-1 sources),
    // and KU units per thread per round when the tile is small: a thread with
    // several units waits one poll round trip per KU units, not per unit
    constexpr int kGrp = N * MAXG - 1 < 1 ? 1 : (N * MAXG - 1 > 8 ? 8 : N * MAXG - 1);
    constexpr int KU = kGrp <= 4 ? 2 : 1;
    for (uint64_t u0 = ub + threadIdx.x; u0 < ue; u0 += static_cast<uint64_t>(blockDim.x) * KU) {
      uint64_t uk[KU];
#pragma unroll
      for (int k = 0; k < KU; ++k) uk[k] = u0 + static_cast<uint64_t>(k) * blockDim.x;
      for (int j0 = 1; j0 < P; j0 += kGrp) {
        uint32_t r[KU][kGrp][RDW];
        uint4* slots[KU][kGrp];
        int qs[KU][kGrp];
        int valid[KU][kGrp];
        uint32_t pending = 0;
#pragma unroll
        for (int k = 0; k < KU; ++k) {
#pragma unroll
          for (int t = 0; t < kGrp; ++t) {
            int q = me - (j0 + t);
            if (q < 0) q += P;
            valid[k][t] = 0;
            qs[k][t] = q;
            slots[k][t] = reinterpret_cast<uint4*>(b_mine + static_cast<uint64_t>(q) * b_stride);
            if (j0 + t < P && uk[k] < ue) {
              const uint32_t e0 = static_cast<uint32_t>(q * SP) + UE * static_cast<uint32_t>(uk[k]);
              valid[k][t] = clamp_valid<UE>(static_cast<int64_t>(n32) - static_cast<int64_t>(e0));
              if (valid[k][t] > 0) {
                pending |= 1u << (k * kGrp + t);
                prefetch_resid<E>(resid, e0);
              }
            }
          }
        }
        recv_rows<Raw, RDW, KU, kGrp>(c, slots, uk, r, pending, qs);
#pragma unroll
        for (int k = 0; k < KU; ++k) {
#pragma unroll
          for (int t = 0; t < kGrp; ++t) {
            if (valid[k][t] > 0) {
              emit<E, UE>(recv, resid,
                          static_cast<uint32_t>(qs[k][t] * SP) + UE * static_cast<uint32_t>(uk[k]),
                          valid[k][t], r[k][t]);
            }
          }
        }
      }
    }
  }
  if (lazy_len) {
    // the peers' (seq, len) words, published before their data, were read
    // after it arrived: usually no wait is left
    c.phase = 3;
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      if (p == me) continue;
      const uint64_t v = p == static_cast<int>(threadIdx.x) ? len_seen : 0ull;
      if (static_cast<uint32_t>(v >> 32) == c.seq) {
        if ((v & 0xFFFFFFFFull) != (n & 0xFFFFFFFFull)) {
          record_fault(c, kProtocolFault, kLenMismatch, p, 0, v);
        }
      } else {
        wait_seq_len(c, d, p, n);
      }
    }
  }
  stamp(d, 5);
  if (!(lp.flags & kFlagEarlySeq) && !seq_mid) end_call(d, c.seq);
}

// ---------------------------------------------------------------------------
// Direct schedule for virtual ranks that share one HBM (EMU launches with every
// rank present): there is nothing to exchange, so each unit of the vector is
// folded once — in the same reference order — from all ranks' inputs and
// written to every rank's output. CTA (b, y) covers slice y of the units; the
// per-rank call counters advance exactly as with the message-passing schedules.
template <class E, int N, int MAXG>
__global__ void __launch_bounds__(kDirectThreads) direct_kernel(const __grid_constant__ LaunchParams lp) {
  using A = typename E::acc;
  constexpr int UE = 16 / E::kBytes;
  constexpr int RDW = 4;
  constexpr int kLevels = Log2<N>::value + 1;
  const RankDesc& d = *lp.desc[blockIdx.y];
  // the descriptor is immutable while calls run: read it before the wait
  RankState* const st = d.state;
  begin_wait(d);
  const uint32_t n = static_cast<uint32_t>(lp.count);
  const int G = lp.d0.gpus, P = lp.nlocal;  // param space: no dependent load
  const uint32_t n_ord = lp.n_order ? static_cast<uint32_t>(lp.n_order) : n;
  const uint32_t SG = (n_ord + G - 1) / G;  // order in the whole vector's frame
  const uint32_t e_off = static_cast<uint32_t>(lp.e_off);
  const bool l2pf = (lp.flags & kFlagL2Fetch256) != 0;
  const bool stream_st = (lp.flags & kFlagDirectStream) != 0;
  const uint32_t U = (n + UE - 1) / UE;
  const uint32_t slice = (U + P - 1) / P;
  // small vectors leave the last ranks' slices empty (s0 clamps to U)
  const uint32_t s0 = slice * blockIdx.y < U ? slice * blockIdx.y : U;
  const uint32_t s1 = s0 + slice < U ? s0 + slice : U;
  const uint32_t ub = s0 + static_cast<uint32_t>(static_cast<uint64_t>(s1 - s0) * blockIdx.x / gridDim.x);
  const uint32_t ue = s0 + static_cast<uint32_t>(static_cast<uint64_t>(s1 - s0) * (blockIdx.x + 1) / gridDim.x);

  // Nothing here waits on a peer, so the call number is never needed: advance
  // this CTA's replicated counter slots by one without reading them (a sticky
  // fault cannot arise in this schedule; the host refuses a failed comm). Done
  // first, so the atomics complete while the loads are in flight instead of
  // on the kernel's tail (the next call reads the slots after this grid).
  if (threadIdx.x < 32) {
    for (int i = blockIdx.x + static_cast<int>(threadIdx.x) * gridDim.x; i < kSeqSlots;
         i += 32 * gridDim.x) {
      atomicAdd(&st->seq[i], 1u);
    }
  }
  uint32_t r[N][MAXG][RDW];
  // loads of unit u from every rank, in each node's fold order (starting at the
  // chunk after the unit's own, ring.hpp fold order)
  auto load_unit = [&](uint32_t u) {
    const uint32_t e0 = UE * u;
    const int valid = clamp_valid<UE>(static_cast<int64_t>(n) - static_cast<int64_t>(e0));
    int l0 = static_cast<int>((e0 + e_off) / SG) + 1;
    if (l0 >= G) l0 -= G;
#pragma unroll
    for (int nn = 0; nn < N; ++nn) {
      int l = l0;
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        if (j < G) {
          const void* src = lp.send[nn * G + l];
          const uint8_t* at = static_cast<const uint8_t*>(src) + static_cast<uint64_t>(e0) * E::kBytes;
          if (l2pf && valid == UE && (reinterpret_cast<uintptr_t>(at) & 15u) == 0) {
            // host (PCIe) inputs: ask the L2 for 256-byte fetches (fewer, larger
            // read requests on the link)
            const uint4 v = ld_l2_256(at);
            r[nn][j][0] = v.x;
            r[nn][j][1] = v.y;
            r[nn][j][2] = v.z;
            r[nn][j][3] = v.w;
          } else {
            load_raw<E, UE>(src, e0, valid, r[nn][j]);
          }
          l = l + 1 == G ? 0 : l + 1;
        }
      }
    }
  };
  uint32_t u = ub + threadIdx.x;
  if (u < ue) load_unit(u);
  while (u < ue) {
    const uint32_t e0 = UE * u;
    const uint32_t eg0 = e0 + e_off;
    const int valid = clamp_valid<UE>(static_cast<int64_t>(n) - static_cast<int64_t>(e0));
    const int c0 = static_cast<int>(eg0 / SG);
    const bool straddle = eg0 + static_cast<uint32_t>(valid) - 1u >= static_cast<uint32_t>(c0 + 1) * SG;
    A stack[kLevels][UE];
#pragma unroll
    for (int nn = 0; nn < N; ++nn) {
      A v[UE];
      if (!straddle) {
        raw_to_acc<UE>(E{}, r[nn][0], v);
#pragma unroll
        for (int j = 1; j < MAXG; ++j) {
          if (j < G) {
            A a[UE];
            raw_to_acc<UE>(E{}, r[nn][j], a);
#pragma unroll
            for (int q = 0; q < UE; ++q) v[q] = acc_add(v[q], a[q]);
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < UE; ++q) {
          const int cq = q < valid ? static_cast<int>((eg0 + q) / SG) : c0;
          const int rot = cq - c0;
          A x = pick<E, UE, RDW, N, MAXG>(r, nn, rot % G, q);
#pragma unroll
          for (int j = 1; j < MAXG; ++j) {
            if (j < G) x = acc_add(x, pick<E, UE, RDW, N, MAXG>(r, nn, (j + rot) % G, q));
          }
          v[q] = x;
        }
      }
      // pairwise tree over nodes in node order (XOR-step adds)
      int lvl = 0;
#pragma unroll
      for (int k = 0; k < kLevels - 1; ++k) {
        if (((nn >> k) & 1) && lvl == k) {
#pragma unroll
          for (int q = 0; q < UE; ++q) v[q] = acc_add(stack[k][q], v[q]);
          lvl = k + 1;
        }
      }
#pragma unroll
      for (int k = 0; k < kLevels; ++k) {
        if (k == lvl) {
#pragma unroll
          for (int q = 0; q < UE; ++q) stack[k][q] = v[q];
        }
      }
    }
    uint32_t o[RDW];
    acc_to_raw<UE>(E{}, stack[kLevels - 1], o);
    u += blockDim.x;
    if (u < ue) load_unit(u);
    if (stream_st && valid == UE && lp.resid[0] == nullptr) {
      // experiment (kFlagDirectStream): evict-first stores of the P outputs
      for (int r2 = 0; r2 < P; ++r2) {
        uint8_t* at = static_cast<uint8_t*>(lp.recv[r2]) + static_cast<uint64_t>(e0) * E::kBytes;
        if ((reinterpret_cast<uintptr_t>(at) & 15u) == 0) {
          asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(at), "r"(o[0]), "r"(o[1]),
                       "r"(o[2]), "r"(o[3]));
        } else {
          emit<E, UE>(lp.recv[r2], lp.resid[r2], e0, valid, o);
        }
      }
    } else {
      for (int r2 = 0; r2 < P; ++r2) emit<E, UE>(lp.recv[r2], lp.resid[r2], e0, valid, o);
    }
  }
  stamp(d, 6);
}

using KernelFn = void (*)(LaunchParams);

// ---------------------------------------------------------------------------
// Registered-buffer one-shot (nvrar_allreduce_registered): every rank's INPUT
// lives in a buffer registered with the comm and mapped into every peer
// (Ctx::alloc_region's symmetric regions, transport.hpp:146-148), so nothing
// is staged: each rank announces that its input is final (the seq/len word),
// reads every peer's input in place over NVLink, folds each unit in the
// reference order (as direct_kernel) and writes its own output. Its input may
// be overwritten by the caller once this launch completes, so the launch does
// not complete before every peer has finished reading it: the last CTA to
// finish reading posts done(seq) to each peer and waits for theirs.
// lp.send[r] = rank r's input as mapped here (r = global rank, P <= 32).
template <class E, int N, int MAXG>
__global__ void __launch_bounds__(kThreads, 1) pull_kernel(const __grid_constant__ LaunchParams lp) {
  using A = typename E::acc;
  constexpr int UE = 16 / E::kBytes;
  constexpr int RDW = 4;
  constexpr int kLevels = Log2<N>::value + 1;
  const RankDesc& d = lp.d0;
  begin_wait(d);
  Ctl c;
  if (!begin_seq(d, c, lp.flags)) return;
  const int P = d.world, me = d.rank, G = d.gpus;
  const uint32_t n = static_cast<uint32_t>(lp.count);
  const uint32_t SG = (n + G - 1) / G;
  const uint32_t U = (n + UE - 1) / UE;
  const uint32_t ub = static_cast<uint32_t>(static_cast<uint64_t>(U) * blockIdx.x / gridDim.x);
  const uint32_t ue = static_cast<uint32_t>(static_cast<uint64_t>(U) * (blockIdx.x + 1) / gridDim.x);
  // ready: our input is final (stream order), peers may read it
  jitter(c, 1);
  if (blockIdx.x == 0) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      if (p != me) publish_seq_len(d, p, c.seq, n);
    }
  }
  c.phase = 3;
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    if (p != me) wait_seq_len(c, d, p, n);
  }
  __syncthreads();  // also a compiler barrier: no input load moves above the wait
  c.phase = 4;
  for (uint32_t u = ub + threadIdx.x; u < ue && !c.aborted; u += blockDim.x) {
    const uint32_t e0 = UE * u;
    const int valid = clamp_valid<UE>(static_cast<int64_t>(n) - static_cast<int64_t>(e0));
    const int c0 = static_cast<int>(e0 / SG);
    const bool straddle = e0 + static_cast<uint32_t>(valid) - 1u >= static_cast<uint32_t>(c0 + 1) * SG;
    int l0 = c0 + 1;
    if (l0 >= G) l0 -= G;
    uint32_t r[N][MAXG][RDW];
#pragma unroll
    for (int nn = 0; nn < N; ++nn) {
      int l = l0;
#pragma unroll
      for (int j = 0; j < MAXG; ++j) {
        if (j < G) {
          load_raw<E, UE>(lp.send[nn * G + l], e0, valid, r[nn][j]);
          l = l + 1 == G ? 0 : l + 1;
        }
      }
    }
    A stack[kLevels][UE];
#pragma unroll
    for (int nn = 0; nn < N; ++nn) {
      A v[UE];
      if (!straddle) {
        raw_to_acc<UE>(E{}, r[nn][0], v);
#pragma unroll
        for (int j = 1; j < MAXG; ++j) {
          if (j < G) {
            A a[UE];
            raw_to_acc<UE>(E{}, r[nn][j], a);
#pragma unroll
            for (int q = 0; q < UE; ++q) v[q] = acc_add(v[q], a[q]);
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < UE; ++q) {
          const int cq = q < valid ? static_cast<int>((e0 + q) / SG) : c0;
          const int rot = cq - c0;
          A x = pick<E, UE, RDW, N, MAXG>(r, nn, rot % G, q);
#pragma unroll
          for (int j = 1; j < MAXG; ++j) {
            if (j < G) x = acc_add(x, pick<E, UE, RDW, N, MAXG>(r, nn, (j + rot) % G, q));
          }
          v[q] = x;
        }
      }
      int lvl = 0;
#pragma unroll
      for (int k = 0; k < kLevels - 1; ++k) {
        if (((nn >> k) & 1) && lvl == k) {
#pragma unroll
          for (int q = 0; q < UE; ++q) v[q] = acc_add(stack[k][q], v[q]);
          lvl = k + 1;
        }
      }
#pragma unroll
      for (int k = 0; k < kLevels; ++k) {
        if (k == lvl) {
#pragma unroll
          for (int q = 0; q < UE; ++q) stack[k][q] = v[q];
        }
      }
    }
    uint32_t o[RDW];
    acc_to_raw<UE>(E{}, stack[kLevels - 1], o);
    emit<E, UE>(lp.recv[0], lp.resid[0], e0, valid, o);
  }
  // every thread's loads have returned (their values were stored): count this CTA
  __syncthreads();
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    s_last = atomicAdd(&d.state->arrive, 1u) == gridDim.x - 1u;
    if (s_last) d.state->arrive = 0u;  // the next call's CTAs start after this grid
  }
  __syncthreads();
  c.phase = 5;
  jitter(c, 5);
  if (s_last) {
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      if (p != me) {
        st_volatile64(done_words(d, p) + me, (static_cast<uint64_t>(c.seq) << 32) | n);
      }
    }
    for (int p = threadIdx.x; p < P; p += blockDim.x) {
      if (p == me) continue;
      const uint64_t* w = done_words(d, me) + p;
      while (true) {
        const uint64_t v = ld_volatile64(w);
        const uint32_t s = static_cast<uint32_t>(v >> 32);
        if (s == c.seq || flag_ahead(s, c.seq)) break;
        if (wait_tick(c, kSeqWait, p, 0, v)) break;
        poll_pause(c);
      }
    }
  }
  end_call(d, c.seq);
}

template <class E>
KernelFn pull_for(int nodes, int gpus) {
  KernelFn k = nullptr;
  switch (nodes) {
    case 1:
      k = gpus <= 1 ? pull_kernel<E, 1, 1> : gpus <= 2 ? pull_kernel<E, 1, 2>
        : gpus <= 4 ? pull_kernel<E, 1, 4> : gpus <= 8 ? pull_kernel<E, 1, 8> : nullptr;
      break;
    case 2:
      k = gpus <= 1 ? pull_kernel<E, 2, 1> : gpus <= 2 ? pull_kernel<E, 2, 2>
        : gpus <= 4 ? pull_kernel<E, 2, 4> : gpus <= 8 ? pull_kernel<E, 2, 8> : nullptr;
      break;
    case 4:
      k = gpus <= 1 ? pull_kernel<E, 4, 1> : gpus <= 2 ? pull_kernel<E, 4, 2>
        : gpus <= 4 ? pull_kernel<E, 4, 4> : gpus <= 8 ? pull_kernel<E, 4, 8> : nullptr;
      break;
    case 8:
      k = gpus <= 1 ? pull_kernel<E, 8, 1> : gpus <= 2 ? pull_kernel<E, 8, 2>
        : gpus <= 4 ? pull_kernel<E, 8, 4> : nullptr;
      break;
    default:
      break;
  }
  return k;
}

// MAXG = pow2 >= gpus per node (the per-thread source tile r[N][MAXG]), N * MAXG <= 32.
template <class E, int N>
KernelFn direct_for_n(int gpus) {
  if (gpus <= 1) return direct_kernel<E, N, 1>;
  if (gpus <= 2) return direct_kernel<E, N, 2>;
  if (gpus <= 4) return direct_kernel<E, N, 4>;
  if constexpr (N <= 4) {
    if (gpus <= 8) return direct_kernel<E, N, 8>;
  }
  return nullptr;
}

template <class E>
KernelFn direct_for(int nodes, int gpus) {
  switch (nodes) {
    case 1: return direct_for_n<E, 1>(gpus);
    case 2: return direct_for_n<E, 2>(gpus);
    case 4: return direct_for_n<E, 4>(gpus);
    case 8: return direct_for_n<E, 8>(gpus);
    default: return nullptr;
  }
}

template <class E, bool LAMPORT, bool EMU, int MODE>
KernelFn phase_for(int nodes) {
  switch (nodes) {
    case 1: return hier_kernel<E, LAMPORT, 1, EMU, MODE>;
    case 2: return hier_kernel<E, LAMPORT, 2, EMU, MODE>;
    case 4: return hier_kernel<E, LAMPORT, 4, EMU, MODE>;
    case 8: return hier_kernel<E, LAMPORT, 8, EMU, MODE>;
    default: return nullptr;
  }
}

// The all-reduce kernels are specialised on MG = pow2 >= gpus per node (min 2):
// the per-member tiles (prefetch, fold sources) are sized to the group.
template <class E, bool LAMPORT, bool EMU, int N>
KernelFn hier_for_n(int gpus) {
  if (gpus <= 2) return hier_kernel<E, LAMPORT, N, EMU, kModeFull, 2>;
  if (gpus <= 4) return hier_kernel<E, LAMPORT, N, EMU, kModeFull, 4>;
  if (gpus <= 8) return hier_kernel<E, LAMPORT, N, EMU, kModeFull, 8>;
  return nullptr;
}

template <class E, bool LAMPORT, bool EMU>
KernelFn hier_for(int nodes, int gpus) {
  switch (nodes) {
    case 1: return hier_for_n<E, LAMPORT, EMU, 1>(gpus);
    case 2: return hier_for_n<E, LAMPORT, EMU, 2>(gpus);
    case 4: return hier_for_n<E, LAMPORT, EMU, 4>(gpus);
    case 8: return hier_for_n<E, LAMPORT, EMU, 8>(gpus);
    default: return nullptr;
  }
}

// Flat kernels are specialised on MAXG = the next power of two >= gpus per node
// (register tiles r[N][MAXG] sized to the topology: a 2x1 launch must not
// carry the 2x8 tile — measured +1.5 us per call at P=2). N * MAXG <= 16.
template <class E, bool LAMPORT, bool EMU, int N, int SHOT>
KernelFn flat_for_n(int gpus) {
  if (gpus <= 1) return flat_kernel<E, LAMPORT, N, 1, EMU, SHOT>;
  if (gpus <= 2) return flat_kernel<E, LAMPORT, N, 2, EMU, SHOT>;
  if constexpr (N <= 4) {
    if (gpus <= 4) return flat_kernel<E, LAMPORT, N, 4, EMU, SHOT>;
  }
  if constexpr (N <= 2) {
    if (gpus <= 8) return flat_kernel<E, LAMPORT, N, 8, EMU, SHOT>;
  }
  return nullptr;
}

template <class E, bool LAMPORT, bool EMU, int SHOT = 0>
KernelFn flat_for(int nodes, int gpus) {
  switch (nodes) {
    case 1: return flat_for_n<E, LAMPORT, EMU, 1, SHOT>(gpus);
    case 2: return flat_for_n<E, LAMPORT, EMU, 2, SHOT>(gpus);
    case 4: return flat_for_n<E, LAMPORT, EMU, 4, SHOT>(gpus);
    case 8: return flat_for_n<E, LAMPORT, EMU, 8, SHOT>(gpus);
    default: return nullptr;
  }
}

// fast: the one-shot specialisation (SHOT = 1), per-rank launches only
template <class E, bool LAMPORT>
KernelFn flat_kernel_for(int nodes, int gpus, bool emu, bool fast = false) {
  if (fast && !emu) return flat_for<E, LAMPORT, false, 1>(nodes, gpus);
  return emu ? flat_for<E, LAMPORT, true>(nodes, gpus) : flat_for<E, LAMPORT, false>(nodes, gpus);
}

template <class E, bool LAMPORT>
KernelFn hier_kernel_for(int nodes, int gpus, bool emu) {
  return emu ? hier_for<E, LAMPORT, true>(nodes, gpus) : hier_for<E, LAMPORT, false>(nodes, gpus);
}

KernelFn kernel_hier_f32(int nodes, int gpus, bool emu, bool lamport);
KernelFn kernel_hier_bf16(int nodes, int gpus, bool emu, bool lamport);
KernelFn kernel_hier_i32(int nodes, int gpus, bool emu, bool lamport);
KernelFn kernel_flat_f32(int nodes, int gpus, bool emu, bool lamport, bool fast);
KernelFn kernel_flat_bf16(int nodes, int gpus, bool emu, bool lamport, bool fast);
KernelFn kernel_flat_i32(int nodes, int gpus, bool emu, bool lamport, bool fast);
KernelFn kernel_direct_f32(int nodes, int gpus);
KernelFn kernel_direct_bf16(int nodes, int gpus);
KernelFn kernel_direct_i32(int nodes, int gpus);
KernelFn kernel_phase_f32(int mode, int nodes, bool emu);
KernelFn kernel_phase_bf16(int mode, int nodes, bool emu);
KernelFn kernel_phase_i32(int mode, int nodes, bool emu);
KernelFn kernel_pull_f32(int nodes, int gpus);
KernelFn kernel_pull_bf16(int nodes, int gpus);
KernelFn kernel_pull_i32(int nodes, int gpus);

}  // namespace nvrar
