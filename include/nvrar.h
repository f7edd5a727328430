/*
 * nvrar.h — C ABI of the B200-native NVRAR all-reduce (libnvrar_b200.so).
 *
 * This is the drop-in boundary for the reference's all-reduce path. The
 * reference (/root/reference/proj, a header-only C++20 library) exposes the
 * path as a per-rank C++ object; each entry point below replaces one piece of
 * it:
 *
 *   reference                                            | this ABI
 *   -----------------------------------------------------+-----------------------------
 *   NvrarAllreduce<T>(Ctx&, max_elems)  nvrar.hpp:44-78  | nvrar_init / nvrar_comm_create
 *     + ClusterTopology{nodes,gpus}     topology.hpp:24-48 |   + nvrar_comm_export
 *     + Ctx::alloc_region (symmetric)   transport.hpp:146-148 |   + nvrar_comm_connect
 *   Ctx::alloc_region for caller data   transport.hpp:146-148 | nvrar_alloc_symmetric,
 *                                                        |   nvrar_register_buffer +
 *                                                        |   nvrar_connect_buffer
 *   NvrarAllreduce<T>::run(in,out,cfg)  nvrar.hpp:84-129 | nvrar_allreduce
 *   NvrarConfig{blocks,chunk_bytes}     fused.hpp:106-116 | nvrar_set_config
 *   NvrarAllreduce<T>::sequence()       nvrar.hpp:80     | nvrar_get_sequence
 *   NvrarAllreduce<T>::peers()          nvrar.hpp:158    | nvrar_get_peers
 *   run_ranks(...) all ranks in 1 process run.hpp:15-24  | nvrar_allreduce_local (all
 *                                                        |   comms of one device, one launch)
 *   ~NvrarAllreduce / engine teardown                    | nvrar_finalize
 *   exceptions (errors.hpp:15-85), DeadlockError blocked | nvrar_status_t, nvrar_last_error,
 *     set (errors.hpp:46-85)                             |   nvrar_get_blocked
 *
 * Status codes map the reference's exception classes one to one:
 *   InvalidArgumentError  -> NVRAR_ERR_INVALID_ARGUMENT
 *   InvalidTopologyError  -> NVRAR_ERR_INVALID_TOPOLOGY
 *   ProtocolFaultError    -> NVRAR_ERR_PROTOCOL_FAULT  (length mismatch, stale/future flag)
 *   DeadlockError         -> NVRAR_ERR_DEADLOCK        (device watchdog; see nvrar_get_blocked)
 *
 * Semantics kept from the reference: global rank =
 * node*gpus_per_node + local; nodes must be a power of two; sum only; int32
 * adds wrap; fp32 results are bit-identical to NvrarAllreduce<float> for the
 * same (nodes, gpus_per_node); bf16 results equal the fp32 reference on the
 * up-cast inputs rounded once to bf16; every call (count == 0 included) bumps
 * the sequence number by one; all ranks must issue the same calls with equal
 * counts (a mismatch across an XOR-peer or flat-schedule pair is a protocol
 * fault). Calls are asynchronous and ordered on `stream`; device-side faults
 * are sticky and surface through nvrar_check().
 *
 * No torch or CUDA types appear here: streams and device pointers are plain
 * pointers (a cudaStream_t is passed as void*).
 */
#ifndef NVRAR_H
#define NVRAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NVRAR_ABI_VERSION 1
#define NVRAR_MAX_RANKS 64
#define NVRAR_MAX_LOCAL 32
#define NVRAR_HANDLE_BYTES 256

typedef struct nvrar_comm* nvrar_comm_t;

typedef enum {
  NVRAR_SUCCESS = 0,
  NVRAR_ERR_INTERNAL = 1,
  NVRAR_ERR_INVALID_ARGUMENT = 2,
  NVRAR_ERR_INVALID_TOPOLOGY = 3,
  NVRAR_ERR_PROTOCOL_FAULT = 4,
  NVRAR_ERR_DEADLOCK = 5,
  NVRAR_ERR_CUDA = 6,
  NVRAR_ERR_NOT_CONNECTED = 7
} nvrar_status_t;

typedef enum { NVRAR_INT32 = 0, NVRAR_FLOAT32 = 1, NVRAR_BF16 = 2 } nvrar_dtype_t;

typedef enum { NVRAR_SUM = 0 } nvrar_op_t;

/* Communication schedule. Every schedule computes the SAME bits (the
 * reference's reduction order for the comm's nodes x gpus_per_node); they
 * differ only in how data moves over NVLink:
 *   HIER    — the paper's three phases: intra-group reduce-scatter, inter-group
 *             recursive doubling on the shard, intra-group all-gather.
 *   TWOSHOT — flat reduce-scatter over all ranks + flat all-gather.
 *   ONESHOT — every rank receives every input and reduces the whole vector.
 *   AUTO    — the measured selector picks per (world, bytes). */
typedef enum {
  NVRAR_ALGO_AUTO = 0,
  NVRAR_ALGO_HIER = 1,
  NVRAR_ALGO_TWOSHOT = 2,
  NVRAR_ALGO_ONESHOT = 3,
  /* virtual ranks sharing ONE device (nvrar_allreduce_local with every rank
   * present): no exchange — each unit is folded once, in the same order, from
   * all ranks' inputs and written to every rank's output. Elsewhere: HIER. */
  NVRAR_ALGO_DIRECT = 4,
  /* one-shot whose pushes go through an NVSwitch multicast (NVLS) mapping:
   * one 16-byte multimem store per cell reaches every rank (egress M instead
   * of (P-1)M). Needs nvrar_mc_attach; float32/bf16 with the
   * Lamport protocol, messages up to 1 MB; otherwise runs ONESHOT. */
  NVRAR_ALGO_MCAST = 5
} nvrar_algo_t;

/* Wire protocol. Both are self-validating (arrival of data = arrival of its
 * signal) and give identical results:
 *   LL      — the reference's fused word: 4-byte payload + 4-byte sequence flag
 *             per 8 bytes (fused.hpp:4-8); 2x wire bytes. Always used for int32.
 *   LAMPORT — raw payload (1x wire bytes); the all-ones bit pattern (a NaN) marks
 *             "not arrived", and an all-ones NaN input travels as another NaN.
 *   AUTO    — LAMPORT for float32/bf16, LL for int32. */
typedef enum { NVRAR_PROTO_AUTO = 0, NVRAR_PROTO_LL = 1, NVRAR_PROTO_LAMPORT = 2 } nvrar_proto_t;

/* One row of a measured selector table: messages of at most `max_bytes` run
 * `algo` (HIER / TWOSHOT / ONESHOT) on `blocks` CTAs per rank. */
typedef struct {
  uint64_t max_bytes;
  int algo;
  int blocks;
} nvrar_plan_entry;

/* Bootstrap collective supplied by the caller for nvrar_init: gather `bytes`
 * from every rank into recv (rank-major). Return 0 on success. */
typedef int (*nvrar_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes);

typedef struct {
  int world_size;
  int rank;               /* global rank = node * gpus_per_node + local */
  int nodes;              /* virtual nodes; power of two (nvrar.hpp:46) */
  int gpus_per_node;
  int device;             /* CUDA device ordinal this rank runs on */
  size_t max_bytes;       /* largest message; sizes the symmetric staging */
  int blocks;             /* default NvrarConfig.blocks (0 = selector) */
  uint64_t chunk_bytes;   /* default NvrarConfig.chunk_bytes (0 = 65536) */
  double timeout_s;       /* device watchdog (DeadlockError); 0 = 10 s */
  nvrar_allgather_fn allgather; /* used by nvrar_init only */
  void* allgather_ctx;
} nvrar_init_args;

typedef struct {
  unsigned char bytes[NVRAR_HANDLE_BYTES];
} nvrar_handle_t;

/* One blocked wait recorded by the device watchdog (BlockedRank,
 * errors.hpp:46-57). kind: 0 = FlagWait (data word), 1 = SeqWait (peer
 * sequence/length word), 2 = length mismatch, 3 = stale/future flag. */
typedef struct {
  int global_rank;
  int kind;
  int peer_rank;
  uint32_t expected;  /* awaited sequence number */
  uint64_t word_index;
  uint64_t observed;
  int status;         /* nvrar_status_t of the fault */
  int phase;          /* kernel phase: 2 push, 3 peer sync, 4 reduce/RD, 5 all-gather */
  int cta;            /* CTA index that recorded the wait */
} nvrar_blocked_t;

/* ---- lifecycle ---------------------------------------------------------- */
int nvrar_init(const nvrar_init_args* args, nvrar_comm_t* comm);
int nvrar_comm_create(const nvrar_init_args* args, nvrar_comm_t* comm);
int nvrar_comm_export(nvrar_comm_t comm, nvrar_handle_t* handle);
int nvrar_comm_connect(nvrar_comm_t comm, const nvrar_handle_t* handles, int count);
int nvrar_finalize(nvrar_comm_t comm);

/* ---- buffer registration (Ctx::alloc_region's symmetric regions for caller
 * data, transport.hpp:146-148) ---------------------------------
 * A caller's device buffer becomes peer-accessible in two steps, so the host
 * can use any bootstrap: nvrar_register_buffer exports this rank's range
 * (any range inside a cudaMalloc allocation) as an opaque handle and returns
 * its id; after an all-gather of the handles, nvrar_connect_buffer maps every
 * peer's range (CUDA IPC; same-process ranks directly) — once per
 * registration (a second call, or one after a failed call, is
 * INVALID_ARGUMENT: deregister and register again). Symmetric: every rank
 * registers the same number of bytes, in the same order (ids then agree).
 * Registered inputs can be all-reduced in place (nvrar_allreduce_registered);
 * nvrar_buffer_peer_ptr gives the caller peer rank p's range as mapped here.
 * nvrar_deregister_buffer (not collective; synchronises the device) unmaps.
 * The caller keeps registered memory alive until it deregisters or finalizes. */
int nvrar_register_buffer(nvrar_comm_t comm, void* dev_ptr, size_t bytes,
                          nvrar_handle_t* handle, int* buf);
int nvrar_connect_buffer(nvrar_comm_t comm, int buf, const nvrar_handle_t* handles, int count);
int nvrar_deregister_buffer(nvrar_comm_t comm, int buf);
int nvrar_buffer_peer_ptr(nvrar_comm_t comm, int buf, int peer, void** ptr);
/* Symmetric allocation (Ctx::alloc_region itself): collective — every rank
 * calls it in the same order with the same size; the memory is zeroed,
 * registered and connected through the allgather callback the comm was
 * created with (nvrar_init; a comm from nvrar_comm_create has none and gets
 * INVALID_ARGUMENT), and freed by nvrar_finalize. */
int nvrar_alloc_symmetric(nvrar_comm_t comm, size_t bytes, void** dev_ptr);

/* ---- the collective ----------------------------------------------------- */
int nvrar_allreduce(nvrar_comm_t comm, const void* send, void* recv, size_t count,
                    nvrar_dtype_t dtype, nvrar_op_t op, void* stream);

/* All-reduce whose INPUT lies in a registered, connected buffer (at the same
 * offset on every rank): no staging — every rank reads its peers' inputs in
 * place over NVLink and folds them in the reference order (same bits as
 * nvrar_allreduce). The launch completes only after every peer has finished
 * reading this rank's input, so the caller may overwrite it right after.
 * Consumes one sequence number like any call; world <= 32. */
int nvrar_allreduce_registered(nvrar_comm_t comm, const void* send, void* recv, size_t count,
                               nvrar_dtype_t dtype, nvrar_op_t op, void* stream);

/* All ranks that live on ONE device (virtual ranks sharing a GPU) in ONE
 * launch: cooperative when the schedule makes ranks wait on each other (so
 * they are co-resident); with every rank present the default is the DIRECT
 * schedule (no waits). comms[i] runs send[i] -> recv[i]. `active_mask` bit i clear
 * means comms[i] does not take part in this call (a stalled rank, used by
 * the peer-only-sync fixture); pass ~0ull for all. */
int nvrar_allreduce_local(nvrar_comm_t* comms, int ncomms, const void* const* send,
                          void* const* recv, size_t count, nvrar_dtype_t dtype, nvrar_op_t op,
                          void* stream, uint64_t active_mask);

/* Host buffers — the reference's own API shape (NvrarAllreduce<T>::run over
 * host spans, nvrar.hpp:84-129): host_send / host_recv are HOST memory. Pinned
 * (device-mapped) buffers are used in place: the kernels read the inputs and
 * write the results over PCIe themselves (zero-copy; the transfers overlap the
 * exchange). Otherwise — or with an explicit nvrar_set_host_chunk — the vector
 * moves through device staging. The vector is processed in WINDOWS: one window
 * (one launch) unless it is longer than the comm's max_bytes or a host chunk is
 * set (nvrar_set_host_chunk, or NVRAR_HOST_CHUNK bytes per rank); with several
 * windows the staged path overlaps the H2D copy of window i+1, the all-reduce
 * of window i and the D2H copy of window i-1. The window schedule depends only
 * on (count, dtype, max_bytes, host chunk) — never on whether a rank's buffers
 * are pinned — so ranks mixing pinned and pageable memory issue the same
 * launches. Each window is reduced as a window of the whole vector, so the bits
 * equal nvrar_allreduce of all `count` elements. Vectors of 2^31 or more
 * elements are rejected (INVALID_ARGUMENT). Stream-ordered: host_recv is
 * complete once `stream` reaches this point. */
int nvrar_allreduce_host(nvrar_comm_t comm, const void* host_send, void* host_recv, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream);
/* Window (bytes per rank) of the host path for this comm; 0 = automatic.
 * Every rank must set the same value (the chunking is part of the call
 * sequence). For a local group, comms[0]'s value applies. */
int nvrar_set_host_chunk(nvrar_comm_t comm, size_t bytes);
int nvrar_allreduce_local_host(nvrar_comm_t* comms, int ncomms, const void* const* host_send,
                               void* const* host_recv, size_t count, nvrar_dtype_t dtype,
                               nvrar_op_t op, void* stream);

/* Fused epilogue for the TP-decode caller (x = x + all_reduce(a), SURVEY §8f
 * row 2): recv[i] = residual[i] + sum_r send_r[i], where the sum is the
 * all-reduce's own result (same bits as nvrar_allreduce) and the add is the
 * element type's (bf16: fp32 add of the two bf16 values, one RNE) — bit-
 * identical to the unfused all-reduce followed by an elementwise add, without
 * the extra kernel and memory pass. recv may alias residual (in place). */
int nvrar_allreduce_residual(nvrar_comm_t comm, const void* send, void* recv,
                             const void* residual, size_t count, nvrar_dtype_t dtype,
                             nvrar_op_t op, void* stream);
int nvrar_allreduce_local_residual(nvrar_comm_t* comms, int ncomms, const void* const* send,
                                   void* const* recv, const void* const* residual, size_t count,
                                   nvrar_dtype_t dtype, nvrar_op_t op, void* stream,
                                   uint64_t active_mask);

/* ---- the reference's baseline collectives --------------------------------
 * The same sum with the reduction ORDER of the reference's other two
 * all-reduces, for model validation against them (they run on the flat
 * schedules; NCCL remains the performance baseline):
 *   RING — RingAllreduce<T> (ring.hpp): ring fold over all P ranks in ring
 *          positions p -> rank (p mod N, p div N), chunk = ceil(n/P);
 *          P <= 8.
 *   TREE — TreeAllreduce<T> (tree.hpp:10-12): in[0] + (in[1] + (... + in[G-1]))
 *          per node, then the pairwise tree over nodes.
 * Bit-exact to tests/oracles.hpp ring_order_sum / tree_order_sum. */
typedef enum {
  NVRAR_ORDER_NVRAR = 0,
  NVRAR_ORDER_RING = 1,
  NVRAR_ORDER_TREE = 2
} nvrar_order_t;
int nvrar_ring_allreduce(nvrar_comm_t comm, const void* send, void* recv, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream);
int nvrar_tree_allreduce(nvrar_comm_t comm, const void* send, void* recv, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream);
/* nvrar_allreduce_local with an explicit nvrar_order_t. */
int nvrar_allreduce_local_order(nvrar_comm_t* comms, int ncomms, int order,
                                const void* const* send, void* const* recv, size_t count,
                                nvrar_dtype_t dtype, nvrar_op_t op, void* stream,
                                uint64_t active_mask);

/* ---- phase-only entry points --------------------------------------------
 * One phase of the hierarchical all-reduce on its own, run by the same kernel
 * code as nvrar_allreduce (debugging and phase-level parity). Each call
 * consumes one sequence number of the comm, like an all-reduce; all ranks must
 * issue the same sequence of calls. Participants are the rank's node group
 * (local ranks 0..gpus_per_node-1 of its node), in local-rank order. */
typedef enum {
  NVRAR_PHASE_ALL = 0,             /* the full all-reduce */
  NVRAR_PHASE_REDUCE_SCATTER = 1,  /* IntraReduceScatter<T>::run (nvrar.hpp:280-299) */
  NVRAR_PHASE_RD_INTER = 2,        /* NvrarAllreduce<T>::rd_inter (nvrar.hpp:132-155) */
  NVRAR_PHASE_ALL_GATHER = 3       /* IntraAllGather<T>::run (nvrar.hpp:348-364) */
} nvrar_phase_t;

/* Node-local sum of `count` elements; this rank (local rank g) receives chunk g
 * of the zero-padded vector: ceil(count / gpus_per_node) elements, in the
 * reference's fold order. count == 0 is INVALID_ARGUMENT (nvrar.hpp:282-284);
 * members' counts must agree, else PROTOCOL_FAULT. */
int nvrar_reduce_scatter(nvrar_comm_t comm, const void* send, void* recv_shard, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream);
/* Concatenate the node members' `shard_count`-element shards in local-rank
 * order into recv (gpus_per_node * shard_count elements). Shard lengths must
 * agree, else PROTOCOL_FAULT (collectives_test.cpp:226-237). */
int nvrar_all_gather(nvrar_comm_t comm, const void* shard, void* recv, size_t shard_count,
                     nvrar_dtype_t dtype, void* stream);
/* Inter-node recursive doubling only. `packed` holds this rank's shard as LL
 * words (data = low 32 bits, flag = high 32 bits) packed with sequence()+1;
 * `out` receives the reduced shard packed with that call number. A flag other
 * than the call's is PROTOCOL_FAULT. dtype: INT32 or FLOAT32. With one node
 * the words are copied unchanged (nvrar.hpp:140-143). */
int nvrar_rd_inter(nvrar_comm_t comm, const uint64_t* packed, uint64_t* out, size_t words,
                   nvrar_dtype_t dtype, void* stream);
/* The phase entry points for the virtual ranks of one device (as
 * nvrar_allreduce_local); `phase` is an nvrar_phase_t. */
int nvrar_phase_local(nvrar_comm_t* comms, int ncomms, int phase, const void* const* send,
                      void* const* recv, size_t count, nvrar_dtype_t dtype, void* stream,
                      uint64_t active_mask);

/* ---- NVLS multicast (optional; NVRAR_ALGO_MCAST) -------------------------
 * The host supplies memory bound to an NVSwitch multicast object (torch
 * symmetric memory, NCCL NVLS buffers, or its own cuMulticast* setup): the
 * multicast mapping `mc_base` (a store reaches every rank's copy) and this
 * rank's own mapping `local_base` of the same memory, at least
 * nvrar_mc_bytes() bytes, at the same offset on every rank. Collective: every
 * rank attaches before any rank selects NVRAR_ALGO_MCAST; the caller keeps the
 * memory alive until nvrar_finalize. attach(comm, NULL, NULL, 0) detaches
 * (when a peer failed to attach). */
int nvrar_mc_bytes(nvrar_comm_t comm, size_t* bytes);
int nvrar_mc_attach(nvrar_comm_t comm, void* mc_base, void* local_base, size_t bytes);
int nvrar_mc_ready(nvrar_comm_t comm, int* ready);

/* ---- config / introspection -------------------------------------------- */
/* NvrarConfig (fused.hpp:106-116), validated like the reference's (blocks >= 0
 * here, 0 = the selector's choice; chunk_bytes >= 8 and a multiple of 8).
 * `blocks` = CTAs per rank (the reference's independent block ranges).
 * `chunk_bytes` is accepted for the reference's call shape but does NOT change
 * the GPU schedule: the reference pipelines the recursive-doubling steps in
 * chunks of chunk_bytes (nvrar.hpp:193-220); the kernels forward every 16-byte
 * unit to the next step as soon as it is reduced, i.e. the pipeline already
 * runs at the finest granularity, and — as in the reference — results are
 * invariant to (blocks, chunk_bytes). */
int nvrar_set_config(nvrar_comm_t comm, int blocks, uint64_t chunk_bytes);
int nvrar_set_algo(nvrar_comm_t comm, nvrar_algo_t algo);
int nvrar_set_timeout(nvrar_comm_t comm, double timeout_s);
int nvrar_set_protocol(nvrar_comm_t comm, nvrar_proto_t proto);
/* Selected schedule and CTA count for a message (what nvrar_allreduce runs). */
int nvrar_plan(nvrar_comm_t comm, size_t count, nvrar_dtype_t dtype, int* algo, int* blocks);
/* The same for an nvrar_allreduce_local launch of the active comms (virtual
 * ranks of one device may take the DIRECT schedule). */
int nvrar_plan_local(nvrar_comm_t* comms, int ncomms, size_t count, nvrar_dtype_t dtype,
                     uint64_t active_mask, int* algo, int* blocks);
/* Install a measured selector table (ascending max_bytes; messages larger than
 * the last row fall back to the built-in policy). All ranks must install the
 * same table — paper_2511_09557_b200.selector.autotune() measures it with a
 * max-over-ranks consensus. n = 0 clears it. */
int nvrar_set_plan_table(nvrar_comm_t comm, const nvrar_plan_entry* entries, int n);
/* The same selector as a pure function (no device): every rank evaluates it
 * identically, which is what keeps all ranks on one schedule. */
int nvrar_plan_for(int world, int nodes, int gpus_per_node, size_t count, nvrar_dtype_t dtype,
                   int algo_pref, int blocks_pref, int max_ctas, int* algo, int* blocks);
/* Host-visible sequence number: synchronises with the device. */
int nvrar_get_sequence(nvrar_comm_t comm, uint32_t* seq);
/* Step-l exchange peers (global ranks), `steps` = log2(nodes). */
int nvrar_get_peers(nvrar_comm_t comm, int* peers, int max_peers, int* steps);
/* Synchronises the device and returns the sticky device status (0 = ok). */
int nvrar_check(nvrar_comm_t comm);
int nvrar_get_blocked(nvrar_comm_t comm, nvrar_blocked_t* out);
/* Diagnostics: phase timestamps (globaltimer ns) of CTA 0 of the last call,
 * recorded when profiling is on; and the NVLink signal latency probe — a flag
 * ping-pong with `peer` (both ranks call it; one with initiator = 1), which
 * returns the initiator's elapsed ns for `iters` round trips (alpha_signal =
 * elapsed / iters / 2, the latency floor of the roofline). */
int nvrar_set_profile(nvrar_comm_t comm, int on);
int nvrar_get_phase_times(nvrar_comm_t comm, uint64_t* ts, int n);
int nvrar_pingpong(nvrar_comm_t comm, int peer, int iters, int initiator, void* stream,
                   uint64_t* elapsed_ns);
/* Absolute %globaltimer stamps of the last ping-pong round on this rank:
 * initiator {last send, last receive}; responder {last receive, same}. With both
 * sides one can estimate the offset between the two GPUs' global timers. */
int nvrar_pingpong_clock(nvrar_comm_t comm, uint64_t* stamps);
/* Invariant check (tests): count the 8-byte words of the slot areas that are
 * not empty (all ones) — between calls every slot must be empty. Synchronises.
 * `first_offset` receives the byte offset of the first dirty word (or ~0). */
int nvrar_debug_dirty_cells(nvrar_comm_t comm, uint64_t* dirty, uint64_t* first_offset);
/* Debug: copy `bytes` of this rank's symmetric region at `offset` to host;
 * `layout` (if non-null) receives the 8 layout words (ctrl, a_off, a_src, b_off,
 * b_src, c_off, c_step, bytes). Synchronises. */
int nvrar_debug_read_region(nvrar_comm_t comm, uint64_t offset, uint64_t bytes, void* host,
                            uint64_t* layout);
/* Delay injection (tests; the reference's RunOptions::delay_max_us,
 * concurrent_transport.hpp:393-419, acceptance_test.cpp:314-330): every warp
 * sleeps a seeded pseudo-random 0..max_ns ns before its remote stores and
 * between unsatisfied polls, so adversarial interleavings are exercised. The
 * results must not change. max_ns = 0 turns it off; at most 1 ms. */
int nvrar_set_jitter(nvrar_comm_t comm, uint32_t max_ns, uint32_t seed);
/* Word-atomicity canary (acceptance_test.cpp:338-364): the writer (writer = 1)
 * streams `iters` 16-byte fused cells into `peer`'s canary cell, the reader
 * (the peer, writer = 0, launched first or concurrently) checks every cell it
 * observes for tearing. Asynchronous on `stream` (the two sides may be comms
 * of one process on two streams); nvrar_debug_canary_result synchronises and
 * gives the torn observations (reader) or 0 (writer). Both sides call it the
 * same number of times per pair. */
int nvrar_debug_canary(nvrar_comm_t comm, int peer, int iters, int writer, uint32_t jitter_ns,
                       uint32_t seed, void* stream);
int nvrar_debug_canary_result(nvrar_comm_t comm, uint32_t* torn);
/* Debug: the per-CTA replicas of the call counter (all equal between calls). */
int nvrar_debug_seq_slots(nvrar_comm_t comm, uint32_t* out, int n);
const char* nvrar_last_error(nvrar_comm_t comm);
const char* nvrar_status_string(int status);
int nvrar_abi_version(void);
size_t nvrar_symmetric_bytes(nvrar_comm_t comm);

#ifdef __cplusplus
}
#endif

#endif /* NVRAR_H */
