// Reference-side binding: a drop-in for ccsim::NvrarAllreduce<T>
// (/root/reference/proj/include/ccsim/collectives/nvrar.hpp:41-250) that runs
// the all-reduce on B200s through the C ABI in include/nvrar.h.
//
// This is the header a maintainer of the reference would add next to
// collectives/nvrar.hpp. It keeps the reference's names, argument meaning and
// exception types (errors.hpp); the transport context (Ctx) is replaced by
// real GPUs: one process per GPU, a bootstrap allgather supplied by the host
// program (MPI, torch.distributed, a file store...).
//
// Differences a caller must know:
//  * buffers are DEVICE pointers (std::span over device memory), and run() is
//    stream-ordered; run() synchronises the stream and checks the device
//    status so that faults surface as the reference's exceptions;
//  * the DeadlockError blocked set carries this rank's entry only (each
//    process sees its own watchdog record); the all-ranks view is
//    LocalGroup.check() on one device or a host-side gather.
#pragma once

#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ccsim/collectives/fused.hpp"  // Element, NvrarConfig
#include "ccsim/errors.hpp"
#include "ccsim/topology.hpp"
#include "nvrar.h"

namespace ccsim {

template <Element T>
class NvrarB200Allreduce {
 public:
  using Allgather = nvrar_allgather_fn;

  NvrarB200Allreduce(const ClusterTopology& topo, int rank, int device, std::size_t max_elems,
                     Allgather allgather, void* allgather_ctx, double timeout_s = 5.0)
      : max_elems_(max_elems) {
    topo.require_power_of_two_nodes("nvrar");  // InvalidTopologyError, nvrar.hpp:46
    nvrar_init_args a{};
    a.world_size = topo.world_size();
    a.rank = rank;
    a.nodes = topo.nodes;
    a.gpus_per_node = topo.gpus_per_node;
    a.device = device;
    a.max_bytes = std::max<std::size_t>(max_elems, 1) * sizeof(T);
    a.timeout_s = timeout_s;
    a.allgather = allgather;
    a.allgather_ctx = allgather_ctx;
    throw_on(nvrar_init(&a, &comm_), nullptr);
  }
  NvrarB200Allreduce(const NvrarB200Allreduce&) = delete;
  NvrarB200Allreduce& operator=(const NvrarB200Allreduce&) = delete;
  ~NvrarB200Allreduce() { nvrar_finalize(comm_); }

  std::uint32_t sequence() const {
    std::uint32_t s = 0;
    throw_on(nvrar_get_sequence(comm_, &s), comm_);
    return s;
  }

  /// Same contract as NvrarAllreduce<T>::run (nvrar.hpp:84-129), on device memory.
  void run(std::span<const T> in, std::span<T> out, const NvrarConfig& cfg = {},
           void* stream = nullptr) {
    cfg.validate();
    if (in.size() != out.size()) {
      throw InvalidArgumentError("nvrar: input and output lengths differ");
    }
    if (in.size() > max_elems_) {
      throw InvalidArgumentError("nvrar: vector longer than the preallocated maximum");
    }
    throw_on(nvrar_set_config(comm_, cfg.blocks, cfg.chunk_bytes), comm_);
    throw_on(nvrar_allreduce(comm_, in.data(), out.data(), in.size(), dtype(), NVRAR_SUM, stream),
             comm_);
    throw_on(nvrar_check(comm_), comm_);  // synchronises; device faults -> exceptions
  }

  /// The reference's exact call shape: HOST spans in and out (nvrar.hpp:84-129).
  /// Pinned host memory (cudaHostRegister / cudaMallocHost) is used in place by
  /// the kernels (zero-copy over PCIe); pageable memory is staged through device
  /// memory. Either way the bits equal run() on device buffers.
  void run_host(std::span<const T> in, std::span<T> out, const NvrarConfig& cfg = {},
                void* stream = nullptr) {
    cfg.validate();
    if (in.size() != out.size()) {
      throw InvalidArgumentError("nvrar: input and output lengths differ");
    }
    if (in.size() > max_elems_) {
      throw InvalidArgumentError("nvrar: vector longer than the preallocated maximum");
    }
    throw_on(nvrar_set_config(comm_, cfg.blocks, cfg.chunk_bytes), comm_);
    throw_on(nvrar_allreduce_host(comm_, in.data(), out.data(), in.size(), dtype(), NVRAR_SUM,
                                  stream),
             comm_);
    throw_on(nvrar_check(comm_), comm_);  // synchronises: `out` is complete on return
  }

  /// Inter-node phase only (NvrarAllreduce<T>::rd_inter, nvrar.hpp:132-155):
  /// `packed` = this rank's shard as fused words {data, seq} packed with
  /// sequence()+1; `out` receives the reduced shard packed with that call.
  void rd_inter(std::span<const std::uint64_t> packed, std::span<std::uint64_t> out,
                const NvrarConfig& cfg = {}, void* stream = nullptr) {
    cfg.validate();
    if (packed.size() != out.size()) throw InvalidArgumentError("rd_inter: bad shard length");
    throw_on(nvrar_set_config(comm_, cfg.blocks, cfg.chunk_bytes), comm_);
    throw_on(nvrar_rd_inter(comm_, packed.data(), out.data(), packed.size(), dtype(), stream),
             comm_);
    throw_on(nvrar_check(comm_), comm_);
  }

  /// IntraReduceScatter<T>::run (nvrar.hpp:280-299) over this rank's node:
  /// `shard` gets ceil(n / gpus_per_node) elements of the node-local sum.
  void reduce_scatter(std::span<const T> in, std::span<T> shard, void* stream = nullptr) {
    throw_on(nvrar_reduce_scatter(comm_, in.data(), shard.data(), in.size(), dtype(), NVRAR_SUM,
                                  stream),
             comm_);
    throw_on(nvrar_check(comm_), comm_);
  }

  /// IntraAllGather<T>::run (nvrar.hpp:348-364) over this rank's node.
  void all_gather(std::span<const T> shard, std::span<T> out, void* stream = nullptr) {
    throw_on(nvrar_all_gather(comm_, shard.data(), out.data(), shard.size(), dtype(), stream),
             comm_);
    throw_on(nvrar_check(comm_), comm_);
  }

  /// The result bits of RingAllreduce<T>::run / TreeAllreduce<T>::run
  /// (ring.hpp, tree.hpp) on the same communicator.
  void run_ring(std::span<const T> in, std::span<T> out, void* stream = nullptr) {
    throw_on(nvrar_ring_allreduce(comm_, in.data(), out.data(), in.size(), dtype(), NVRAR_SUM,
                                  stream),
             comm_);
    throw_on(nvrar_check(comm_), comm_);
  }
  void run_tree(std::span<const T> in, std::span<T> out, void* stream = nullptr) {
    throw_on(nvrar_tree_allreduce(comm_, in.data(), out.data(), in.size(), dtype(), NVRAR_SUM,
                                  stream),
             comm_);
    throw_on(nvrar_check(comm_), comm_);
  }

  /// Step-l exchange peers (nvrar.hpp:158).
  std::vector<RankId> peers(const ClusterTopology& topo) const {
    int p[8];
    int steps = 0;
    throw_on(nvrar_get_peers(comm_, p, 8, &steps), comm_);
    std::vector<RankId> out;
    for (int l = 0; l < steps; ++l) out.push_back(RankId::from_global(p[l], topo));
    return out;
  }

 private:
  static constexpr nvrar_dtype_t dtype() {
    return std::same_as<T, float> ? NVRAR_FLOAT32 : NVRAR_INT32;
  }

  static void throw_on(int rc, nvrar_comm_t comm) {
    if (rc == NVRAR_SUCCESS) return;
    const std::string msg = nvrar_last_error(comm);
    switch (rc) {
      case NVRAR_ERR_INVALID_ARGUMENT: throw InvalidArgumentError(msg);
      case NVRAR_ERR_INVALID_TOPOLOGY: throw InvalidTopologyError(msg);
      case NVRAR_ERR_PROTOCOL_FAULT: throw ProtocolFaultError(msg);
      case NVRAR_ERR_DEADLOCK: {
        nvrar_blocked_t b{};
        nvrar_get_blocked(comm, &b);
        BlockedRank br;
        br.global_rank = b.global_rank;
        br.kind = b.kind == 1 ? BlockedRank::Kind::SeqWait : BlockedRank::Kind::FlagWait;
        br.peer_rank = b.peer_rank;
        br.word_index = b.word_index;
        br.expected = b.expected;
        throw DeadlockError({br});
      }
      default: throw std::runtime_error("nvrar: " + msg);
    }
  }

  nvrar_comm_t comm_ = nullptr;
  std::size_t max_elems_;
};

/// Drop-ins for the reference's baseline collectives (RingAllreduce<T>,
/// TreeAllreduce<T>): the same constructor as NvrarB200Allreduce, `run(in, out)`
/// gives the reference's result bits for that algorithm's reduction order.
template <Element T>
class B200RingAllreduce {
 public:
  template <class... A>
  explicit B200RingAllreduce(A&&... a) : impl_(std::forward<A>(a)...) {}
  void run(std::span<const T> in, std::span<T> out, void* stream = nullptr) {
    impl_.run_ring(in, out, stream);
  }
  std::uint32_t sequence() const { return impl_.sequence(); }

 private:
  NvrarB200Allreduce<T> impl_;
};

template <Element T>
class B200TreeAllreduce {
 public:
  template <class... A>
  explicit B200TreeAllreduce(A&&... a) : impl_(std::forward<A>(a)...) {}
  void run(std::span<const T> in, std::span<T> out, void* stream = nullptr) {
    impl_.run_tree(in, out, stream);
  }
  std::uint32_t sequence() const { return impl_.sequence(); }

 private:
  NvrarB200Allreduce<T> impl_;
};

}  // namespace ccsim
