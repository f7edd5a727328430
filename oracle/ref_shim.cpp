// TEST INFRASTRUCTURE ONLY — a C shim over the UNMODIFIED reference headers.
//
// Built by oracle/Makefile straight from /root/reference/proj/include and
// /root/reference/proj/tests (nothing is copied into this repo) into
// oracle/_ref/libccsim_ref.so. It exposes the reference's own NVRAR
// implementation "all ranks at once" (the reference runs every rank inside one
// process: run.hpp:15-24), so tests can pin the C restatement
// (oracle/nvrar_oracle.c) and generate tests/golden/ fixtures, and bench.py's
// reference arm can time ccsim::NvrarAllreduce on ConcurrentEngine.
//
// Return codes mirror include/nvrar.h: 0 ok, 1 internal, 2 invalid argument,
// 3 invalid topology, 4 protocol fault, 5 deadlock.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "ccsim/collectives.hpp"
#include "ccsim/run.hpp"
#include "oracles.hpp"

using namespace ccsim;

namespace {

void put_err(char* err, std::size_t len, const std::string& s) {
  if (!err || len == 0) return;
  std::snprintf(err, len, "%s", s.c_str());
}

template <class F>
int guarded(char* err, std::size_t len, F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidTopologyError& e) {
    put_err(err, len, e.what());
    return 3;
  } catch (const InvalidArgumentError& e) {
    put_err(err, len, e.what());
    return 2;
  } catch (const ProtocolFaultError& e) {
    put_err(err, len, e.what());
    return 4;
  } catch (const DeadlockError& e) {
    put_err(err, len, e.what());
    return 5;
  } catch (const std::exception& e) {
    put_err(err, len, e.what());
    return 1;
  }
}

template <Element T>
std::vector<std::vector<T>> unflatten(const T* p, int ranks, std::size_t n) {
  std::vector<std::vector<T>> v(ranks);
  for (int r = 0; r < ranks; ++r) v[r].assign(p + static_cast<std::size_t>(r) * n,
                                              p + static_cast<std::size_t>(r + 1) * n);
  return v;
}

template <Element T>
int run_all(int nodes, int gpus, std::size_t n, const T* inputs, T* outputs, int blocks,
            std::uint64_t chunk, int mode, std::uint64_t seed, double delay_us,
            double timeout_s, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ClusterTopology topo{nodes, gpus};
    topo.validate();
    const int ng = topo.world_size();
    auto in = unflatten(inputs, ng, n);
    std::vector<std::vector<T>> out(ng, std::vector<T>(n));
    const NvrarConfig cfg{blocks, chunk};
    auto program = [&](Ctx& ctx) -> Task {
      const int me = ctx.global();
      NvrarAllreduce<T> coll(ctx, n);
      co_await coll.run(std::span<const T>(in[me]), std::span<T>(out[me]), cfg);
    };
    RunOptions opts;
    opts.seed = seed;
    opts.delay_max_us = mode == 1 ? delay_us : 0.0;
    opts.timeout_s = timeout_s;
    CostParams params;  // latency_only() of collectives_test.cpp:19-24
    params.alpha_intra = 0.5e-6;
    params.alpha_inter = 2.0e-6;
    run_ranks(topo, mode == 1 ? CostParams{} : params, mode == 1 ? TransportMode::Concurrent
                                           : TransportMode::VirtualTime,
              opts, program);
    for (int r = 0; r < ng; ++r) {
      std::memcpy(outputs + static_cast<std::size_t>(r) * n, out[r].data(), n * sizeof(T));
    }
  });
}

// The standalone phases through the reference's own classes on VirtualTime:
// IntraReduceScatter / IntraAllGather with each node's members as participants
// (nvrar.hpp:254-373), and NvrarAllreduce::rd_inter on fused-packed shards
// (nvrar.hpp:132-155; the collectives_test.cpp:286-302 driver).
template <Element T>
int intra_phase(int which, int nodes, int gpus, std::size_t len, const T* inputs, T* outputs,
                char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ClusterTopology topo{nodes, gpus};
    topo.validate();
    const int ng = topo.world_size();
    const std::size_t ce = which == 0 ? (len + gpus - 1) / gpus : len;
    const std::size_t out_len = which == 0 ? ce : len * gpus;
    auto in = unflatten(inputs, ng, len);
    std::vector<std::vector<T>> out(ng, std::vector<T>(out_len));
    auto program = [&](Ctx& ctx) -> Task {
      const int me = ctx.global();
      std::vector<RankId> mates;
      for (int g = 0; g < gpus; ++g) mates.push_back(RankId{ctx.self().node_rank, g});
      if (which == 0) {
        IntraReduceScatter<T> rs(ctx, len, mates);
        co_await rs.run(std::span<const T>(in[me]), std::span<T>(out[me]));
      } else {
        IntraAllGather<T> ag(ctx, len, mates);
        co_await ag.run(std::span<const T>(in[me]), std::span<T>(out[me]));
      }
    };
    run_ranks(topo, CostParams{}, TransportMode::VirtualTime, {}, program);
    for (int r = 0; r < ng; ++r) {
      std::memcpy(outputs + static_cast<std::size_t>(r) * out_len, out[r].data(),
                  out_len * sizeof(T));
    }
  });
}

template <Element T>
int rd_inter_all(int nodes, int gpus, std::size_t w, const T* shards, T* outputs, int blocks,
                 std::uint64_t chunk, char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ClusterTopology topo{nodes, gpus};
    topo.validate();
    const int ng = topo.world_size();
    auto in = unflatten(shards, ng, w);
    std::vector<std::vector<T>> out(ng);
    const NvrarConfig cfg{blocks, chunk};
    auto program = [&](Ctx& ctx) -> Task {
      const int me = ctx.global();
      NvrarAllreduce<T> st(ctx, w * ctx.topo().gpus_per_node);
      auto packed = pack_fused<T>(in[me], st.sequence() + 1);
      std::vector<std::uint64_t> reduced(w);
      co_await st.rd_inter(packed, reduced, cfg);
      out[me] = unpack_fused<T>(reduced, st.sequence());
    };
    run_ranks(topo, CostParams{}, TransportMode::VirtualTime, {}, program);
    for (int r = 0; r < ng; ++r) {
      std::memcpy(outputs + static_cast<std::size_t>(r) * w, out[r].data(), w * sizeof(T));
    }
  });
}

// RingAllreduce<T> / TreeAllreduce<T> (ring.hpp, tree.hpp) on every rank.
template <Element T>
int baseline_all(int which, int nodes, int gpus, std::size_t n, const T* inputs, T* outputs,
                 char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ClusterTopology topo{nodes, gpus};
    topo.validate();
    const int ng = topo.world_size();
    auto in = unflatten(inputs, ng, n);
    std::vector<std::vector<T>> out(ng, std::vector<T>(n));
    auto program = [&](Ctx& ctx) -> Task {
      const int me = ctx.global();
      if (which == 0) {
        RingAllreduce<T> coll(ctx, n);
        co_await coll.run(std::span<const T>(in[me]), std::span<T>(out[me]));
      } else {
        TreeAllreduce<T> coll(ctx, n);
        co_await coll.run(std::span<const T>(in[me]), std::span<T>(out[me]));
      }
    };
    run_ranks(topo, CostParams{}, TransportMode::VirtualTime, {}, program);
    for (int r = 0; r < ng; ++r) {
      std::memcpy(outputs + static_cast<std::size_t>(r) * n, out[r].data(), n * sizeof(T));
    }
  });
}

// Times NvrarAllreduce<T>::run on ConcurrentEngine with pre-generated inputs
// (unlike run_bench_point, which generates inputs inside its timed loop,
// bench.hpp:92-93). Per call: makespan = max over ranks of the wall time at
// which the rank's run() returned (the reference's own convention,
// bench.hpp:116-122); per_call_us[i] = makespan[i] - makespan[i-1].
template <Element T>
int time_concurrent(int nodes, int gpus, std::size_t n, const T* inputs, int blocks,
                    std::uint64_t chunk, int warmup, int calls, double* per_call_us,
                    char* err, std::size_t errlen) {
  return guarded(err, errlen, [&] {
    const ClusterTopology topo{nodes, gpus};
    topo.validate();
    const int ng = topo.world_size();
    auto in = unflatten(inputs, ng, n);
    const int total = warmup + calls;
    std::vector<std::vector<double>> fin(total, std::vector<double>(ng, 0.0));
    const NvrarConfig cfg{blocks, chunk};
    auto program = [&](Ctx& ctx) -> Task {
      const int me = ctx.global();
      NvrarAllreduce<T> coll(ctx, n);
      std::vector<T> out(n);
      for (int it = 0; it < total; ++it) {
        co_await coll.run(std::span<const T>(in[me]), std::span<T>(out), cfg);
        fin[it][me] = ctx.now_us();
      }
    };
    RunOptions opts;
    opts.timeout_s = 60.0;
    run_ranks(topo, CostParams{}, TransportMode::Concurrent, opts, program);
    auto makespan = [&](int it) { return *std::max_element(fin[it].begin(), fin[it].end()); };
    for (int i = 0; i < calls; ++i) {
      const int it = warmup + i;
      const double before = it == 0 ? 0.0 : makespan(it - 1);
      per_call_us[i] = makespan(it) - before;
    }
  });
}

}  // namespace

extern "C" {

void ref_random_inputs_f32(int ranks, std::size_t n, std::uint64_t seed, float* out) {
  auto v = oracles::random_inputs<float>(ranks, n, seed);
  for (int r = 0; r < ranks; ++r) std::memcpy(out + r * n, v[r].data(), n * sizeof(float));
}

void ref_random_inputs_i32(int ranks, std::size_t n, std::uint64_t seed, std::int32_t* out) {
  auto v = oracles::random_inputs<std::int32_t>(ranks, n, seed);
  for (int r = 0; r < ranks; ++r) {
    std::memcpy(out + r * n, v[r].data(), n * sizeof(std::int32_t));
  }
}

int ref_nvrar_order_sum_f32(int nodes, int gpus, std::size_t n, const float* inputs,
                            float* out) {
  const ClusterTopology topo{nodes, gpus};
  auto v = oracles::nvrar_order_sum(unflatten(inputs, nodes * gpus, n), topo);
  std::memcpy(out, v.data(), n * sizeof(float));
  return 0;
}

int ref_nvrar_order_sum_i32(int nodes, int gpus, std::size_t n, const std::int32_t* inputs,
                            std::int32_t* out) {
  const ClusterTopology topo{nodes, gpus};
  auto v = oracles::nvrar_order_sum(unflatten(inputs, nodes * gpus, n), topo);
  std::memcpy(out, v.data(), n * sizeof(std::int32_t));
  return 0;
}

void ref_serial_sum_f32(int ranks, std::size_t n, const float* inputs, float* out) {
  auto v = oracles::serial_sum(unflatten(inputs, ranks, n));
  std::memcpy(out, v.data(), n * sizeof(float));
}

int ref_nvrar_run_all_f32(int nodes, int gpus, std::size_t n, const float* inputs,
                          float* outputs, int blocks, std::uint64_t chunk, int mode,
                          std::uint64_t seed, double delay_us, double timeout_s, char* err,
                          std::size_t errlen) {
  return run_all<float>(nodes, gpus, n, inputs, outputs, blocks, chunk, mode, seed, delay_us,
                        timeout_s, err, errlen);
}

int ref_nvrar_run_all_i32(int nodes, int gpus, std::size_t n, const std::int32_t* inputs,
                          std::int32_t* outputs, int blocks, std::uint64_t chunk, int mode,
                          std::uint64_t seed, double delay_us, double timeout_s, char* err,
                          std::size_t errlen) {
  return run_all<std::int32_t>(nodes, gpus, n, inputs, outputs, blocks, chunk, mode, seed,
                               delay_us, timeout_s, err, errlen);
}

int ref_ring_run_all_f32(int nodes, int gpus, std::size_t n, const float* in, float* out,
                         char* err, std::size_t errlen) {
  return baseline_all<float>(0, nodes, gpus, n, in, out, err, errlen);
}
int ref_ring_run_all_i32(int nodes, int gpus, std::size_t n, const std::int32_t* in,
                         std::int32_t* out, char* err, std::size_t errlen) {
  return baseline_all<std::int32_t>(0, nodes, gpus, n, in, out, err, errlen);
}
int ref_tree_run_all_f32(int nodes, int gpus, std::size_t n, const float* in, float* out,
                         char* err, std::size_t errlen) {
  return baseline_all<float>(1, nodes, gpus, n, in, out, err, errlen);
}
int ref_tree_run_all_i32(int nodes, int gpus, std::size_t n, const std::int32_t* in,
                         std::int32_t* out, char* err, std::size_t errlen) {
  return baseline_all<std::int32_t>(1, nodes, gpus, n, in, out, err, errlen);
}

int ref_intra_rs_f32(int nodes, int gpus, std::size_t n, const float* in, float* out, char* err,
                     std::size_t errlen) {
  return intra_phase<float>(0, nodes, gpus, n, in, out, err, errlen);
}
int ref_intra_rs_i32(int nodes, int gpus, std::size_t n, const std::int32_t* in,
                     std::int32_t* out, char* err, std::size_t errlen) {
  return intra_phase<std::int32_t>(0, nodes, gpus, n, in, out, err, errlen);
}
int ref_intra_ag_f32(int nodes, int gpus, std::size_t ce, const float* in, float* out, char* err,
                     std::size_t errlen) {
  return intra_phase<float>(1, nodes, gpus, ce, in, out, err, errlen);
}
int ref_intra_ag_i32(int nodes, int gpus, std::size_t ce, const std::int32_t* in,
                     std::int32_t* out, char* err, std::size_t errlen) {
  return intra_phase<std::int32_t>(1, nodes, gpus, ce, in, out, err, errlen);
}
int ref_rd_inter_f32(int nodes, int gpus, std::size_t w, const float* in, float* out, int blocks,
                     std::uint64_t chunk, char* err, std::size_t errlen) {
  return rd_inter_all<float>(nodes, gpus, w, in, out, blocks, chunk, err, errlen);
}
int ref_rd_inter_i32(int nodes, int gpus, std::size_t w, const std::int32_t* in,
                     std::int32_t* out, int blocks, std::uint64_t chunk, char* err,
                     std::size_t errlen) {
  return rd_inter_all<std::int32_t>(nodes, gpus, w, in, out, blocks, chunk, err, errlen);
}

int ref_nvrar_time_concurrent_f32(int nodes, int gpus, std::size_t n, const float* inputs,
                                  int blocks, std::uint64_t chunk, int warmup, int calls,
                                  double* per_call_us, char* err, std::size_t errlen) {
  return time_concurrent<float>(nodes, gpus, n, inputs, blocks, chunk, warmup, calls,
                                per_call_us, err, errlen);
}

// The stalled-rank fixture (collectives_test.cpp:462-497; acceptance_test.cpp:268-310):
// every rank runs call 1, then every rank except `stall_rank` runs call 2.
// Writes the blocked set as rows {global_rank, kind(0 flag,1 seq), peer, expected}.
int ref_nvrar_stalled_rank(int nodes, int gpus, std::size_t n, int stall_rank,
                           std::uint64_t seed1, std::uint64_t seed2, int* rows, int max_rows,
                           int* n_rows, char* err, std::size_t errlen) {
  *n_rows = 0;
  try {
    const ClusterTopology topo{nodes, gpus};
    const int ng = topo.world_size();
    auto in1 = oracles::random_inputs<std::int32_t>(ng, n, seed1);
    auto in2 = oracles::random_inputs<std::int32_t>(ng, n, seed2);
    auto program = [&](Ctx& ctx) -> Task {
      const int me = ctx.global();
      NvrarAllreduce<std::int32_t> st(ctx, n);
      std::vector<std::int32_t> first(n), second(n);
      co_await st.run(std::span<const std::int32_t>(in1[me]), std::span<std::int32_t>(first),
                      {});
      if (me == stall_rank) co_return;
      co_await st.run(std::span<const std::int32_t>(in2[me]), std::span<std::int32_t>(second),
                      {});
    };
    CostParams params;  // latency_only() of collectives_test.cpp:19-24
    params.alpha_intra = 0.5e-6;
    params.alpha_inter = 2.0e-6;
    run_ranks(topo, params, TransportMode::VirtualTime, {}, program);
    return 0;
  } catch (const DeadlockError& e) {
    int k = 0;
    for (const auto& b : e.blocked()) {
      if (k >= max_rows) break;
      rows[4 * k + 0] = b.global_rank;
      rows[4 * k + 1] = b.kind == BlockedRank::Kind::FlagWait ? 0 : 1;
      rows[4 * k + 2] = b.peer_rank;
      rows[4 * k + 3] = static_cast<int>(b.expected >> 32 ? b.expected >> 32 : b.expected);
      ++k;
    }
    *n_rows = k;
    put_err(err, errlen, e.what());
    return 5;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return 1;
  }
}

}  // extern "C"

#ifdef CCSIM_REF_TOOL
// oracle/_ref/ref_tool: `ref_tool stalled N G n stall seed1 seed2` prints the
// blocked set, one "rank kind peer expected" row per line. (Run as a separate
// process: the deadlock unwind of the virtual-time engine crashes when driven
// through ctypes from the Python interpreter, though it is clean standalone.)
#include <cstdlib>
int main(int argc, char** argv) {
  if (argc != 8 || std::string(argv[1]) != "stalled") return 2;
  int rows[256];
  int nr = 0;
  char err[1024] = {0};
  int rc = ref_nvrar_stalled_rank(std::atoi(argv[2]), std::atoi(argv[3]),
                                  std::strtoull(argv[4], nullptr, 10), std::atoi(argv[5]),
                                  std::strtoull(argv[6], nullptr, 10),
                                  std::strtoull(argv[7], nullptr, 10), rows, 64, &nr, err, 1024);
  std::printf("rc %d\n", rc);
  for (int i = 0; i < nr; ++i) {
    std::printf("%d %d %d %d\n", rows[4 * i], rows[4 * i + 1], rows[4 * i + 2], rows[4 * i + 3]);
  }
  std::printf("msg %s\n", err);
  return 0;
}
#endif
