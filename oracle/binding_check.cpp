// TEST INFRASTRUCTURE ONLY (built by `make -C oracle ref` into oracle/_ref/,
// never shipped as product): one rank of the reference-side C++ binding
// (integration/ccsim_nvrar_b200.hpp, the drop-in for ccsim::NvrarAllreduce<T>)
// running real all-reduces on a GPU, checked bit for bit against the
// reference's own oracle (tests/oracles.hpp: random_inputs, nvrar_order_sum).
//
//   binding_check <dir> <rank> <nodes> <gpus> <device>
//
// Ranks are separate processes; the bootstrap all-gather the binding asks for
// is a shared directory. Exit 0 = every result bit-exact.
#include <cuda_runtime.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "ccsim_nvrar_b200.hpp"
#include "oracles.hpp"

namespace {

struct FileGather {
  std::string dir;
  int rank, world;
  int round = 0;
};

// nvrar_allgather_fn over files <dir>/g<round>_<rank> (atomic rename)
int file_allgather(void* ctx, const void* send, void* recv, size_t bytes) {
  auto* g = static_cast<FileGather*>(ctx);
  const int r = g->round++;
  const std::string mine = g->dir + "/g" + std::to_string(r) + "_" + std::to_string(g->rank);
  {
    std::ofstream f(mine + ".tmp", std::ios::binary);
    f.write(static_cast<const char*>(send), static_cast<std::streamsize>(bytes));
  }
  std::rename((mine + ".tmp").c_str(), mine.c_str());
  for (int q = 0; q < g->world; ++q) {
    const std::string p = g->dir + "/g" + std::to_string(r) + "_" + std::to_string(q);
    for (int t = 0;; ++t) {
      std::ifstream f(p, std::ios::binary);
      if (f && f.read(static_cast<char*>(recv) + q * bytes, static_cast<std::streamsize>(bytes))) {
        break;
      }
      if (t > 60000) return 1;
      std::this_thread::sleep_for(std::chrono::milliseconds(2));
    }
  }
  return 0;
}

template <class T>
int check(ccsim::NvrarB200Allreduce<T>& ar, int rank, int nodes, int gpus, std::size_t n,
          std::uint64_t seed, bool host) {
  const int world = nodes * gpus;
  const auto in = oracles::random_inputs<T>(world, n, seed);
  const auto want = oracles::nvrar_order_sum<T>(in, ccsim::ClusterTopology{nodes, gpus});
  std::vector<T> got(n);
  if (host) {
    ar.run_host(std::span<const T>(in[rank]), std::span<T>(got));  // host spans, the reference's shape
  } else {
    T *d_in = nullptr, *d_out = nullptr;
    cudaMalloc(&d_in, n * sizeof(T));
    cudaMalloc(&d_out, n * sizeof(T));
    cudaMemcpy(d_in, in[rank].data(), n * sizeof(T), cudaMemcpyHostToDevice);
    ar.run(std::span<const T>(d_in, n), std::span<T>(d_out, n), ccsim::NvrarConfig{3, 4096});
    cudaMemcpy(got.data(), d_out, n * sizeof(T), cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
  }
  if (std::memcmp(got.data(), want.data(), n * sizeof(T)) != 0) {
    std::printf("rank %d: %s n=%zu differs from oracles::nvrar_order_sum\n", rank,
                host ? "run_host" : "run", n);
    return 1;
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 6) {
    std::fprintf(stderr, "usage: %s dir rank nodes gpus device\n", argv[0]);
    return 2;
  }
  FileGather g{argv[1], std::atoi(argv[2]), std::atoi(argv[3]) * std::atoi(argv[4])};
  const int nodes = std::atoi(argv[3]), gpus = std::atoi(argv[4]), dev = std::atoi(argv[5]);
  cudaSetDevice(dev);
  const ccsim::ClusterTopology topo{nodes, gpus};
  int fails = 0;
  try {
    ccsim::NvrarB200Allreduce<float> f(topo, g.rank, dev, 1 << 18, file_allgather, &g, 60.0);
    ccsim::NvrarB200Allreduce<std::int32_t> i(topo, g.rank, dev, 1 << 18, file_allgather, &g, 60.0);
    for (std::size_t n : {std::size_t{1}, std::size_t{4099}, std::size_t{65539}}) {
      fails += check(f, g.rank, nodes, gpus, n, 1234 + n, false);
      fails += check(f, g.rank, nodes, gpus, n, 2234 + n, true);
      fails += check(i, g.rank, nodes, gpus, n, 3234 + n, false);
    }
    if (f.sequence() != 6 || i.sequence() != 3) {
      std::printf("rank %d: sequence %u / %u, expected 6 / 3\n", g.rank, f.sequence(),
                  i.sequence());
      ++fails;
    }
    // the reference's error for an over-long vector (nvrar.hpp:86-91)
    try {
      std::vector<float> big((1 << 18) + 1), out(big.size());
      f.run_host(std::span<const float>(big), std::span<float>(out));
      ++fails;
    } catch (const ccsim::InvalidArgumentError&) {
    }
    // every rank leaves together (the comms' regions are mapped by the peers)
    char one = 1;
    std::vector<char> all(g.world);
    file_allgather(&g, &one, all.data(), 1);
  } catch (const std::exception& e) {
    std::printf("rank %d: exception %s\n", g.rank, e.what());
    return 1;
  }
  std::printf("rank %d: %s\n", g.rank, fails ? "FAILURES" : "OK");
  return fails ? 1 : 0;
}
