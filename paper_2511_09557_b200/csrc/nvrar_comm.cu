// Host runtime behind include/nvrar.h: communicator lifecycle, symmetric
// region + CUDA IPC peer mapping, schedule selection, launches and fault
// reporting. One communicator per rank (per process, or several virtual ranks
// per device for the all-ranks-in-one-launch mode).
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nvrar.h"
#include "nvrar_device.cuh"

namespace nvrar {
using KernelFn = void (*)(LaunchParams);
KernelFn select_kernel(int dtype, bool flat, int nodes, int gpus, bool emu, bool lamport,
                       bool fast = false);
KernelFn bump_kernel();
KernelFn select_direct(int dtype, int nodes, int gpus);
KernelFn select_phase(int dtype, int mode, int nodes, bool emu);
KernelFn select_pull(int dtype, int nodes, int gpus);
using PingFn = void (*)(LaunchParams, int, int, uint64_t, int, uint64_t*);
PingFn pingpong_fn();
using CanaryFn = void (*)(LaunchParams, int, int, int, uint32_t, uint32_t, uint32_t, uint32_t*);
CanaryFn canary_fn();
int flat_max_gpus(int nodes);
}  // namespace nvrar

using namespace nvrar;

namespace {

constexpr uint32_t kMagic = 0x4E565241u;  // "NVRA"
constexpr uint64_t kOneshotMaxBytes = 1ull << 20;

struct HandleBlob {
  uint32_t magic;
  uint32_t version;
  int32_t pid;
  int32_t device;
  int32_t rank, world, nodes, gpus;
  uint64_t max_bytes;
  uint64_t region_ptr;
  uint64_t region_bytes;
  uint64_t layout_bytes;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(HandleBlob) <= NVRAR_HANDLE_BYTES, "handle too large");

std::string g_global_error;

int log2_exact(int v) {
  int l = 0;
  while ((1 << l) < v) ++l;
  return l;
}
bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

size_t dtype_bytes(int dt) { return dt == NVRAR_BF16 ? 2 : 4; }


}  // namespace

struct nvrar_comm {
  int world = 0, rank = 0, nodes = 1, gpus = 1, device = 0, steps = 0;
  size_t max_bytes = 0;
  Layout lay{};
  uint8_t* region = nullptr;
  RankState* state = nullptr;
  RankDesc* d_desc = nullptr;
  RankDesc h_desc{};
  std::vector<uint8_t*> opened;  // IPC mappings to close
  // caller buffers registered with the comm (nvrar_register_buffer): this
  // rank's range and every peer's mapping of its own registration
  struct RegBuf {
    int id = 0;
    uint8_t* local = nullptr;
    size_t bytes = 0;
    bool owned = false;      // nvrar_alloc_symmetric memory, freed with the registration
    bool connected = false;
    uint8_t* peer[kMaxRanks] = {};
    std::vector<uint8_t*> opened;
  };
  std::vector<RegBuf> regs;
  int next_reg = 1;
  nvrar_allgather_fn allgather = nullptr;  // nvrar_init's bootstrap (nvrar_alloc_symmetric)
  void* allgather_ctx = nullptr;
  int blocks = 0;
  uint64_t chunk_bytes = 65536;
  int algo = NVRAR_ALGO_AUTO;
  double timeout_s = 10.0;
  bool connected = false;
  int sticky = 0;
  std::string last_error;
  int max_ctas = 148;  // co-resident CTAs of one kernel on this device
  int sms = 148;
  int direct_ctas[3] = {148, 148, 148};  // co-resident direct-schedule CTAs per dtype
  bool pdl = true;     // programmatic dependent launch for single-rank launches
  int proto = NVRAR_PROTO_AUTO;
  int flags = 0;  // LaunchParams.flags (schedule variants; NVRAR_FLAGS)
  bool fast_oneshot = true;  // one-shot calls run the specialised kernel (SHOT = 1)
  bool host_l2fetch = true;  // 256-byte L2 fetches for host inputs (NVRAR_HOST_L2FETCH=0: off)
  bool dev_l2fetch = false;  // the same hint on device inputs (NVRAR_DEV_L2FETCH=1; experiment)
  int threads = kThreads;  // threads per CTA (multiple of 32, <= kThreads)
  uint64_t pp_base[kMaxRanks] = {};  // per-peer ping-pong counter (same on both sides)
  uint32_t canary_base[kMaxRanks] = {};  // per-peer canary flag base (same on both sides)
  uint64_t* d_scratch = nullptr;
  std::vector<nvrar_plan_entry> table;  // measured selector (ascending max_bytes)
  bool mc_ready = false;  // NVLS multicast area attached (nvrar_mc_attach)
  // host-buffer pipeline (nvrar_allreduce_host): device staging [2 in | 2 out]
  // of `stage_chunk` bytes each, copy streams and the events that order them
  uint8_t* stage = nullptr;
  size_t stage_chunk = 0;
  size_t host_chunk = 0;  // nvrar_set_host_chunk (0 = automatic)
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_start = nullptr, ev_h2d[2] = {}, ev_ar[2] = {}, ev_d2h[2] = {};
};

namespace {

int fail(nvrar_comm* c, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (c) {
    c->last_error = buf;
  } else {
    g_global_error = buf;
  }
  return code;
}

#define CUDA_TRY(c, expr)                                                         \
  do {                                                                            \
    cudaError_t e_ = (expr);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      return fail((c), NVRAR_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                            \
    }                                                                             \
  } while (0)

Layout make_layout(int world, int nodes, int gpus, size_t max_bytes) {
  // Sized for the worst dtype (bf16: most elements per byte) and every schedule.
  // Worst wire cost is 8 bytes per element (LL words / LL fp32 partials), and
  // a unit holds at most 8 elements; slots round up to 32-unit groups.
  const uint64_t max_elems = std::max<uint64_t>(max_bytes / 2, 8);
  const uint64_t eg = (max_elems + gpus - 1) / gpus;
  const uint64_t ep = (max_elems + world - 1) / world + 8;
  const uint64_t e1 = std::min<uint64_t>(max_elems, kOneshotMaxBytes / 2) + 8;
  const int steps = log2_exact(nodes);
  Layout l{};
  uint64_t off = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t o = off;
    off += (bytes + 255) & ~255ull;
    return o;
  };
  // counters, the ping-pong word and the done words each get their own block
  // (the ping-pong word once sat past a 64-word block, on the first A slot)
  l.ctrl_off = take(sizeof(uint64_t) * kCtrlWords);
  // 8-byte words per slot: one per element (8 B/element worst) rounded up to
  // whole 32-unit groups of up to 8 elements.
  auto slot_words = [](uint64_t elems) { return ((elems + 255) & ~255ull) + 256; };
  l.a_src = slot_words(std::max({gpus > 1 ? eg : 0, ep, e1}));
  l.a_off = take(2ull * world * l.a_src * 8);
  l.b_src = slot_words(std::max(gpus > 1 ? eg : 0, ep));
  l.b_off = take(2ull * world * l.b_src * 8);
  l.c_step = slot_words(eg);
  l.c_off = take(2ull * std::max(steps, 1) * l.c_step * 8);
  l.bytes = off;
  return l;
}

int validate_args(const nvrar_init_args* a) {
  if (!a) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null init args");
  if (a->nodes < 1 || a->gpus_per_node < 1) {
    return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT,
                "topology: nodes and gpus_per_node must be >= 1");
  }
  if (!is_pow2(a->nodes)) {
    return fail(nullptr, NVRAR_ERR_INVALID_TOPOLOGY,
                "nvrar: node count must be a power of two, got %d", a->nodes);
  }
  if (a->nodes > 8 || a->gpus_per_node > 8) {
    return fail(nullptr, NVRAR_ERR_INVALID_TOPOLOGY,
                "nvrar_b200: supports nodes <= 8 and gpus_per_node <= 8 (got %dx%d)",
                a->nodes, a->gpus_per_node);
  }
  if (a->world_size != a->nodes * a->gpus_per_node) {
    return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "world_size %d != nodes*gpus %d",
                a->world_size, a->nodes * a->gpus_per_node);
  }
  if (a->rank < 0 || a->rank >= a->world_size) {
    return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "rank %d out of range", a->rank);
  }
  if (a->blocks < 0) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "blocks must be >= 0");
  if (a->chunk_bytes != 0 && (a->chunk_bytes < 8 || a->chunk_bytes % 8 != 0)) {
    return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT,
                "nvrar config: chunk_bytes must be a multiple of 8, >= 8");
  }
  return NVRAR_SUCCESS;
}

// Schedule + CTA count for one call (nvrar_plan / nvrar_plan_for). A pure
// function of its arguments, so every rank picks the same schedule. The
// default policy is the measured one from the B200 sweep (DESIGN.md,
// "selector"); user overrides (algo / blocks) win.
// Default policy, from the B200 sweeps (paper_2511_09557_b200/tune.py; DESIGN.md
// §selector): one-shot while the (P-1)·M inbound bytes stay small, the
// hierarchical schedule in the middle (fewer wire bytes than one-shot, fewer
// hops than two-shot at these P), two-shot for large messages; CTAs grow with
// the message. `table` (from nvrar_set_plan_table, measured on the running
// system) overrides it.
void default_plan(int world, int nodes, uint64_t bytes, bool emu, int* algo, int* blocks) {
  // one-shot moves (P-1)*M into every GPU: cheapest while that stays small
  const uint64_t one_max = world <= 4 ? (1u << 20) : (256u << 10);
  if (world == 1) {
    *algo = NVRAR_ALGO_ONESHOT;
  } else if (emu) {
    // virtual ranks share one HBM: no exchange at all (falls back to HIER
    // when not every rank takes part in the launch)
    *algo = NVRAR_ALGO_DIRECT;
  } else if (bytes <= one_max) {
    *algo = NVRAR_ALGO_ONESHOT;
  } else if (bytes <= (1u << 20) && nodes > 1 && world >= 8) {
    // the hierarchy where the P=4 sweep measured it ahead of both flat
    // schedules (1 MB: 8.9 vs one-shot 9.2 / two-shot 10.7 us); at 2 MB it was
    // level with two-shot and behind above (its bf16 RD partials travel as fp32
    // cells). Unmeasured at P=8 here: bench.py / selector.autotune replace this
    // row with the measured table on the running box.
    *algo = NVRAR_ALGO_HIER;
  } else {
    *algo = NVRAR_ALGO_TWOSHOT;
  }
  *blocks = bytes <= (256u << 10) ? 64 : 128;
}

void plan_shape(int world, int nodes, int gpus, int algo_pref, int blocks_pref, int max_ctas,
                uint64_t count, int dtype, int* algo, int* blocks,
                const std::vector<nvrar_plan_entry>* table = nullptr, bool emu = false) {
  const uint64_t bytes = count * dtype_bytes(dtype);
  const bool flat_ok = gpus <= flat_max_gpus(nodes) && world <= 16;
  int a = algo_pref, b = blocks_pref;
  int da = NVRAR_ALGO_TWOSHOT, db = 32;
  default_plan(world, nodes, bytes, emu, &da, &db);
  if (table) {
    for (const auto& e : *table) {
      if (bytes <= e.max_bytes) {
        da = e.algo;
        db = e.blocks;
        break;
      }
    }
  }
  if (a == NVRAR_ALGO_AUTO) a = da;
  if (b <= 0) b = da == a ? db : std::max(db, 16);
  if ((a == NVRAR_ALGO_ONESHOT || a == NVRAR_ALGO_MCAST) && bytes > kOneshotMaxBytes) {
    a = NVRAR_ALGO_TWOSHOT;
  }
  // after the size rewrite: a flat schedule on a topology its register tile
  // cannot hold runs the hierarchical kernel
  if ((a == NVRAR_ALGO_TWOSHOT || a == NVRAR_ALGO_ONESHOT || a == NVRAR_ALGO_MCAST) && !flat_ok) {
    a = NVRAR_ALGO_HIER;
  }
  if (a == NVRAR_ALGO_DIRECT && !emu) a = NVRAR_ALGO_HIER;
  b = std::max(1, std::min(b, max_ctas));
  *algo = a;
  *blocks = b;
}

void plan(const nvrar_comm* c, uint64_t count, int dtype, int* algo, int* blocks,
          bool emu = false) {
  plan_shape(c->world, c->nodes, c->gpus, c->algo, c->blocks, c->max_ctas, count, dtype, algo,
             blocks, c->table.empty() ? nullptr : &c->table, emu);
}

int check_sticky(nvrar_comm* c) {
  if (c->sticky) return c->sticky;
  return NVRAR_SUCCESS;
}

}  // namespace

extern "C" {

int nvrar_abi_version(void) { return NVRAR_ABI_VERSION; }

const char* nvrar_status_string(int s) {
  switch (s) {
    case NVRAR_SUCCESS: return "success";
    case NVRAR_ERR_INTERNAL: return "internal error";
    case NVRAR_ERR_INVALID_ARGUMENT: return "invalid argument";
    case NVRAR_ERR_INVALID_TOPOLOGY: return "invalid topology";
    case NVRAR_ERR_PROTOCOL_FAULT: return "protocol fault";
    case NVRAR_ERR_DEADLOCK: return "deadlock";
    case NVRAR_ERR_CUDA: return "cuda error";
    case NVRAR_ERR_NOT_CONNECTED: return "not connected";
    default: return "unknown";
  }
}

const char* nvrar_last_error(nvrar_comm_t comm) {
  return comm ? comm->last_error.c_str() : g_global_error.c_str();
}

int nvrar_comm_create(const nvrar_init_args* a, nvrar_comm_t* out) {
  if (!out) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm out");
  *out = nullptr;
  int rc = validate_args(a);
  if (rc) return rc;
  auto* c = new nvrar_comm();
  c->world = a->world_size;
  c->rank = a->rank;
  c->nodes = a->nodes;
  c->gpus = a->gpus_per_node;
  c->device = a->device;
  c->steps = log2_exact(a->nodes);
  c->max_bytes = std::max<size_t>(a->max_bytes, 16);
  c->blocks = a->blocks;
  c->chunk_bytes = a->chunk_bytes ? a->chunk_bytes : 65536;
  c->timeout_s = a->timeout_s > 0 ? a->timeout_s : 10.0;
  c->lay = make_layout(c->world, c->nodes, c->gpus, c->max_bytes);

  auto cleanup = [&](int code) {
    if (c->region) cudaFree(c->region);
    if (c->state) cudaFree(c->state);
    if (c->d_desc) cudaFree(c->d_desc);
    g_global_error = c->last_error;
    delete c;
    return code;
  };
  cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) {
    fail(c, NVRAR_ERR_CUDA, "cudaSetDevice(%d): %s", c->device, cudaGetErrorString(e));
    return cleanup(NVRAR_ERR_CUDA);
  }
  if ((e = cudaMalloc(&c->region, c->lay.bytes)) != cudaSuccess ||
      // all-ones = empty cell for both wire protocols (and a counter no seq matches)
      (e = cudaMemset(c->region, 0xFF, c->lay.bytes)) != cudaSuccess ||
      (e = cudaMalloc(&c->state, sizeof(RankState))) != cudaSuccess ||
      (e = cudaMemset(c->state, 0, sizeof(RankState))) != cudaSuccess ||
      (e = cudaMalloc(&c->d_desc, sizeof(RankDesc))) != cudaSuccess ||
      (e = cudaMalloc(&c->d_scratch, 64)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess) {
    fail(c, NVRAR_ERR_CUDA, "allocating %llu B symmetric region: %s",
         static_cast<unsigned long long>(c->lay.bytes), cudaGetErrorString(e));
    return cleanup(NVRAR_ERR_CUDA);
  }
  int sms = 148, occ = 1;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  for (int flat = 0; flat < 2; ++flat) {
    for (int dt = 0; dt < 3; ++dt) {
      for (int emu = 0; emu < 2; ++emu) {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &o, reinterpret_cast<const void*>(
                        select_kernel(dt, flat, c->nodes,
                                      flat ? std::min(c->gpus, flat_max_gpus(c->nodes)) : c->gpus,
                                      emu, true)),
                kThreads, 0) == cudaSuccess &&
            o > 0) {
          occ = flat + dt + emu == 0 ? o : std::min(occ, o);
        }
      }
    }
  }
  c->max_ctas = std::max(1, std::min(kSeqSlots, sms * std::max(occ, 1)));
  c->sms = sms;
  for (int dt = 0; dt < 3; ++dt) {
    int o = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &o, reinterpret_cast<const void*>(select_direct(dt, c->nodes, c->gpus)), kDirectThreads, 0) !=
        cudaSuccess) {
      o = 1;
    }
    c->direct_ctas[dt] = sms * std::max(o, 1);
  }
  if (const char* v = getenv("NVRAR_PDL")) c->pdl = atoi(v) != 0;
  if (const char* v = getenv("NVRAR_FAST_ONESHOT")) c->fast_oneshot = atoi(v) != 0;
  if (const char* v = getenv("NVRAR_HOST_L2FETCH")) c->host_l2fetch = atoi(v) != 0;
  if (const char* v = getenv("NVRAR_DEV_L2FETCH")) c->dev_l2fetch = atoi(v) != 0;
  if (const char* v = getenv("NVRAR_FLAGS")) {
    c->flags = atoi(v) & (kFlagEarlySeq | kFlagLazyLen | kFlagSeqBarrier | kFlagDirectStream);
  }
  if (const char* v = getenv("NVRAR_THREADS")) {
    const int t = atoi(v);
    if (t >= 32 && t <= kThreads && t % 32 == 0) c->threads = t;
  }
  if (const char* v = getenv("NVRAR_PROTO")) {
    c->proto = std::string(v) == "ll" ? NVRAR_PROTO_LL
               : std::string(v) == "lamport" ? NVRAR_PROTO_LAMPORT : NVRAR_PROTO_AUTO;
  }
  c->h_desc = RankDesc{};
  c->h_desc.state = c->state;
  c->h_desc.lay = c->lay;
  c->h_desc.rank = c->rank;
  c->h_desc.world = c->world;
  c->h_desc.nodes = c->nodes;
  c->h_desc.gpus = c->gpus;
  c->h_desc.steps = c->steps;
  c->h_desc.node = c->rank / c->gpus;
  c->h_desc.local = c->rank % c->gpus;
  c->h_desc.timeout_ns = static_cast<uint64_t>(c->timeout_s * 1e9);
  c->h_desc.poll_ns = 0;
  if (const char* v = getenv("NVRAR_POLL_NS")) c->h_desc.poll_ns = static_cast<uint32_t>(atoi(v));
  c->h_desc.base[c->rank] = c->region;
  *out = c;
  return NVRAR_SUCCESS;
}

int nvrar_comm_export(nvrar_comm_t c, nvrar_handle_t* h) {
  if (!c || !h) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  HandleBlob b{};
  b.magic = kMagic;
  b.version = NVRAR_ABI_VERSION;
  b.pid = static_cast<int32_t>(getpid());
  b.device = c->device;
  b.rank = c->rank;
  b.world = c->world;
  b.nodes = c->nodes;
  b.gpus = c->gpus;
  b.max_bytes = c->max_bytes;
  b.region_ptr = reinterpret_cast<uint64_t>(c->region);
  b.region_bytes = c->lay.bytes;
  b.layout_bytes = c->lay.bytes;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaIpcGetMemHandle(&b.ipc, c->region));
  std::memset(h->bytes, 0, sizeof(h->bytes));
  std::memcpy(h->bytes, &b, sizeof(b));
  return NVRAR_SUCCESS;
}

int nvrar_comm_connect(nvrar_comm_t c, const nvrar_handle_t* hs, int count) {
  if (!c || !hs) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  if (count != c->world) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "expected %d handles, got %d", c->world, count);
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int32_t mypid = static_cast<int32_t>(getpid());
  for (int r = 0; r < count; ++r) {
    HandleBlob b;
    std::memcpy(&b, hs[r].bytes, sizeof(b));
    if (b.magic != kMagic || b.version != NVRAR_ABI_VERSION) {
      return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "handle %d: bad magic/version", r);
    }
    if (b.rank != r || b.world != c->world || b.nodes != c->nodes || b.gpus != c->gpus ||
        b.max_bytes != c->max_bytes || b.layout_bytes != c->lay.bytes) {
      return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                  "handle %d: peer comm shape differs (rank %d world %d %dx%d max %llu)", r,
                  b.rank, b.world, b.nodes, b.gpus,
                  static_cast<unsigned long long>(b.max_bytes));
    }
    if (r == c->rank) continue;
    if (b.pid == mypid) {
      if (b.device != c->device) {
        int can = 0;
        CUDA_TRY(c, cudaDeviceCanAccessPeer(&can, c->device, b.device));
        if (!can) {
          return fail(c, NVRAR_ERR_CUDA, "device %d cannot access peer %d", c->device, b.device);
        }
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          return fail(c, NVRAR_ERR_CUDA, "enable peer access: %s", cudaGetErrorString(e));
        }
        cudaGetLastError();
      }
      c->h_desc.base[r] = reinterpret_cast<uint8_t*>(b.region_ptr);
    } else {
      void* p = nullptr;
      CUDA_TRY(c, cudaIpcOpenMemHandle(&p, b.ipc, cudaIpcMemLazyEnablePeerAccess));
      c->h_desc.base[r] = static_cast<uint8_t*>(p);
      c->opened.push_back(static_cast<uint8_t*>(p));
    }
  }
  CUDA_TRY(c, cudaMemcpy(c->d_desc, &c->h_desc, sizeof(RankDesc), cudaMemcpyHostToDevice));
  c->connected = true;
  return NVRAR_SUCCESS;
}

int nvrar_init(const nvrar_init_args* a, nvrar_comm_t* out) {
  int rc = validate_args(a);
  if (rc) return rc;
  if (!a->allgather) {
    return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "nvrar_init needs an allgather callback");
  }
  nvrar_comm_t c = nullptr;
  rc = nvrar_comm_create(a, &c);
  if (rc) return rc;
  nvrar_handle_t mine;
  rc = nvrar_comm_export(c, &mine);
  if (rc) {
    g_global_error = c->last_error;
    nvrar_finalize(c);
    return rc;
  }
  std::vector<nvrar_handle_t> all(a->world_size);
  if (a->allgather(a->allgather_ctx, &mine, all.data(), sizeof(nvrar_handle_t)) != 0) {
    nvrar_finalize(c);
    return fail(nullptr, NVRAR_ERR_INTERNAL, "bootstrap allgather failed");
  }
  rc = nvrar_comm_connect(c, all.data(), a->world_size);
  if (rc) {
    g_global_error = c->last_error;
    nvrar_finalize(c);
    return rc;
  }
  c->allgather = a->allgather;
  c->allgather_ctx = a->allgather_ctx;
  *out = c;
  return NVRAR_SUCCESS;
}

static void mc_teardown(nvrar_comm* c);

static void host_pipe_teardown(nvrar_comm* c) {
  if (c->stage) cudaFree(c->stage);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  cudaEvent_t* evs[] = {&c->ev_start, &c->ev_h2d[0], &c->ev_h2d[1], &c->ev_ar[0], &c->ev_ar[1],
                        &c->ev_d2h[0], &c->ev_d2h[1]};
  for (cudaEvent_t* e : evs) {
    if (*e) cudaEventDestroy(*e);
    *e = nullptr;
  }
  c->stage = nullptr;
  c->s_h2d = c->s_d2h = nullptr;
}

int nvrar_finalize(nvrar_comm_t c) {
  if (!c) return NVRAR_SUCCESS;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  mc_teardown(c);
  host_pipe_teardown(c);
  for (auto& r : c->regs) {
    for (auto* p : r.opened) cudaIpcCloseMemHandle(p);
    if (r.owned) cudaFree(r.local);
  }
  c->regs.clear();
  for (auto* p : c->opened) cudaIpcCloseMemHandle(p);
  if (c->region) cudaFree(c->region);
  if (c->state) cudaFree(c->state);
  if (c->d_desc) cudaFree(c->d_desc);
  if (c->d_scratch) cudaFree(c->d_scratch);
  delete c;
  return NVRAR_SUCCESS;
}

// ---- registered buffers (Ctx::alloc_region's symmetric regions for caller
// data, transport.hpp:146-148) ------------------------------------------------
namespace {

constexpr uint32_t kRegMagic = 0x4E565242u;  // "NVRB"

struct RegBlob {
  uint32_t magic;
  int32_t pid, device, rank, id;
  uint64_t base_ptr;  // the allocation's base (what cudaIpcOpenMemHandle maps)
  uint64_t offset;    // the registered range's offset in it
  uint64_t bytes;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(RegBlob) <= NVRAR_HANDLE_BYTES, "registration handle too large");

// cuMemGetAddressRange through the runtime's driver entry point (no libcuda link)
int alloc_base(nvrar_comm* c, const void* p, uint8_t** base, size_t* size) {
  using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
  static Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      f = nullptr;
    }
    return reinterpret_cast<Fn>(f);
  }();
  if (!fn) return fail(c, NVRAR_ERR_CUDA, "cuMemGetAddressRange is unavailable");
  unsigned long long b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<unsigned long long>(p)) != 0) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "buffer %p is not device memory of this process", p);
  }
  *base = reinterpret_cast<uint8_t*>(b);
  *size = sz;
  return NVRAR_SUCCESS;
}

nvrar_comm::RegBuf* find_reg(nvrar_comm* c, int id) {
  for (auto& r : c->regs) {
    if (r.id == id) return &r;
  }
  return nullptr;
}

}  // namespace

int nvrar_register_buffer(nvrar_comm_t c, void* dev_ptr, size_t bytes, nvrar_handle_t* handle,
                          int* buf) {
  if (!c || !dev_ptr || !handle || !buf || bytes == 0) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "register: null argument or empty range");
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  uint8_t* base = nullptr;
  size_t size = 0;
  if (int rc = alloc_base(c, dev_ptr, &base, &size)) return rc;
  const uint8_t* p = static_cast<const uint8_t*>(dev_ptr);
  if (p + bytes > base + size) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "register: range runs past its allocation");
  }
  RegBlob b{};
  b.magic = kRegMagic;
  b.pid = static_cast<int32_t>(getpid());
  b.device = c->device;
  b.rank = c->rank;
  b.base_ptr = reinterpret_cast<uint64_t>(base);
  b.offset = static_cast<uint64_t>(p - base);
  b.bytes = bytes;
  CUDA_TRY(c, cudaIpcGetMemHandle(&b.ipc, base));
  nvrar_comm::RegBuf r;
  r.id = c->next_reg++;
  r.local = const_cast<uint8_t*>(p);
  r.bytes = bytes;
  b.id = r.id;
  c->regs.push_back(std::move(r));
  std::memset(handle->bytes, 0, sizeof(handle->bytes));
  std::memcpy(handle->bytes, &b, sizeof(b));
  *buf = b.id;
  return NVRAR_SUCCESS;
}

int nvrar_connect_buffer(nvrar_comm_t c, int buf, const nvrar_handle_t* hs, int count) {
  if (!c || !hs) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  nvrar_comm::RegBuf* r = find_reg(c, buf);
  if (!r) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "no registered buffer %d", buf);
  if (r->connected || !r->opened.empty()) {
    // a second connect would map the peers again (and leak the first mappings)
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "buffer %d is already connected", buf);
  }
  if (count != c->world) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "expected %d handles, got %d", c->world, count);
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  const int32_t mypid = static_cast<int32_t>(getpid());
  for (int q = 0; q < count; ++q) {
    RegBlob b;
    std::memcpy(&b, hs[q].bytes, sizeof(b));
    if (b.magic != kRegMagic || b.rank != q) {
      return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "registration handle %d: bad magic or rank", q);
    }
    if (b.bytes != r->bytes) {
      // symmetric: every rank registers the same size in the same order
      return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                  "registration %d: rank %d registered %llu bytes, this rank %zu", buf, q,
                  static_cast<unsigned long long>(b.bytes), r->bytes);
    }
    if (q == c->rank) {
      r->peer[q] = r->local;
      continue;
    }
    if (b.pid == mypid) {
      r->peer[q] = reinterpret_cast<uint8_t*>(b.base_ptr) + b.offset;
    } else {
      void* m = nullptr;
      CUDA_TRY(c, cudaIpcOpenMemHandle(&m, b.ipc, cudaIpcMemLazyEnablePeerAccess));
      r->opened.push_back(static_cast<uint8_t*>(m));
      r->peer[q] = static_cast<uint8_t*>(m) + b.offset;
    }
  }
  r->connected = true;
  return NVRAR_SUCCESS;
}

int nvrar_deregister_buffer(nvrar_comm_t c, int buf) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  for (size_t i = 0; i < c->regs.size(); ++i) {
    if (c->regs[i].id != buf) continue;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaDeviceSynchronize());
    for (auto* p : c->regs[i].opened) cudaIpcCloseMemHandle(p);
    if (c->regs[i].owned) cudaFree(c->regs[i].local);
    c->regs.erase(c->regs.begin() + static_cast<long>(i));
    return NVRAR_SUCCESS;
  }
  return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "no registered buffer %d", buf);
}

int nvrar_buffer_peer_ptr(nvrar_comm_t c, int buf, int peer, void** ptr) {
  if (!c || !ptr || peer < 0 || peer >= c->world) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad argument");
  }
  nvrar_comm::RegBuf* r = find_reg(c, buf);
  if (!r || !r->connected) {
    return fail(c, NVRAR_ERR_NOT_CONNECTED, "buffer %d is not registered and connected", buf);
  }
  *ptr = r->peer[peer];
  return NVRAR_SUCCESS;
}

int nvrar_alloc_symmetric(nvrar_comm_t c, size_t bytes, void** p) {
  if (!c || !p) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  if (!c->allgather) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                "nvrar_alloc_symmetric needs the bootstrap of nvrar_init; a comm from "
                "nvrar_comm_create registers caller memory with nvrar_register_buffer + "
                "nvrar_connect_buffer");
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  const size_t sz = std::max<size_t>(bytes, 16);
  void* q = nullptr;
  CUDA_TRY(c, cudaMalloc(&q, sz));
  CUDA_TRY(c, cudaMemset(q, 0, sz));
  CUDA_TRY(c, cudaDeviceSynchronize());
  nvrar_handle_t mine;
  int id = 0;
  if (int rc = nvrar_register_buffer(c, q, sz, &mine, &id)) {
    cudaFree(q);
    return rc;
  }
  find_reg(c, id)->owned = true;
  std::vector<nvrar_handle_t> all(c->world);
  if (c->allgather(c->allgather_ctx, &mine, all.data(), sizeof(nvrar_handle_t)) != 0) {
    nvrar_deregister_buffer(c, id);
    return fail(c, NVRAR_ERR_INTERNAL, "bootstrap allgather failed");
  }
  if (int rc = nvrar_connect_buffer(c, id, all.data(), c->world)) {
    const std::string e = c->last_error;
    nvrar_deregister_buffer(c, id);
    return fail(c, rc, "%s", e.c_str());
  }
  *p = q;
  return NVRAR_SUCCESS;
}

int nvrar_set_config(nvrar_comm_t c, int blocks, uint64_t chunk_bytes) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  // NvrarConfig::validate (fused.hpp:110-115); blocks == 0 selects automatically.
  if (blocks < 0) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "nvrar config: blocks must be >= 1");
  if (chunk_bytes < 8 || chunk_bytes % 8 != 0) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                "nvrar config: chunk_bytes must be a multiple of 8, >= 8");
  }
  c->blocks = blocks;
  c->chunk_bytes = chunk_bytes;
  return NVRAR_SUCCESS;
}

int nvrar_set_algo(nvrar_comm_t c, nvrar_algo_t algo) {
  if (!c || algo < NVRAR_ALGO_AUTO || algo > NVRAR_ALGO_MCAST) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad algo");
  }
  if ((algo == NVRAR_ALGO_TWOSHOT || algo == NVRAR_ALGO_ONESHOT) &&
      (c->gpus > flat_max_gpus(c->nodes) || c->world > 16)) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "flat schedules support at most %d gpus per node at %d nodes",
                flat_max_gpus(c->nodes), c->nodes);
  }
  c->algo = algo;
  return NVRAR_SUCCESS;
}

int nvrar_set_protocol(nvrar_comm_t c, nvrar_proto_t proto) {
  if (!c || proto < NVRAR_PROTO_AUTO || proto > NVRAR_PROTO_LAMPORT) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad protocol");
  }
  c->proto = proto;
  return NVRAR_SUCCESS;
}

int nvrar_set_timeout(nvrar_comm_t c, double timeout_s) {
  if (!c || !(timeout_s > 0)) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad timeout");
  c->timeout_s = timeout_s;
  c->h_desc.timeout_ns = static_cast<uint64_t>(timeout_s * 1e9);
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpy(c->d_desc, &c->h_desc, sizeof(RankDesc), cudaMemcpyHostToDevice));
  return NVRAR_SUCCESS;
}

int nvrar_plan(nvrar_comm_t c, size_t count, nvrar_dtype_t dtype, int* algo, int* blocks) {
  if (!c || !algo || !blocks) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  plan(c, count, dtype, algo, blocks);
  return NVRAR_SUCCESS;
}

static void resolve(nvrar_comm* c0, int nl, size_t count, int dtype, bool emu, int* algo_out,
                    int* blocks_out, int upt = 1);

int nvrar_plan_local(nvrar_comm_t* comms, int ncomms, size_t count, nvrar_dtype_t dtype,
                     uint64_t active_mask, int* algo, int* blocks) {
  if (!comms || ncomms < 1 || ncomms > NVRAR_MAX_LOCAL || !comms[0] || !algo || !blocks ||
      dtype < NVRAR_INT32 || dtype > NVRAR_BF16) {
    return fail(comms ? comms[0] : nullptr, NVRAR_ERR_INVALID_ARGUMENT, "bad plan query");
  }
  int nl = 0;
  for (int i = 0; i < ncomms; ++i) nl += static_cast<int>((active_mask >> i) & 1ull);
  resolve(comms[0], std::max(nl, 1), count, dtype, true, algo, blocks);
  return NVRAR_SUCCESS;
}

int nvrar_set_plan_table(nvrar_comm_t c, const nvrar_plan_entry* entries, int n) {
  if (!c || n < 0 || (n > 0 && !entries)) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad table");
  std::vector<nvrar_plan_entry> t(entries, entries + n);
  for (int i = 0; i < n; ++i) {
    if (t[i].algo < NVRAR_ALGO_HIER || t[i].algo > NVRAR_ALGO_MCAST ||
        t[i].algo == NVRAR_ALGO_DIRECT || t[i].blocks < 1 ||
        (i > 0 && t[i].max_bytes <= t[i - 1].max_bytes)) {
      return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                  "plan table entry %d: need ascending max_bytes, a concrete algo, blocks >= 1", i);
    }
  }
  c->table = std::move(t);
  return NVRAR_SUCCESS;
}

int nvrar_plan_for(int world, int nodes, int gpus, size_t count, nvrar_dtype_t dtype,
                   int algo_pref, int blocks_pref, int max_ctas, int* algo, int* blocks) {
  if (!algo || !blocks || world != nodes * gpus || !is_pow2(nodes) || max_ctas < 1) {
    return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "bad plan query");
  }
  plan_shape(world, nodes, gpus, algo_pref, blocks_pref, max_ctas, count, dtype, algo, blocks);
  return NVRAR_SUCCESS;
}

size_t nvrar_symmetric_bytes(nvrar_comm_t c) { return c ? c->lay.bytes : 0; }

int nvrar_get_peers(nvrar_comm_t c, int* peers, int max_peers, int* steps) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  if (steps) *steps = c->steps;
  const int node = c->rank / c->gpus, local = c->rank % c->gpus;
  for (int l = 0; l < c->steps && l < max_peers; ++l) {
    peers[l] = ((node ^ (1 << l)) * c->gpus) + local;  // nvrar.hpp:72-75
  }
  return NVRAR_SUCCESS;
}

// The schedule and CTAs per rank a launch of nl ranks of c0's topology uses
// (emu: the ranks are virtual ranks of one local group, one launch).
static void resolve(nvrar_comm* c0, int nl, size_t count, int dtype, bool emu, int* algo_out,
                    int* blocks_out, int upt) {
  int algo = 0, blocks = 1;
  plan(c0, count, dtype, &algo, &blocks, emu && nl > 1);
  // the direct schedule needs every rank of the topology in this launch
  if (algo == NVRAR_ALGO_DIRECT && (!emu || nl != c0->world)) algo = NVRAR_ALGO_HIER;
  if (algo == NVRAR_ALGO_DIRECT) {
    // no CTA waits on another: units per rank spread over at least one CTA per
    // SM while every CTA keeps >= a warp of units, at most one unit per thread,
    // and no more CTAs than fit at once (threads loop, prefetching the next unit)
    const size_t upr = ((count * dtype_bytes(dtype) + 15) / 16 + nl - 1) / nl;
    // upt > 1 (host buffers over PCIe): fewer CTAs, each thread loops, so the
    // loads of unit i+1 overlap the stores of unit i across the link
    static const int dev_upt = [] {  // units per thread on device buffers (tuning knob)
      const char* e = getenv("NVRAR_DIRECT_UPT");
      const int v = e ? atoi(e) : 1;
      return v >= 1 && v <= 64 ? v : 1;
    }();
    const bool host = upt > 1;
    if (!host) upt = dev_upt;
    const size_t full = (upr + kDirectThreads * upt - 1) / (kDirectThreads * upt);
    // two CTAs per SM over the whole launch (measured at 2x4, 1 MB fp32:
    // 1 / 2 / 4 per SM -> 6.17 / 5.11 / 5.28 us; the round-1 rule, 256 CTAs,
    // left 40 SMs with one CTA and 108 with two: 5.23 us)
    const size_t spread = host || upt > 1 ? 1
                                          : std::min<size_t>((2 * c0->sms + nl - 1) / nl,
                                                             (upr + 31) / 32);
    const size_t resident = std::max(1, c0->direct_ctas[dtype] / nl);
    blocks = static_cast<int>(std::max<size_t>(
        1, std::min<size_t>({std::max(full, spread), resident, static_cast<size_t>(kSeqSlots)})));
    static const int dev_ctas = [] {  // CTAs per rank on device buffers (tuning knob)
      const char* e = getenv("NVRAR_DIRECT_CTAS");
      return e ? atoi(e) : 0;
    }();
    if (!host && dev_ctas > 0) blocks = std::min(dev_ctas, static_cast<int>(resident));
  } else if (emu) {
    blocks = std::max(1, std::min(blocks, c0->max_ctas / nl));
  }
  if (upt > 1 && algo != NVRAR_ALGO_DIRECT) {
    // host buffers over PCIe: at most 64 CTAs, so threads loop and the link
    // reads/writes of consecutive units overlap (measured at 1 MB: P=2
    // 63.8 -> 53.7 us, P=4 65.2 -> 57.0 us against 128 CTAs)
    static const int host_ctas = [] {  // the cap (env NVRAR_HOST_CTAS; tuning knob)
      const char* e = getenv("NVRAR_HOST_CTAS");
      const int v = e ? atoi(e) : 64;
      return v >= 1 && v <= kSeqSlots ? v : 64;
    }();
    blocks = std::min(blocks, host_ctas);
  }
  *algo_out = algo;
  *blocks_out = blocks;
}

// Bytes of the full-vector equivalent a call of `phase` moves (what max_bytes bounds).
static size_t phase_bytes(const nvrar_comm* c, int phase, size_t count, int dtype) {
  switch (phase) {
    case NVRAR_PHASE_ALL_GATHER: return count * c->gpus * dtype_bytes(dtype);  // G shards
    case NVRAR_PHASE_RD_INTER: return count * c->gpus * 4;  // one shard of 4-byte words
    default: return count * dtype_bytes(dtype);
  }
}

static int launch(nvrar_comm_t* comms, int ncomms, const void* const* send, void* const* recv,
                  size_t count, int dtype, int op, void* stream, uint64_t mask, bool local_group,
                  int phase = NVRAR_PHASE_ALL, int order = NVRAR_ORDER_NVRAR,
                  const void* const* resid = nullptr, uint64_t e_off = 0,
                  uint64_t n_order = 0, int upt = 1) {
  nvrar_comm* c0 = comms[0];
  if (op != NVRAR_SUM) return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "only SUM is supported");
  if (order < NVRAR_ORDER_NVRAR || order > NVRAR_ORDER_TREE) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "bad reduction order %d", order);
  }
  // ring / tree orders run on the flat kernel: its register tile bounds them
  if (order == NVRAR_ORDER_RING && c0->world > flat_max_gpus(1)) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "ring order: at most %d ranks",
                flat_max_gpus(1));
  }
  if (order == NVRAR_ORDER_TREE &&
      (c0->gpus > flat_max_gpus(c0->nodes) || c0->world > 16)) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "tree order: unsupported topology %dx%d",
                c0->nodes, c0->gpus);
  }
  if (dtype < NVRAR_INT32 || dtype > NVRAR_BF16) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  }
  if (phase < NVRAR_PHASE_ALL || phase > NVRAR_PHASE_ALL_GATHER) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "bad phase %d", phase);
  }
  if (phase == NVRAR_PHASE_RD_INTER && dtype == NVRAR_BF16) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "rd_inter: packed words carry int32 or fp32");
  }
  // the standalone intra phases reject empty vectors (nvrar.hpp:282-284,350-352)
  if (count == 0 && (phase == NVRAR_PHASE_REDUCE_SCATTER || phase == NVRAR_PHASE_ALL_GATHER)) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "intra phase: bad vector length 0");
  }
  // the order frame (shard index, window offsets) is 32-bit in the flat and
  // direct kernels: whole vectors stay below 2^31 elements
  if ((n_order ? n_order : count) >= (1ull << 31)) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "nvrar: vectors of 2^31 or more elements are not supported");
  }
  LaunchParams lp{};
  int nl = 0;
  for (int i = 0; i < ncomms; ++i) {
    nvrar_comm* c = comms[i];
    if (!c) return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "null comm %d", i);
    if (!c->connected) return fail(c, NVRAR_ERR_NOT_CONNECTED, "comm not connected");
    if (c->device != c0->device || c->nodes != c0->nodes || c->gpus != c0->gpus) {
      return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "comms differ in device or topology");
    }
    if (int s = check_sticky(c)) return fail(c, s, "comm is in a failed state: %s", c->last_error.c_str());
    if (phase_bytes(c, phase, count, dtype) > c->max_bytes) {
      return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                  "nvrar: vector longer than the preallocated maximum (%zu B > %zu B)",
                  phase_bytes(c, phase, count, dtype), c->max_bytes);
    }
    if (count > 0 && (!send[i] || !recv[i])) {
      return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null buffer");
    }
    if (!((mask >> i) & 1ull)) continue;
    lp.desc[nl] = c->d_desc;
    lp.send[nl] = send[i];
    lp.recv[nl] = recv[i];
    lp.resid[nl] = resid ? resid[i] : nullptr;
    ++nl;
  }
  if (nl == 0) return NVRAR_SUCCESS;
  lp.nlocal = nl;
  lp.count = count;
  lp.e_off = e_off;
  lp.n_order = n_order;
  lp.flags = c0->flags;
  if (upt > 1 && c0->host_l2fetch) lp.flags |= kFlagL2Fetch256;  // host buffers over PCIe
  if (upt <= 1 && c0->dev_l2fetch) lp.flags |= kFlagL2Fetch256;   // experiment: device inputs
  CUDA_TRY(c0, cudaSetDevice(c0->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (count == 0) {
    // n == 0 still consumes a sequence number (nvrar.hpp:93-96).
    bump_kernel()<<<dim3(1, nl), 32, 0, s>>>(lp);
    CUDA_TRY(c0, cudaGetLastError());
    return NVRAR_SUCCESS;
  }
  int algo = 0, blocks = 1;
  const bool emu = local_group;
  resolve(c0, nl, phase == NVRAR_PHASE_ALL ? count : phase_bytes(c0, phase, count, dtype) /
                                                         dtype_bytes(dtype),
          dtype, emu, &algo, &blocks, upt);
  if (phase != NVRAR_PHASE_ALL) {
    // the phase-only entry points run the hierarchical kernel's phase code
    algo = NVRAR_ALGO_HIER;
    if (emu) blocks = std::max(1, std::min(blocks, c0->max_ctas / nl));
  }
  const bool lamport = dtype != NVRAR_INT32 && c0->proto != NVRAR_PROTO_LL;
  // one-shot over NVLS multicast: a single real rank with the multicast area
  // bound; anything else runs the unicast one-shot (same bits either way)
  bool mc = false;
  if (algo == NVRAR_ALGO_MCAST) {
    mc = !emu && nl == 1 && c0->mc_ready && lamport && phase == NVRAR_PHASE_ALL &&
         count * dtype_bytes(dtype) <= kOneshotMaxBytes;
    algo = NVRAR_ALGO_ONESHOT;
  }
  lp.mc = mc ? 1 : 0;
  if (n_order && algo == NVRAR_ALGO_HIER) {
    // a window of a longer vector runs on the flat schedules (their order is
    // computed per element in the whole vector's frame)
    algo = count * dtype_bytes(dtype) <= kOneshotMaxBytes ? NVRAR_ALGO_ONESHOT : NVRAR_ALGO_TWOSHOT;
    if (emu) blocks = std::max(1, std::min(blocks, c0->max_ctas / nl));
  }
  if (order != NVRAR_ORDER_NVRAR && algo != NVRAR_ALGO_ONESHOT && algo != NVRAR_ALGO_TWOSHOT) {
    // the ring / tree orders exist on the flat schedules only
    algo = count * dtype_bytes(dtype) <= (c0->world <= 4 ? (1u << 20) : (256u << 10)) &&
                   count * dtype_bytes(dtype) <= kOneshotMaxBytes
               ? NVRAR_ALGO_ONESHOT
               : NVRAR_ALGO_TWOSHOT;
    if (emu) blocks = std::max(1, std::min(blocks, c0->max_ctas / nl));
  }
  lp.order = order;
  if (order == NVRAR_ORDER_RING) {
    // ring positions are local-rank-major: position p -> rank (p mod N, p div N)
    for (int p = 0; p < c0->world; ++p) {
      lp.perm[p] = static_cast<uint8_t>((p % c0->nodes) * c0->gpus + p / c0->nodes);
    }
  }
  const bool direct = algo == NVRAR_ALGO_DIRECT;
  lp.oneshot = algo == NVRAR_ALGO_ONESHOT;
  // by value: the kernel reads it from param space (EMU: only the topology fields
  // are shared by the virtual ranks; each reads the rest through desc[])
  lp.d0 = c0->h_desc;
  KernelFn k = phase != NVRAR_PHASE_ALL ? select_phase(dtype, phase, c0->nodes, emu)
               : direct ? select_direct(dtype, c0->nodes, c0->gpus)
                        : select_kernel(dtype, algo != NVRAR_ALGO_HIER,
                                        order == NVRAR_ORDER_RING ? 1 : c0->nodes,
                                        order == NVRAR_ORDER_RING ? c0->world : c0->gpus, emu,
                                        lamport,
                                        // the one-shot specialisation (NVRAR_FAST_ONESHOT=0: off)
                                        c0->fast_oneshot && algo == NVRAR_ALGO_ONESHOT &&
                                            order == NVRAR_ORDER_NVRAR && !mc);
  if (!k) return fail(c0, NVRAR_ERR_INTERNAL, "no kernel for nodes=%d", c0->nodes);

  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks, nl);
  cfg.blockDim = dim3(direct ? kDirectThreads : c0->threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (emu && !direct) {
    // virtual ranks wait on each other: all CTAs must be co-resident
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.numAttrs = 1;
  } else if (c0->pdl) {
    // overlap this launch with the tail of the previous kernel on the stream;
    // the kernel's griddepcontrol.wait keeps every data access after it
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 1;
  }
  CUDA_TRY(c0, cudaLaunchKernelEx(&cfg, k, lp));
  return NVRAR_SUCCESS;
}

int nvrar_allreduce(nvrar_comm_t comm, const void* send, void* recv, size_t count,
                    nvrar_dtype_t dtype, nvrar_op_t op, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  const void* s[1] = {send};
  void* r[1] = {recv};
  return launch(&comm, 1, s, r, count, dtype, op, stream, ~0ull, false);
}

int nvrar_allreduce_registered(nvrar_comm_t c, const void* send, void* recv, size_t count,
                               nvrar_dtype_t dtype, nvrar_op_t op, void* stream) {
  if (!c) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  if (count == 0) {
    const void* s[1] = {send};
    void* r[1] = {recv};
    return launch(&c, 1, s, r, 0, dtype, op, stream, ~0ull, false);
  }
  if (op != NVRAR_SUM) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "only SUM is supported");
  if (dtype < NVRAR_INT32 || dtype > NVRAR_BF16) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  }
  if (!c->connected) return fail(c, NVRAR_ERR_NOT_CONNECTED, "comm not connected");
  if (int s = check_sticky(c)) return fail(c, s, "comm is in a failed state: %s", c->last_error.c_str());
  if (!recv) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null buffer");
  if (count >= (1ull << 31)) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "nvrar: vectors of 2^31 or more elements are not supported");
  }
  if (c->world > kMaxLocal) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "registered all-reduce: at most %d ranks", kMaxLocal);
  }
  const size_t bytes = count * dtype_bytes(dtype);
  const uint8_t* sp = static_cast<const uint8_t*>(send);
  const nvrar_comm::RegBuf* reg = nullptr;
  for (const auto& r : c->regs) {
    if (r.connected && sp >= r.local && sp + bytes <= r.local + r.bytes) {
      reg = &r;
      break;
    }
  }
  if (!reg) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                "registered all-reduce: send (%zu B) is not inside a registered, connected buffer",
                bytes);
  }
  KernelFn k = select_pull(dtype, c->nodes, c->gpus);
  if (!k) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "registered all-reduce: topology %dx%d unsupported",
                c->nodes, c->gpus);
  }
  LaunchParams lp{};
  lp.d0 = c->h_desc;
  lp.nlocal = 1;
  lp.count = count;
  const size_t off = static_cast<size_t>(sp - reg->local);
  for (int q = 0; q < c->world; ++q) lp.send[q] = reg->peer[q] + off;
  lp.recv[0] = recv;
  const size_t units = (bytes + 15) / 16;
  int blocks = c->blocks > 0 ? c->blocks
                             : static_cast<int>(std::min<size_t>(c->max_ctas,
                                                                 (units + c->threads - 1) / c->threads));
  blocks = std::max(1, std::min({blocks, c->max_ctas, kSeqSlots}));
  CUDA_TRY(c, cudaSetDevice(c->device));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(blocks, 1);
  cfg.blockDim = dim3(c->threads);
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (c->pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.numAttrs = 1;
  }
  CUDA_TRY(c, cudaLaunchKernelEx(&cfg, k, lp));
  return NVRAR_SUCCESS;
}

int nvrar_allreduce_residual(nvrar_comm_t comm, const void* send, void* recv,
                             const void* residual, size_t count, nvrar_dtype_t dtype,
                             nvrar_op_t op, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  if (count > 0 && !residual) return fail(comm, NVRAR_ERR_INVALID_ARGUMENT, "null residual");
  const void* s[1] = {send};
  void* r[1] = {recv};
  const void* x[1] = {residual};
  return launch(&comm, 1, s, r, count, dtype, op, stream, ~0ull, false, NVRAR_PHASE_ALL,
                NVRAR_ORDER_NVRAR, x);
}

int nvrar_allreduce_local_residual(nvrar_comm_t* comms, int ncomms, const void* const* send,
                                   void* const* recv, const void* const* residual, size_t count,
                                   nvrar_dtype_t dtype, nvrar_op_t op, void* stream,
                                   uint64_t active_mask) {
  if (!comms || ncomms < 1 || ncomms > NVRAR_MAX_LOCAL || !send || !recv || !residual) {
    return fail(comms ? comms[0] : nullptr, NVRAR_ERR_INVALID_ARGUMENT, "bad local group");
  }
  return launch(comms, ncomms, send, recv, count, dtype, op, stream, active_mask, true,
                NVRAR_PHASE_ALL, NVRAR_ORDER_NVRAR, residual);
}

int nvrar_ring_allreduce(nvrar_comm_t comm, const void* send, void* recv, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  const void* s[1] = {send};
  void* r[1] = {recv};
  return launch(&comm, 1, s, r, count, dtype, op, stream, ~0ull, false, NVRAR_PHASE_ALL,
                NVRAR_ORDER_RING);
}

int nvrar_tree_allreduce(nvrar_comm_t comm, const void* send, void* recv, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  const void* s[1] = {send};
  void* r[1] = {recv};
  return launch(&comm, 1, s, r, count, dtype, op, stream, ~0ull, false, NVRAR_PHASE_ALL,
                NVRAR_ORDER_TREE);
}

int nvrar_allreduce_local_order(nvrar_comm_t* comms, int ncomms, int order,
                                const void* const* send, void* const* recv, size_t count,
                                nvrar_dtype_t dtype, nvrar_op_t op, void* stream,
                                uint64_t active_mask) {
  if (!comms || ncomms < 1 || ncomms > NVRAR_MAX_LOCAL || !send || !recv) {
    return fail(comms ? comms[0] : nullptr, NVRAR_ERR_INVALID_ARGUMENT, "bad local group");
  }
  return launch(comms, ncomms, send, recv, count, dtype, op, stream, active_mask, true,
                NVRAR_PHASE_ALL, order);
}

int nvrar_reduce_scatter(nvrar_comm_t comm, const void* send, void* recv_shard, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  const void* s[1] = {send};
  void* r[1] = {recv_shard};
  return launch(&comm, 1, s, r, count, dtype, op, stream, ~0ull, false,
                NVRAR_PHASE_REDUCE_SCATTER);
}

int nvrar_all_gather(nvrar_comm_t comm, const void* shard, void* recv, size_t shard_count,
                     nvrar_dtype_t dtype, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  const void* s[1] = {shard};
  void* r[1] = {recv};
  return launch(&comm, 1, s, r, shard_count, dtype, NVRAR_SUM, stream, ~0ull, false,
                NVRAR_PHASE_ALL_GATHER);
}

int nvrar_rd_inter(nvrar_comm_t comm, const uint64_t* packed, uint64_t* out, size_t words,
                   nvrar_dtype_t dtype, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  const void* s[1] = {packed};
  void* r[1] = {out};
  return launch(&comm, 1, s, r, words, dtype, NVRAR_SUM, stream, ~0ull, false,
                NVRAR_PHASE_RD_INTER);
}

int nvrar_phase_local(nvrar_comm_t* comms, int ncomms, int phase, const void* const* send,
                      void* const* recv, size_t count, nvrar_dtype_t dtype, void* stream,
                      uint64_t active_mask) {
  if (!comms || ncomms < 1 || ncomms > NVRAR_MAX_LOCAL || !send || !recv) {
    return fail(comms ? comms[0] : nullptr, NVRAR_ERR_INVALID_ARGUMENT, "bad local group");
  }
  return launch(comms, ncomms, send, recv, count, dtype, NVRAR_SUM, stream, active_mask, true,
                phase);
}

int nvrar_allreduce_local(nvrar_comm_t* comms, int ncomms, const void* const* send,
                          void* const* recv, size_t count, nvrar_dtype_t dtype, nvrar_op_t op,
                          void* stream, uint64_t active_mask) {
  if (!comms || ncomms < 1 || ncomms > NVRAR_MAX_LOCAL || !send || !recv) {
    return fail(comms ? comms[0] : nullptr, NVRAR_ERR_INVALID_ARGUMENT, "bad local group");
  }
  return launch(comms, ncomms, send, recv, count, dtype, op, stream, active_mask, true);
}

int nvrar_get_sequence(nvrar_comm_t c, uint32_t* seq) {
  if (!c || !seq) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  RankState st;
  CUDA_TRY(c, cudaMemcpy(&st, c->state, sizeof(st), cudaMemcpyDeviceToHost));
  *seq = st.seq[0];
  return NVRAR_SUCCESS;
}

int nvrar_set_profile(nvrar_comm_t c, int on) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  c->h_desc.profile = on ? 1 : 0;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpy(c->d_desc, &c->h_desc, sizeof(RankDesc), cudaMemcpyHostToDevice));
  return NVRAR_SUCCESS;
}

int nvrar_get_phase_times(nvrar_comm_t c, uint64_t* ts, int n) {
  if (!c || !ts || n < 1) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  RankState st;
  CUDA_TRY(c, cudaMemcpy(&st, c->state, sizeof(st), cudaMemcpyDeviceToHost));
  for (int i = 0; i < n && i < kSeqSlots * kPhases; ++i) ts[i] = (&st.ts[0][0])[i];
  return NVRAR_SUCCESS;
}

int nvrar_pingpong(nvrar_comm_t c, int peer, int iters, int initiator, void* stream,
                   uint64_t* elapsed_ns) {
  if (!c || !elapsed_ns || peer < 0 || peer >= c->world || peer == c->rank || iters < 1) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad pingpong argument");
  }
  if (!c->connected) return fail(c, NVRAR_ERR_NOT_CONNECTED, "comm not connected");
  CUDA_TRY(c, cudaSetDevice(c->device));
  LaunchParams lp{};
  lp.d0 = c->h_desc;
  lp.nlocal = 1;
  // values unique per (pair, call): a stale echo from another pair never matches
  const int lo = std::min(peer, c->rank), hi = std::max(peer, c->rank);
  const uint64_t base = (static_cast<uint64_t>(lo * kMaxRanks + hi + 1) << 40) + c->pp_base[peer];
  c->pp_base[peer] += static_cast<uint64_t>(iters) + 1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  pingpong_fn()<<<1, 32, 0, s>>>(lp, peer, iters, base, initiator, c->d_scratch);
  CUDA_TRY(c, cudaGetLastError());
  CUDA_TRY(c, cudaStreamSynchronize(s));
  CUDA_TRY(c, cudaMemcpy(elapsed_ns, c->d_scratch, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (*elapsed_ns == ~0ull) return fail(c, NVRAR_ERR_DEADLOCK, "pingpong timed out");
  return NVRAR_SUCCESS;
}

int nvrar_set_jitter(nvrar_comm_t c, uint32_t max_ns, uint32_t seed) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  if (max_ns > 1000000u) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "jitter above 1 ms");
  c->h_desc.jitter_ns = max_ns;
  c->h_desc.jitter_seed = seed;
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpy(c->d_desc, &c->h_desc, sizeof(RankDesc), cudaMemcpyHostToDevice));
  return NVRAR_SUCCESS;
}

int nvrar_debug_canary(nvrar_comm_t c, int peer, int iters, int writer, uint32_t jitter_ns,
                       uint32_t seed, void* stream) {
  if (!c || peer < 0 || peer >= c->world || peer == c->rank || iters < 1 ||
      iters > (1 << 20)) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad canary argument");
  }
  if (!c->connected) return fail(c, NVRAR_ERR_NOT_CONNECTED, "comm not connected");
  CUDA_TRY(c, cudaSetDevice(c->device));
  LaunchParams lp{};
  lp.d0 = c->h_desc;
  lp.nlocal = 1;
  // flags unique per (pair, run): a previous run's cell never matches this run's last flag
  const uint32_t base = c->canary_base[peer] + 1u;
  c->canary_base[peer] += static_cast<uint32_t>(iters) + 1u;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* out = reinterpret_cast<uint32_t*>(c->d_scratch) + 8;  // scratch words 4..
  canary_fn()<<<1, 32, 0, s>>>(lp, peer, iters, writer, base, jitter_ns, seed, out);
  CUDA_TRY(c, cudaGetLastError());
  return NVRAR_SUCCESS;
}

int nvrar_debug_canary_result(nvrar_comm_t c, uint32_t* torn) {
  if (!c || !torn) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  CUDA_TRY(c, cudaMemcpy(torn, reinterpret_cast<uint32_t*>(c->d_scratch) + 8, sizeof(uint32_t),
                         cudaMemcpyDeviceToHost));
  if (*torn == ~0u) return fail(c, NVRAR_ERR_DEADLOCK, "canary reader timed out");
  return NVRAR_SUCCESS;
}

int nvrar_debug_dirty_cells(nvrar_comm_t c, uint64_t* dirty, uint64_t* first_offset) {
  if (!c || !dirty) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  std::vector<uint64_t> h((c->lay.bytes - c->lay.a_off) / 8);
  CUDA_TRY(c, cudaMemcpy(h.data(), c->region + c->lay.a_off, h.size() * 8, cudaMemcpyDeviceToHost));
  uint64_t cnt = 0, first = ~0ull;
  for (size_t i = 0; i < h.size(); ++i) {
    if (h[i] != ~0ull) {
      if (first == ~0ull) first = c->lay.a_off + i * 8;
      ++cnt;
    }
  }
  *dirty = cnt;
  if (first_offset) *first_offset = first;
  return NVRAR_SUCCESS;
}

int nvrar_debug_read_region(nvrar_comm_t c, uint64_t offset, uint64_t bytes, void* host,
                            uint64_t* layout) {
  if (!c || (!host && bytes)) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  if (layout) {
    const uint64_t l[8] = {c->lay.ctrl_off, c->lay.a_off, c->lay.a_src, c->lay.b_off,
                           c->lay.b_src, c->lay.c_off, c->lay.c_step, c->lay.bytes};
    std::memcpy(layout, l, sizeof(l));
  }
  if (!bytes) return NVRAR_SUCCESS;
  if (offset + bytes > c->lay.bytes) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "out of range");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  CUDA_TRY(c, cudaMemcpy(host, c->region + offset, bytes, cudaMemcpyDeviceToHost));
  return NVRAR_SUCCESS;
}

int nvrar_debug_seq_slots(nvrar_comm_t c, uint32_t* out, int n) {
  if (!c || !out || n < 1) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "bad argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  CUDA_TRY(c, cudaMemcpy(out, c->state->seq, sizeof(uint32_t) * std::min(n, kSeqSlots),
                         cudaMemcpyDeviceToHost));
  return NVRAR_SUCCESS;
}

int nvrar_pingpong_clock(nvrar_comm_t c, uint64_t* stamps) {
  if (!c || !stamps) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaMemcpy(stamps, c->d_scratch + 1, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return NVRAR_SUCCESS;
}

int nvrar_get_blocked(nvrar_comm_t c, nvrar_blocked_t* out) {
  if (!c || !out) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  CUDA_TRY(c, cudaSetDevice(c->device));
  CUDA_TRY(c, cudaDeviceSynchronize());
  RankState st;
  CUDA_TRY(c, cudaMemcpy(&st, c->state, sizeof(st), cudaMemcpyDeviceToHost));
  out->global_rank = c->rank;
  out->kind = st.err.kind;
  out->peer_rank = st.err.peer;
  out->expected = st.err.expected;
  out->word_index = st.err.word;
  out->observed = st.err.observed;
  out->status = static_cast<int>(st.err.code);
  out->phase = st.err.phase;
  out->cta = st.err.cta;
  return NVRAR_SUCCESS;
}

int nvrar_check(nvrar_comm_t c) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  if (c->sticky) return c->sticky;
  nvrar_blocked_t b;
  int rc = nvrar_get_blocked(c, &b);
  if (rc) return rc;
  if (b.status == 0) return NVRAR_SUCCESS;
  c->sticky = b.status;
  static const char* kinds[] = {"flag", "seq", "length", "stale flag"};
  const char* kind = (b.kind >= 0 && b.kind < 4) ? kinds[b.kind] : "?";
  if (b.status == NVRAR_ERR_DEADLOCK) {
    fail(c, b.status, "deadlock: rank %d awaits %s %u from rank %d (word %llu, saw 0x%llx)",
         c->rank, kind, b.expected, b.peer_rank, static_cast<unsigned long long>(b.word_index),
         static_cast<unsigned long long>(b.observed));
  } else {
    fail(c, b.status, "rank %d: protocol fault (%s) with rank %d at call %u (saw 0x%llx)",
         c->rank, kind, b.peer_rank, b.expected, static_cast<unsigned long long>(b.observed));
  }
  return b.status;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// NVLS multicast area (NVRAR_ALGO_MCAST). The host framework supplies a
// multicast mapping and this rank's own mapping of the same memory (e.g.
// torch symmetric memory, NCCL's NVLS buffers); the library only uses them.
static void mc_teardown(nvrar_comm* c) {
  c->mc_ready = false;
  c->h_desc.mc = nullptr;
  c->h_desc.mc_local = nullptr;
}

int nvrar_mc_bytes(nvrar_comm_t c, size_t* bytes) {
  if (!c || !bytes) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  *bytes = 2ull * c->world * c->lay.a_src * 8;  // [2 parity][P src][a_src words]
  return NVRAR_SUCCESS;
}

int nvrar_mc_attach(nvrar_comm_t c, void* mc_base, void* local_base, size_t bytes) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  if (!c->connected) return fail(c, NVRAR_ERR_NOT_CONNECTED, "comm not connected");
  if (!mc_base && !local_base && bytes == 0) {  // detach (a peer failed to attach)
    mc_teardown(c);
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemcpy(c->d_desc, &c->h_desc, sizeof(RankDesc), cudaMemcpyHostToDevice));
    return NVRAR_SUCCESS;
  }
  size_t need = 0;
  nvrar_mc_bytes(c, &need);
  if (!mc_base || !local_base || bytes < need ||
      (reinterpret_cast<uintptr_t>(mc_base) | reinterpret_cast<uintptr_t>(local_base)) & 15u) {
    return fail(c, NVRAR_ERR_INVALID_ARGUMENT,
                "multicast area: need %zu bytes, 16-byte aligned mappings", need);
  }
  CUDA_TRY(c, cudaSetDevice(c->device));
  // every cell starts empty (the Lamport invariant), like the region
  CUDA_TRY(c, cudaMemset(local_base, 0xFF, need));
  CUDA_TRY(c, cudaDeviceSynchronize());
  c->h_desc.mc = static_cast<uint8_t*>(mc_base);
  c->h_desc.mc_local = static_cast<uint8_t*>(local_base);
  CUDA_TRY(c, cudaMemcpy(c->d_desc, &c->h_desc, sizeof(RankDesc), cudaMemcpyHostToDevice));
  c->mc_ready = true;
  return NVRAR_SUCCESS;
}

int nvrar_mc_ready(nvrar_comm_t c, int* ready) {
  if (!c || !ready) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null argument");
  *ready = c->mc_ready ? 1 : 0;
  return NVRAR_SUCCESS;
}

// ---------------------------------------------------------------------------
// Host buffers (the reference's own API shape: run() over host spans). The
// vector is moved in chunks through device staging: the H2D copy of chunk i+1,
// the all-reduce of chunk i and the D2H copy of chunk i-1 overlap on three
// streams. Every chunk is one all-reduce launch over a WINDOW of the whole
// vector (LaunchParams.e_off / n_order), so the bits equal one all-reduce of
// the whole vector — chunking must not change the reduction order.
namespace {

// Units per thread the direct schedule's grid is sized for when its buffers are
// host memory read and written over PCIe (env NVRAR_HOST_UPT; default 32 —
// measured N=1 e2e, 2x4 x 1 MB fp32: 1 unit 321 us, 4 units 261 us, 8 units
// 246-253 us, 16 248-257 us, 32 240-244 us: few long-running threads, each
// streaming through a contiguous range, drive the PCIe link best).
const int kHostUnitsPerThread = [] {
  const char* e = getenv("NVRAR_HOST_UPT");
  const int v = e ? atoi(e) : 32;
  return v >= 1 && v <= 64 ? v : 32;
}();

// Window of the host path (bytes per rank): nvrar_set_host_chunk or
// NVRAR_HOST_CHUNK if set, else the whole vector (one launch; only vectors
// longer than the comm's max_bytes are split). A function of (count, dtype,
// knobs) only, so every rank issues the same launches. (Measured at <= 4 MB:
// the copies' per-launch and cross-stream costs eat the overlap of a chunked
// pipeline — P=2 1 MB 65 us whole vs 87 us in 256 KB chunks.)
size_t host_chunk_bytes(const nvrar_comm* c, size_t rank_bytes) {
  static const long long env = [] {
    const char* e = getenv("NVRAR_HOST_CHUNK");
    return e ? atoll(e) : 0LL;
  }();
  if (c->host_chunk) return c->host_chunk;
  if (env >= 4096) return static_cast<size_t>(env);
  return std::max<size_t>(rank_bytes, 16);
}

int host_pipe_ready(nvrar_comm* c, size_t chunk) {
  if (c->stage && c->stage_chunk >= chunk) return NVRAR_SUCCESS;
  host_pipe_teardown(c);
  CUDA_TRY(c, cudaMalloc(&c->stage, 4 * chunk));
  c->stage_chunk = chunk;
  CUDA_TRY(c, cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
  CUDA_TRY(c, cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
  cudaEvent_t* evs[] = {&c->ev_start, &c->ev_h2d[0], &c->ev_h2d[1], &c->ev_ar[0], &c->ev_ar[1],
                        &c->ev_d2h[0], &c->ev_d2h[1]};
  for (cudaEvent_t* e : evs) CUDA_TRY(c, cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  return NVRAR_SUCCESS;
}

}  // namespace

static int host_allreduce(nvrar_comm_t* comms, int nc, const void* const* hsend,
                          void* const* hrecv, size_t count, int dtype, int op, void* stream,
                          bool local_group) {
  nvrar_comm* c0 = comms[0];
  if (dtype < NVRAR_INT32 || dtype > NVRAR_BF16) {
    return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "bad dtype %d", dtype);
  }
  for (int i = 0; i < nc; ++i) {
    if (!comms[i]) return fail(c0, NVRAR_ERR_INVALID_ARGUMENT, "null comm %d", i);
    if (count > 0 && (!hsend[i] || !hrecv[i])) {
      return fail(comms[i], NVRAR_ERR_INVALID_ARGUMENT, "null buffer");
    }
  }
  const size_t eb = dtype_bytes(dtype);
  CUDA_TRY(c0, cudaSetDevice(c0->device));
  // Zero-copy: pinned host memory is mapped into the device's address space
  // (UVA), so the kernels read the inputs and write the results over PCIe
  // themselves — no staging copies, the transfers overlap the exchange.
  bool mapped = count > 0;
  std::vector<const void*> zsend(nc);
  std::vector<void*> zrecv(nc);
  for (int r = 0; r < nc && mapped; ++r) {
    cudaPointerAttributes a{}, b{};
    if (cudaPointerGetAttributes(&a, hsend[r]) != cudaSuccess ||
        cudaPointerGetAttributes(&b, hrecv[r]) != cudaSuccess ||
        a.type != cudaMemoryTypeHost || b.type != cudaMemoryTypeHost || !a.devicePointer ||
        !b.devicePointer) {
      mapped = false;
      cudaGetLastError();
      break;
    }
    zsend[r] = a.devicePointer;
    zrecv[r] = b.devicePointer;
  }
  // The window schedule is a function of (count, dtype, max_bytes, host chunk)
  // only — never of the memory kind — so every rank issues the
  // same sequence of launches whether its buffers are pinned or pageable.
  // units of 16 bytes, so every window starts on a unit boundary
  const size_t chunk_elems =
      std::max<size_t>(16 / eb, (host_chunk_bytes(c0, count * eb) + 15) / 16 * 16 / eb);
  const bool windows = c0->world <= 16 && c0->gpus <= flat_max_gpus(c0->nodes);
  // a window never exceeds what the comm's staging was sized for
  const size_t ce = windows ? std::min(chunk_elems, std::max<size_t>(16 / eb,
                                                                    c0->max_bytes / eb / 16 * 16))
                            : std::max<size_t>(count, 1);
  const size_t nch = count == 0 ? 1 : (count + ce - 1) / ce;
  if (mapped && !c0->host_chunk) {
    // zero-copy (unless a chunk was asked for, which means staging): the same
    // windows, straight over the mapped host memory
    std::vector<const void*> ws(nc);
    std::vector<void*> wr(nc);
    for (size_t i = 0; i < nch; ++i) {
      const size_t off = i * ce, cnt = std::min(ce, count - off);
      for (int r = 0; r < nc; ++r) {
        ws[r] = static_cast<const uint8_t*>(zsend[r]) + off * eb;
        wr[r] = static_cast<uint8_t*>(zrecv[r]) + off * eb;
      }
      if (int rc = launch(comms, nc, ws.data(), wr.data(), cnt, dtype, op, stream, ~0ull,
                          local_group, NVRAR_PHASE_ALL, NVRAR_ORDER_NVRAR, nullptr,
                          nch > 1 ? off : 0, nch > 1 ? count : 0, kHostUnitsPerThread)) {
        return rc;
      }
    }
    return NVRAR_SUCCESS;
  }
  const size_t chunk = std::max<size_t>(ce * eb, 16);
  for (int i = 0; i < nc; ++i) {
    if (int rc = host_pipe_ready(comms[i], chunk)) return rc;
  }
  CUDA_TRY(c0, cudaSetDevice(c0->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (count == 0) {
    return launch(comms, nc, hsend, const_cast<void* const*>(hrecv), 0, dtype, op, stream,
                  ~0ull, local_group);
  }
  std::vector<const void*> dsend(nc);
  std::vector<void*> drecv(nc);
  if (nch == 1) {
    // one chunk: everything on the caller's stream (no cross-stream hops)
    for (int r = 0; r < nc; ++r) {
      dsend[r] = comms[r]->stage;
      drecv[r] = comms[r]->stage + 2 * chunk;
      CUDA_TRY(c0, cudaMemcpyAsync(comms[r]->stage, hsend[r], count * eb,
                                   cudaMemcpyHostToDevice, s));
    }
    if (int rc = launch(comms, nc, dsend.data(), drecv.data(), count, dtype, op, stream, ~0ull,
                        local_group)) {
      return rc;
    }
    for (int r = 0; r < nc; ++r) {
      CUDA_TRY(c0, cudaMemcpyAsync(hrecv[r], drecv[r], count * eb, cudaMemcpyDeviceToHost, s));
    }
    return NVRAR_SUCCESS;
  }
  // the copies start after the work already queued on the caller's stream
  CUDA_TRY(c0, cudaEventRecord(c0->ev_start, s));
  CUDA_TRY(c0, cudaStreamWaitEvent(c0->s_h2d, c0->ev_start, 0));
  for (size_t i = 0; i < nch; ++i) {
    const int b = static_cast<int>(i & 1);
    const size_t off = i * ce, cnt = std::min(ce, count - off);
    if (i >= 2) CUDA_TRY(c0, cudaStreamWaitEvent(c0->s_h2d, c0->ev_ar[b], 0));
    for (int r = 0; r < nc; ++r) {
      nvrar_comm* c = comms[r];
      uint8_t* din = c->stage + b * chunk;
      CUDA_TRY(c0, cudaMemcpyAsync(din, static_cast<const uint8_t*>(hsend[r]) + off * eb,
                                   cnt * eb, cudaMemcpyHostToDevice, c0->s_h2d));
      dsend[r] = din;
      drecv[r] = c->stage + (2 + b) * chunk;
    }
    CUDA_TRY(c0, cudaEventRecord(c0->ev_h2d[b], c0->s_h2d));
    CUDA_TRY(c0, cudaStreamWaitEvent(s, c0->ev_h2d[b], 0));
    if (i >= 2) CUDA_TRY(c0, cudaStreamWaitEvent(s, c0->ev_d2h[b], 0));
    int rc = launch(comms, nc, dsend.data(), drecv.data(), cnt, dtype, op, stream, ~0ull,
                    local_group, NVRAR_PHASE_ALL, NVRAR_ORDER_NVRAR, nullptr,
                    windows ? off : 0, windows ? count : 0);
    if (rc) return rc;
    CUDA_TRY(c0, cudaEventRecord(c0->ev_ar[b], s));
    CUDA_TRY(c0, cudaStreamWaitEvent(c0->s_d2h, c0->ev_ar[b], 0));
    for (int r = 0; r < nc; ++r) {
      CUDA_TRY(c0, cudaMemcpyAsync(static_cast<uint8_t*>(hrecv[r]) + off * eb, drecv[r],
                                   cnt * eb, cudaMemcpyDeviceToHost, c0->s_d2h));
    }
    CUDA_TRY(c0, cudaEventRecord(c0->ev_d2h[b], c0->s_d2h));
  }
  // the caller's stream completes when the last copies out have landed
  CUDA_TRY(c0, cudaStreamWaitEvent(s, c0->ev_d2h[(nch - 1) & 1], 0));
  if (nch > 1) CUDA_TRY(c0, cudaStreamWaitEvent(s, c0->ev_d2h[nch & 1], 0));
  return NVRAR_SUCCESS;
}

int nvrar_allreduce_host(nvrar_comm_t comm, const void* host_send, void* host_recv, size_t count,
                         nvrar_dtype_t dtype, nvrar_op_t op, void* stream) {
  if (!comm) return fail(nullptr, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  const void* s[1] = {host_send};
  void* r[1] = {host_recv};
  return host_allreduce(&comm, 1, s, r, count, dtype, op, stream, false);
}

int nvrar_allreduce_local_host(nvrar_comm_t* comms, int ncomms, const void* const* host_send,
                               void* const* host_recv, size_t count, nvrar_dtype_t dtype,
                               nvrar_op_t op, void* stream) {
  if (!comms || ncomms < 1 || ncomms > NVRAR_MAX_LOCAL || !host_send || !host_recv) {
    return fail(comms ? comms[0] : nullptr, NVRAR_ERR_INVALID_ARGUMENT, "bad local group");
  }
  return host_allreduce(comms, ncomms, host_send, host_recv, count, dtype, op, stream, true);
}

int nvrar_set_host_chunk(nvrar_comm_t c, size_t bytes) {
  if (!c) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "null comm");
  if (bytes != 0 && bytes < 16) return fail(c, NVRAR_ERR_INVALID_ARGUMENT, "chunk < 16 bytes");
  c->host_chunk = bytes;
  return NVRAR_SUCCESS;
}
