/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the NVRAR all-reduce (see
 * nvrar_oracle.h for the rules on who may call it and what it restates).
 * Compile with -ffp-contract=off: every fp32 add here must round on its own,
 * exactly like the reference's elem_add (collectives/fused.hpp:45-53).
 */
#include "nvrar_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- std::mt19937_64 ---------------------------------------------------- */
#define MT_N 312
#define MT_M 156
#define MT_MATRIX_A 0xB5026F5AA96619E9ULL
#define MT_UPPER 0xFFFFFFFF80000000ULL
#define MT_LOWER 0x000000007FFFFFFFULL

void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) {
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  s->idx = MT_N;
}

static void mt64_twist(orc_mt64* s) {
  for (int i = 0; i < MT_N; ++i) {
    uint64_t y = (s->mt[i] & MT_UPPER) | (s->mt[(i + 1) % MT_N] & MT_LOWER);
    uint64_t v = s->mt[(i + MT_M) % MT_N] ^ (y >> 1);
    if (y & 1ULL) v ^= MT_MATRIX_A;
    s->mt[i] = v;
  }
  s->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* s) {
  if (s->idx >= MT_N) mt64_twist(s);
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

/* libstdc++ generate_canonical<float,24>(mt19937_64): one draw, float(u64)/2^64,
 * clamped below 1; then uniform_real_distribution: u*(b-a)+a in float. */
static float canonical_f32(orc_mt64* s) {
  volatile float sum = (float)orc_mt64_next(s);
  volatile float tmp = 18446744073709551616.0f; /* 2^64 */
  float r = sum / tmp;
  if (r >= 1.0f) r = nextafterf(1.0f, 0.0f);
  return r;
}

void orc_random_inputs_f32(int ranks, size_t n, uint64_t seed, float* out) {
  orc_mt64 s;
  for (int r = 0; r < ranks; ++r) {
    orc_mt64_seed(&s, seed * 7919ULL + (uint64_t)r);
    float* v = out + (size_t)r * n;
    for (size_t i = 0; i < n; ++i) {
      volatile float prod = canonical_f32(&s) * (2.0f - 0.25f);
      v[i] = prod + 0.25f;
    }
  }
}

void orc_random_inputs_i32(int ranks, size_t n, uint64_t seed, int32_t* out) {
  orc_mt64 s;
  for (int r = 0; r < ranks; ++r) {
    orc_mt64_seed(&s, seed * 7919ULL + (uint64_t)r);
    int32_t* v = out + (size_t)r * n;
    for (size_t i = 0; i < n; ++i) v[i] = (int32_t)(uint32_t)orc_mt64_next(&s);
  }
}

/* ---- elem_add (fused.hpp:45-53) ---------------------------------------- */
static inline float add_f32(float a, float b) {
  volatile float r = a + b;
  return r;
}
static inline int32_t add_i32(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}

static int is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

/* ---- nvrar_order_sum (oracles.hpp:101-133) -----------------------------
 * For element e (e < n) with shard = ceil(n/G) and c = e / shard:
 *   node partial  = ring_chunk_fold: x[(c+1)%G] + x[(c+2)%G] + ... + x[c]
 *                   (oracles.hpp:49-61; ring_schedule.hpp:12-15)
 *   across nodes  = for bit = 1,2,..: v[node] = v[node^bit] + v[node]
 *                   (oracles.hpp:122-130)
 * Padding elements (e >= n) are zero and trimmed, so they are skipped here.
 */
#define ORC_MAX_NODES 64

#define DEFINE_ORDER_SUM(NAME, T, ADD)                                              \
  int NAME(int nodes, int gpus, size_t n, const T* inputs, T* out) {                \
    if (nodes < 1 || gpus < 1) return -2;                                           \
    if (!is_pow2(nodes) || nodes > ORC_MAX_NODES) return -1;                        \
    if (n == 0) return 0;                                                           \
    const size_t shard = (n + (size_t)gpus - 1) / (size_t)gpus;                     \
    T v[ORC_MAX_NODES], nx[ORC_MAX_NODES];                                          \
    for (size_t e = 0; e < n; ++e) {                                                \
      const int c = (int)(e / shard);                                               \
      for (int node = 0; node < nodes; ++node) {                                    \
        const T* base = inputs + (size_t)node * (size_t)gpus * n;                   \
        T f;                                                                        \
        if (gpus == 1) {                                                            \
          f = base[e];                                                              \
        } else {                                                                    \
          f = base[(size_t)((c + 1) % gpus) * n + e];                               \
          for (int j = 2; j < gpus; ++j) f = ADD(f, base[(size_t)((c + j) % gpus) * n + e]); \
          f = ADD(f, base[(size_t)c * n + e]);                                      \
        }                                                                           \
        v[node] = f;                                                                \
      }                                                                             \
      for (int bit = 1; bit < nodes; bit <<= 1) {                                   \
        for (int node = 0; node < nodes; ++node) nx[node] = ADD(v[node ^ bit], v[node]); \
        memcpy(v, nx, sizeof(T) * (size_t)nodes);                                   \
      }                                                                             \
      out[e] = v[0];                                                                \
    }                                                                               \
    return 0;                                                                       \
  }

DEFINE_ORDER_SUM(orc_nvrar_order_sum_f32, float, add_f32)
DEFINE_ORDER_SUM(orc_nvrar_order_sum_i32, int32_t, add_i32)

/* ---- standalone phases ---------------------------------------------------
 * intra_rs_sum (tests/oracles.hpp:89-97): the node members' inputs zero-padded
 * to ce*G (ce = ceil(n/G)); chunk c of the result is ring_chunk_fold(c) =
 * x[(c+1)%G] + ... + x[c] (oracles.hpp:49-61). Output: ce*G elements.
 * rd_inter (NvrarAllreduce::rd_inter, nvrar.hpp:132-155): every rank (node, g)
 * holds a w-element shard; the result for local rank g is the XOR-step sum over
 * nodes, v[node] = v[node^bit] + v[node] (rd_block, nvrar.hpp:197-220), the same
 * bits on every node. inputs/out: P x w, rank-major. */
#define DEFINE_INTRA_RS(NAME, T, ADD)                                               \
  int NAME(int gpus, size_t n, const T* inputs, T* out) {                           \
    if (gpus < 1) return -2;                                                        \
    if (n == 0) return 0;                                                           \
    const size_t ce = (n + (size_t)gpus - 1) / (size_t)gpus;                        \
    for (size_t e = 0; e < ce * (size_t)gpus; ++e) {                                \
      const int c = (int)(e / ce);                                                  \
      if (e >= n) {                                                                 \
        out[e] = (T)0;                                                              \
        continue;                                                                   \
      }                                                                             \
      T f = inputs[(size_t)((c + 1) % gpus) * n + e];                               \
      for (int j = 2; j < gpus; ++j) f = ADD(f, inputs[(size_t)((c + j) % gpus) * n + e]); \
      if (gpus > 1) f = ADD(f, inputs[(size_t)c * n + e]);                          \
      out[e] = f;                                                                   \
    }                                                                               \
    return 0;                                                                       \
  }

#define DEFINE_RD_INTER(NAME, T, ADD)                                               \
  int NAME(int nodes, int gpus, size_t w, const T* shards, T* out) {                \
    if (nodes < 1 || gpus < 1) return -2;                                           \
    if (!is_pow2(nodes) || nodes > ORC_MAX_NODES) return -1;                        \
    T v[ORC_MAX_NODES], nx[ORC_MAX_NODES];                                          \
    for (int g = 0; g < gpus; ++g) {                                                \
      for (size_t i = 0; i < w; ++i) {                                              \
        for (int node = 0; node < nodes; ++node) {                                  \
          v[node] = shards[((size_t)node * (size_t)gpus + (size_t)g) * w + i];      \
        }                                                                           \
        for (int bit = 1; bit < nodes; bit <<= 1) {                                 \
          for (int node = 0; node < nodes; ++node) nx[node] = ADD(v[node ^ bit], v[node]); \
          memcpy(v, nx, sizeof(T) * (size_t)nodes);                                 \
        }                                                                           \
        for (int node = 0; node < nodes; ++node) {                                  \
          out[((size_t)node * (size_t)gpus + (size_t)g) * w + i] = v[node];         \
        }                                                                           \
      }                                                                             \
    }                                                                               \
    return 0;                                                                       \
  }

/* ring_order_sum (tests/oracles.hpp:67-86): ring positions p -> rank
 * (p mod N, p div N); ce = ceil(n/P); element e in chunk c = e / ce is the ring
 * fold by position: x[(c+1)%P] + ... + x[c] (ring_chunk_fold, :45-58).
 * tree_order_sum (:137-159): per node t = in[G-1]; t = in[lr] + t for
 * lr = G-2..0; then for bit = 1,2,..: t[node] += t[node+bit] (node % 2bit == 0). */
#define DEFINE_RING_ORDER(NAME, T, ADD)                                             \
  int NAME(int nodes, int gpus, size_t n, const T* inputs, T* out) {                \
    if (nodes < 1 || gpus < 1) return -2;                                           \
    const int p = nodes * gpus;                                                     \
    if (n == 0) return 0;                                                           \
    const size_t ce = (n + (size_t)p - 1) / (size_t)p;                              \
    for (size_t e = 0; e < n; ++e) {                                                \
      const int c = (int)(e / ce);                                                  \
      T f = (T)0;                                                                   \
      for (int j = 1; j <= p; ++j) {                                                \
        const int pos = (c + j) % p;                                                \
        const int rank = (pos % nodes) * gpus + pos / nodes;                        \
        const T x = inputs[(size_t)rank * n + e];                                   \
        f = j == 1 ? x : ADD(f, x);                                                 \
      }                                                                             \
      out[e] = f;                                                                   \
    }                                                                               \
    return 0;                                                                       \
  }

#define DEFINE_TREE_ORDER(NAME, T, ADD)                                             \
  int NAME(int nodes, int gpus, size_t n, const T* inputs, T* out) {                \
    if (nodes < 1 || gpus < 1) return -2;                                           \
    if (!is_pow2(nodes) || nodes > ORC_MAX_NODES) return -1;                        \
    T t[ORC_MAX_NODES];                                                             \
    for (size_t e = 0; e < n; ++e) {                                                \
      for (int node = 0; node < nodes; ++node) {                                    \
        const T* base = inputs + (size_t)node * (size_t)gpus * n;                   \
        T v = base[(size_t)(gpus - 1) * n + e];                                     \
        for (int lr = gpus - 2; lr >= 0; --lr) v = ADD(base[(size_t)lr * n + e], v);  \
        t[node] = v;                                                                \
      }                                                                             \
      for (int bit = 1; bit < nodes; bit <<= 1) {                                   \
        for (int node = 0; node < nodes; node += 2 * bit) t[node] = ADD(t[node], t[node + bit]); \
      }                                                                             \
      out[e] = t[0];                                                                \
    }                                                                               \
    return 0;                                                                       \
  }

DEFINE_RING_ORDER(orc_ring_order_sum_f32, float, add_f32)
DEFINE_RING_ORDER(orc_ring_order_sum_i32, int32_t, add_i32)
DEFINE_TREE_ORDER(orc_tree_order_sum_f32, float, add_f32)
DEFINE_TREE_ORDER(orc_tree_order_sum_i32, int32_t, add_i32)

DEFINE_INTRA_RS(orc_intra_rs_sum_f32, float, add_f32)
DEFINE_INTRA_RS(orc_intra_rs_sum_i32, int32_t, add_i32)
DEFINE_RD_INTER(orc_rd_inter_f32, float, add_f32)
DEFINE_RD_INTER(orc_rd_inter_i32, int32_t, add_i32)

/* ---- bf16 -------------------------------------------------------------- */
float orc_bf16_to_f32(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t orc_f32_to_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) {
    return (uint16_t)((u >> 16) | 0x0040u); /* quiet NaN, payload not in parity */
  }
  const uint32_t lsb = (u >> 16) & 1u;
  u += 0x7FFFu + lsb;
  return (uint16_t)(u >> 16);
}

int orc_nvrar_order_sum_bf16(int nodes, int gpus, size_t n, const uint16_t* inputs,
                             uint16_t* out) {
  const size_t p = (size_t)nodes * (size_t)gpus;
  if (nodes < 1 || gpus < 1) return -2;
  if (!is_pow2(nodes)) return -1;
  if (n == 0) return 0;
  float* up = (float*)malloc(sizeof(float) * p * n);
  float* res = (float*)malloc(sizeof(float) * n);
  if (!up || !res) {
    free(up);
    free(res);
    return -3;
  }
  for (size_t i = 0; i < p * n; ++i) up[i] = orc_bf16_to_f32(inputs[i]);
  int rc = orc_nvrar_order_sum_f32(nodes, gpus, n, up, res);
  if (rc == 0) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_f32_to_bf16(res[i]);
  }
  free(up);
  free(res);
  return rc;
}

/* ---- serial_sum (oracles.hpp:25-34) ------------------------------------ */
void orc_serial_sum_f32(int ranks, size_t n, const float* inputs, float* out) {
  memcpy(out, inputs, sizeof(float) * n);
  for (int r = 1; r < ranks; ++r) {
    const float* x = inputs + (size_t)r * n;
    for (size_t i = 0; i < n; ++i) out[i] = add_f32(out[i], x[i]);
  }
}

void orc_serial_sum_i32(int ranks, size_t n, const int32_t* inputs, int32_t* out) {
  memcpy(out, inputs, sizeof(int32_t) * n);
  for (int r = 1; r < ranks; ++r) {
    const int32_t* x = inputs + (size_t)r * n;
    for (size_t i = 0; i < n; ++i) out[i] = add_i32(out[i], x[i]);
  }
}

/* ---- fused words (transport.hpp:81-87; fused.hpp:56-87) ---------------- */
uint64_t orc_make_word(uint32_t data, uint32_t flag) {
  return (uint64_t)data | ((uint64_t)flag << 32);
}
uint32_t orc_word_data(uint64_t w) { return (uint32_t)w; }
uint32_t orc_word_flag(uint64_t w) { return (uint32_t)(w >> 32); }

void orc_pack_fused(const uint32_t* data, size_t n, uint32_t seq, uint64_t* out) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_make_word(data[i], seq);
}

int orc_unpack_fused(const uint64_t* words, size_t n, uint32_t seq, uint32_t* out,
                     size_t* bad) {
  for (size_t i = 0; i < n; ++i) {
    if (orc_word_flag(words[i]) != seq) {
      if (bad) *bad = i;
      return -1;
    }
    out[i] = orc_word_data(words[i]);
  }
  return 0;
}
