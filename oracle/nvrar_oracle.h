/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the NVRAR all-reduce.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker (or as the timed CPU
 * baseline). The product path (paper_2511_09557_b200) never links or calls it.
 *
 * It restates, in plain C, the arithmetic the reference pins for the path:
 *   - tests/oracles.hpp:161-178  random_inputs (mt19937_64, U[0.25,2) / raw int32)
 *   - tests/oracles.hpp:49-61    ring_chunk_fold (intra-node order)
 *   - tests/oracles.hpp:101-133  nvrar_order_sum (ring fold, then XOR-step adds)
 *   - tests/oracles.hpp:25-34    serial_sum
 *   - collectives/fused.hpp:43-53 elem_add (IEEE fp32 add, wrapping int32 add)
 *   - transport.hpp:81-87        fused word layout (data low 32, flag high 32)
 * plus the bf16 rule this build defines: the fp32 reference run
 * on bf16->fp32 up-cast inputs, rounded once (RNE) to bf16 at the end.
 *
 * Parity of this restatement is pinned against the reference itself: the
 * reference headers are compiled (oracle/ref_shim.cpp -> oracle/_ref) and
 * tests/golden/ holds vectors generated from that build (make_golden.py).
 */
#ifndef NVRAR_ORACLE_H
#define NVRAR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes shared with include/nvrar.h */
enum { ORC_INT32 = 0, ORC_FLOAT32 = 1, ORC_BF16 = 2 };

/* mt19937_64 exactly as std::mt19937_64 (state 312 words). */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_mt64;

void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);

/* oracles::random_inputs<float>: rank r uses mt19937_64(seed*7919 + r),
 * uniform_real_distribution<float>(0.25f, 2.0f). out is [ranks][n]. */
void orc_random_inputs_f32(int ranks, size_t n, uint64_t seed, float* out);
/* oracles::random_inputs<int32_t>: static_cast<int32_t>(rng()). */
void orc_random_inputs_i32(int ranks, size_t n, uint64_t seed, int32_t* out);

/* Hierarchical order sum for one hierarchy (nodes x gpus_per_node), inputs
 * indexed by global rank (node-major). inputs: [nodes*gpus][n].
 * out: n elements (every rank gets identical bits). Returns 0, or -1 when
 * nodes is not a power of two (InvalidTopologyError in the reference). */
int orc_nvrar_order_sum_f32(int nodes, int gpus, size_t n, const float* inputs, float* out);
int orc_nvrar_order_sum_i32(int nodes, int gpus, size_t n, const int32_t* inputs,
                            int32_t* out);
/* bf16 (raw uint16 bits): fp32 order sum of the up-cast inputs, one RNE round. */
int orc_nvrar_order_sum_bf16(int nodes, int gpus, size_t n, const uint16_t* inputs,
                             uint16_t* out);

/* oracles::serial_sum: global-rank order. */
/* The reference's baseline collectives' orders: ring_order_sum
 * (tests/oracles.hpp:67-86) and tree_order_sum (:137-159). */
int orc_ring_order_sum_f32(int nodes, int gpus, size_t n, const float* inputs, float* out);
int orc_ring_order_sum_i32(int nodes, int gpus, size_t n, const int32_t* inputs, int32_t* out);
int orc_tree_order_sum_f32(int nodes, int gpus, size_t n, const float* inputs, float* out);
int orc_tree_order_sum_i32(int nodes, int gpus, size_t n, const int32_t* inputs, int32_t* out);

/* Standalone phases: intra_rs_sum (tests/oracles.hpp:89-97; out = ce*G
 * elements) and the rd_inter result (nvrar.hpp:132-155; P x w rank-major). */
int orc_intra_rs_sum_f32(int gpus, size_t n, const float* inputs, float* out);
int orc_intra_rs_sum_i32(int gpus, size_t n, const int32_t* inputs, int32_t* out);
int orc_rd_inter_f32(int nodes, int gpus, size_t w, const float* shards, float* out);
int orc_rd_inter_i32(int nodes, int gpus, size_t w, const int32_t* shards, int32_t* out);

void orc_serial_sum_f32(int ranks, size_t n, const float* inputs, float* out);
void orc_serial_sum_i32(int ranks, size_t n, const int32_t* inputs, int32_t* out);

/* Fused 8-byte word helpers (transport.hpp:81-87, fused.hpp:56-101). */
uint64_t orc_make_word(uint32_t data, uint32_t flag);
uint32_t orc_word_data(uint64_t w);
uint32_t orc_word_flag(uint64_t w);
/* Returns 0, or -1 (ProtocolFaultError) when a flag differs from seq; *bad gets
 * the first offending word index. */
int orc_unpack_fused(const uint64_t* words, size_t n, uint32_t seq, uint32_t* out,
                     size_t* bad);
void orc_pack_fused(const uint32_t* data, size_t n, uint32_t seq, uint64_t* out);

/* bf16 helpers: RNE fp32 -> bf16 (NaN kept quiet), and up-cast. */
uint16_t orc_f32_to_bf16(float f);
float orc_bf16_to_f32(uint16_t b);

#ifdef __cplusplus
}
#endif

#endif
