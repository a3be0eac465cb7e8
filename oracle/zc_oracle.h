/*
 * TEST INFRASTRUCTURE ONLY — a plain-C restatement of the reference algorithm
 * on the hot path, used by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the CHECKER.  The product library never links or calls it.
 *
 * Parity pinned: tests/test_oracle.py checks every function here against the
 * reference compiled from its own sources (oracle/_ref, see oracle/Makefile)
 * and against the golden fixtures in tests/golden/ (generated from oracle/_ref
 * by tests/golden/make_golden.py) plus the reference tests' hand vectors.
 */
#ifndef ZC_ORACLE_H
#define ZC_ORACLE_H
#include <stdint.h>

#include "zcomm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct zo_huff { /* HuffmanContext, huffman.hpp:20-33 */
  int32_t valid;
  uint8_t len[256];
  uint32_t code[256];
  uint32_t rev[256];
  uint8_t sym_order[256];
  uint32_t count_at_len[33];
  uint64_t first_code[33];
  uint32_t first_index[33];
  uint16_t lut[4096];
  uint32_t min_len, max_len;
} zo_huff;

/* frame.cpp */
void zo_write_header(const zc_frame_header* h, uint8_t* dst);
int zo_parse_header(const uint8_t* src, uint64_t len, zc_frame_header* out);
int zo_validate_header(const zc_frame_header* h, uint64_t region);
uint64_t zo_frame_commit_raw(const uint8_t* raw, uint64_t n, uint8_t* region, uint64_t cap);

/* quant.cpp — return 0 ok, ZC_DERR_NONFINITE / ZC_DERR_RANGE bits, or -1 bad scale */
int zo_eb_quantize_f64(const double* x, uint64_t n, double scale, int32_t* out);
int zo_eb_quantize_f32(const float* x, uint64_t n, double scale, int32_t* out);
int zo_absmax_f32(const float* x, uint64_t n, double* out);
typedef struct zo_mt64 {
  uint64_t x[312];
  int i;
} zo_mt64;
void zo_mt64_seed(zo_mt64* g, uint64_t seed);
uint64_t zo_mt64_next(zo_mt64* g);
int zo_qsgd_quantize_chunk_f32(const float* x, uint64_t n, uint32_t levels, double norm, uint64_t seed, uint64_t skip,
                               int32_t* out);
int zo_qsgd_quantize_f32(const float* x, uint64_t n, uint32_t levels, uint64_t seed, int32_t* out, double* scale);
void zo_dequantize_f64(const int32_t* s, uint64_t n, int mode, double scale, uint32_t levels, double* out);
void zo_dequantize_f32(const int32_t* s, uint64_t n, int mode, double scale, uint32_t levels, float* out);

/* fixedlen.cpp */
uint32_t zo_zigzag(int32_t v);
uint32_t zo_fixedlen_width(const int32_t* s, uint64_t n);
uint64_t zo_fixedlen_encode(const int32_t* s, uint64_t n, uint8_t* out, uint64_t cap, uint32_t* w);
int zo_fixedlen_decode(const zc_frame_header* h, const uint8_t* payload, uint64_t plen, uint8_t* dst,
                       uint64_t dlen);

/* huffman.cpp */
void zo_huff_lengths(const uint64_t* hist, uint8_t* lens);
int zo_huff_build(const uint64_t* hist, zo_huff* out);
int zo_huff_from_lengths(const uint8_t* lens, zo_huff* out);
int zo_huff_from_bytes(const uint8_t* sample, uint64_t n, zo_huff* out); /* +1 smoothing */
int zo_huff_expected_len(const zo_huff* c, const uint64_t* hist, double* bits);
int zo_huff_self_len(const uint64_t* hist, double* bits);
uint64_t zo_huffman_encode(const uint8_t* raw, uint64_t n, const zo_huff* c, uint8_t* out, uint64_t cap,
                           int embed);
int zo_huffman_decode(const zc_frame_header* h, const uint8_t* payload, uint64_t plen, const zo_huff* shared,
                      uint8_t* dst, uint64_t dlen);

/* rea.cpp */
void zo_default_arb_config(zc_arb_config* c);
void zo_profile_sample(const uint8_t* raw, uint64_t n, const zo_huff* ctx, zc_sample_stats* st);
uint64_t zo_predict_payload(int codec, uint64_t raw, const zc_sample_stats* st, const zc_arb_config* cfg);
void zo_arbitrate_plan(uint64_t raw, uint64_t cap, const zc_sample_stats* st, const zc_transport_hint* hint,
                       const zo_huff* ctx, const zc_arb_config* cfg, zc_arbitration_plan* plan);
void zo_encode_best(const uint8_t* raw, uint64_t n, uint8_t* stage, uint64_t cap, const zc_transport_hint* hint,
                    const zo_huff* ctx, const zc_arb_config* cfg, zc_encode_result* r);

/* collectives.cpp: send_batch codec dispatch (pin) and recv_batch decode dispatch.
 * zo_recv_batch returns the codec decoded, or -1 when the raw-copy fallback ran. */
void zo_send_batch(const uint8_t* raw, uint64_t n, uint8_t* stage, uint64_t cap, int pin,
                   const zc_transport_hint* hint, const zo_huff* ctx, const zc_arb_config* cfg,
                   zc_encode_result* r);
int zo_recv_batch(const uint8_t* frame, uint64_t frame_len, const zo_huff* ctx, uint8_t* dst, uint64_t dlen);

/* Serial simulation of the ring algorithms (collectives.cpp:423-503, 525-544) over all ranks.
 * syms: nranks*count, in/out.  Returns 0, or ZC_ERR_OVERFLOW / ZC_ERR_RUNTIME.  wire accumulates
 * exactly what WireStats counts (meta frames included).  scales: per-rank in/out (reconciled). */
/* CollectiveConfig::perSlotFraming (collectives.hpp:33): the ring functions below batch at 512 KiB
 * (RankCtx::chunk_raw_bytes, collectives.cpp:197-199) while on.  Process-wide; tests only. */
void zo_set_per_slot_framing(int on);
int zo_ring_allreduce(int nranks, int32_t* syms, uint64_t count, double* scales, int pin,
                      const zc_transport_hint* hint, const zo_huff* ctx, const zc_arb_config* cfg,
                      uint64_t fused_min_msg_bytes, zc_wire_stats* wire);
int zo_ring_allgather(int nranks, const int32_t* blocks, uint64_t block, int pin, const zc_transport_hint* hint,
                      const zo_huff* ctx, const zc_arb_config* cfg, int32_t* out, zc_wire_stats* wire);

/* bench.cpp generators (mt19937_64 + Box-Muller etc.), values rounded to f32 */
int zo_gen_data(int dist, double geom_p, uint64_t seed, int rank, uint64_t offset, uint64_t count, double* out);

#ifdef __cplusplus
}
#endif
#endif
