/*
 * zcomm_b200.h — C-ABI of the B200-native compressed-collectives path.
 *
 * This is the drop-in boundary for the NCCLZ "zcomm" reference
 * (/root/reference/proj/core/include/zcomm/ headers).  Every entry point below
 * names the reference interface it replaces (file:line, paths relative to
 * /root/reference/proj/core/).  Conventions:
 *
 *   - plain pointers and sizes only; no C++ or torch types cross the ABI;
 *   - pointers documented "d_" are device (HBM) pointers, "h_" host pointers;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - every function returns an int status (ZC_OK or a ZC_ERR_* code) and a
 *     message retrievable with zc_last_error(); the C++ wrapper
 *     (paper_2605_12396_b200/csrc/zcomm_b200.hpp) rethrows these as the
 *     reference's exception types (std::invalid_argument, std::overflow_error,
 *     std::runtime_error, std::logic_error);
 *   - data-dependent failures discovered on the device (non-finite input,
 *     int32 bin overflow, symbol-sum overflow, peer timeout) are reported in a
 *     device error word (uint32 bit set, ZC_DERR_*) so that no kernel needs a
 *     host round-trip; the host checks it when the operation completes.
 *
 * There is no CPU fallback: every compute entry point launches sm_100a
 * kernels and fails with ZC_ERR_CUDA when no device is present.
 */
#ifndef ZCOMM_B200_H
#define ZCOMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- constants (frame.hpp:13-16, transport.hpp:17-23, rea.hpp:16, huffman.hpp:13-15) ---- */
#define ZC_HEADER_BYTES 32u
#define ZC_FRAME_MAGIC 0x464D435Au
#define ZC_FRAME_VERSION 1u
#define ZC_FLAG_EMBEDDED_CODEBOOK 0x0001u
#define ZC_SLOT_BYTES (512ull * 1024ull)
#define ZC_SLOTS_PER_CHANNEL 8u
#define ZC_BATCH_RAW_BYTES (ZC_SLOT_BYTES * ZC_SLOTS_PER_CHANNEL)
#define ZC_STAGE_BANK_BYTES (ZC_HEADER_BYTES + ZC_BATCH_RAW_BYTES)
#define ZC_STAGE_BANKS 8u
#define ZC_SAMPLE_WINDOW_BYTES 65536ull
#define ZC_HUFF_MAX_CODE_LEN 32u
#define ZC_HUFF_CODEBOOK_BYTES 256u
#define ZC_HUFF_ROOT_BITS 12u
/* Companion index of Huffman frames (not part of the frame bytes; see
 * DESIGN.md §4): one u32 payload bit offset per ZC_HUFF_INDEX_GRAIN raw
 * bytes, produced by the encoder's scan and consumed by the chunk-parallel
 * decoder. */
#define ZC_HUFF_INDEX_GRAIN 1024u
#define ZC_HUFF_INDEX_ENTRIES (ZC_BATCH_RAW_BYTES / ZC_HUFF_INDEX_GRAIN)

/* ---- status codes ---- */
#define ZC_OK 0
#define ZC_ERR_INVALID_ARGUMENT 1 /* std::invalid_argument in the reference */
#define ZC_ERR_OVERFLOW 2         /* std::overflow_error */
#define ZC_ERR_RUNTIME 3          /* std::runtime_error */
#define ZC_ERR_LOGIC 4            /* std::logic_error */
#define ZC_ERR_CUDA 5             /* CUDA runtime / launch failure, no device */
#define ZC_ERR_PEER 6             /* a peer aborted or timed out (LinkPoisoned) */

/* ---- device error word bits ---- */
#define ZC_DERR_NONFINITE 0x1u  /* quant.cpp:16 "non-finite input" */
#define ZC_DERR_RANGE 0x2u      /* quant.cpp:24 "bin index exceeds int32 range" */
#define ZC_DERR_OVERFLOW 0x4u   /* collectives.cpp:485-488 "symbol sum exceeds 32-bit range" */
#define ZC_DERR_CAPACITY 0x8u   /* collectives.cpp:278-281 "cannot ship even raw" */
#define ZC_DERR_TIMEOUT 0x10u   /* peer flag wait timed out */
#define ZC_DERR_ABORT 0x20u     /* a peer raised its abort flag (poison, transport.cpp:90-95) */
#define ZC_DERR_MISMATCH 0x40u  /* collectives.cpp:450-451 mismatched streams */
#define ZC_DERR_CORRUPT 0x80u   /* an undecodable frame reached a reduction sink (cannot replay a partial add) */

/* ---- enums (frame.hpp:18, collectives.hpp:22, quant.hpp:10, transport.hpp:25) ---- */
enum { ZC_CODEC_RAW = 0, ZC_CODEC_FIXEDLEN = 1, ZC_CODEC_HUFFMAN = 2 };
enum { ZC_PIN_AUTO = 0, ZC_PIN_RAW = 1, ZC_PIN_FIXEDLEN = 2, ZC_PIN_HUFFMAN = 3 };
enum { ZC_QUANT_ERROR_BOUNDED = 0, ZC_QUANT_QSGD = 1, ZC_QUANT_PREQUANTIZED = 2 };
enum { ZC_REGIME_INTRA = 0, ZC_REGIME_INTER = 1 };

/* ---- POD mirrors of the reference structs ---- */
typedef struct zc_frame_header { /* frame.hpp:28-36 */
  uint32_t magic;
  uint8_t version;
  uint8_t codec;
  uint16_t flags;
  uint64_t raw_bytes;
  uint64_t payload_bytes;
  uint64_t params;
} zc_frame_header;

typedef struct zc_codec_cost { /* rea.hpp:44-48 */
  double alpha_sec;
  double enc_bytes_per_sec;
  double dec_bytes_per_sec;
} zc_codec_cost;

typedef struct zc_cost_model { /* rea.hpp:50-53 */
  zc_codec_cost raw;
  zc_codec_cost fixedlen;
  zc_codec_cost huffman;
} zc_cost_model;

typedef struct zc_arb_config { /* rea.hpp:64-79 */
  uint64_t small_batch_threshold_bytes;
  uint64_t huffman_min_raw_bytes;
  uint32_t min_gain_permil;
  uint32_t embed_codebook;
  double lam_enc;
  double lam_dec;
  zc_cost_model cost;
} zc_arb_config;

typedef struct zc_transport_hint { /* rea.hpp:33-36 */
  int32_t regime;
  int32_t _pad;
  double beta_eff_bytes_per_sec;
} zc_transport_hint;

typedef struct zc_sample_stats { /* rea.hpp:18-29 */
  uint64_t sampled_bytes;
  uint64_t hist[256];
  uint64_t max_zigzag;
  double ctx_code_len_bits;
  double self_code_len_bits;
  uint32_t ctx_code_len_valid;
  uint32_t self_code_len_valid;
} zc_sample_stats;

typedef struct zc_codec_estimate { /* rea.hpp:81-88 */
  uint32_t codec;
  uint32_t admissible;
  uint64_t predicted_payload;
  double enc_sec;
  double dec_sec;
  double predicted_sec;
} zc_codec_estimate;

typedef struct zc_arbitration_plan { /* rea.hpp:90-103 */
  uint32_t choice;
  uint32_t _pad;
  zc_codec_estimate raw;
  zc_codec_estimate fixedlen;
  zc_codec_estimate huffman;
} zc_arbitration_plan;

typedef struct zc_encode_result { /* rea.hpp:105-111 */
  uint32_t codec;
  uint32_t _pad;
  uint64_t payload_bytes;
  uint64_t total_bytes;
} zc_encode_result;

typedef struct zc_wire_stats { /* collectives.hpp:36-43 */
  uint64_t frames_by_codec[3];
  uint64_t raw_bytes;
  uint64_t payload_bytes;
  uint64_t total_bytes;
  uint64_t index_bytes; /* companion Huffman index bytes carried beside frames */
  double wall_codec_sec;
} zc_wire_stats;

typedef struct zc_collective_config { /* collectives.hpp:24-34 */
  zc_arb_config arb;
  zc_transport_hint hint; /* NetworkModel -> hint_from_network (rea.hpp:38-40) */
  int32_t pin;            /* ZC_PIN_* */
  int32_t serialized;     /* OverlapMode::Serialized forces lam = 1 (collectives.cpp:71-74) */
  uint64_t fused_codec_min_msg_bytes;
  int32_t per_slot_framing; /* perSlotFraming: collectives batch at ZC_SLOT_BYTES (collectives.cpp:197-199) */
  int32_t _pad;
} zc_collective_config;

/* Opaque handles. */
typedef struct zc_huff_ctx zc_huff_ctx; /* HuffmanContext (huffman.hpp:20-33), device-resident tables */
typedef struct zc_comm zc_comm;         /* one rank of a Communicator (collectives.hpp:111-153) */

/* ---- library ---- */
const char* zc_last_error(void);
const char* zc_version(void);
/* Kernels this library has launched in this process (all devices and streams). */
uint64_t zc_launch_count(void);
int zc_device_count(int* h_count);
/* Plumbing for callers without the CUDA runtime (the C++ layer's host-returning helpers, C and
 * FFI bindings): device allocation on the current device, and synchronous copies / fills whose
 * direction follows the pointers (unified addressing). */
int zc_device_malloc(uint64_t bytes, void** d_out);
void zc_device_free(void* d_ptr);
int zc_memcpy(void* dst, const void* src, uint64_t bytes);
int zc_memset(void* d_ptr, int value, uint64_t bytes);
int zc_stream_synchronize(void* stream); /* NULL = the legacy default stream */
/* Device memory released while a collective is in flight (a communicator, Huffman context or
 * zc_device_free buffer dropped on a rank thread) is freed at the next quiescent point; this
 * performs those frees now when no collective is in flight. */
void zc_flush_deferred(void);
/* Reference defaults: ArbitrationConfig{} (rea.hpp:64-79), TransportHint{} (rea.hpp:33-36),
 * CollectiveConfig{} (collectives.hpp:24-34). */
void zc_default_arb_config(zc_arb_config* h_cfg);
void zc_default_transport_hint(zc_transport_hint* h_hint);
void zc_default_collective_config(zc_collective_config* h_cfg);
/* load_arbitration_config (rea.cpp:240-263): key=value lines, '#' comments. */
int zc_load_arbitration_config(const char* text, zc_arb_config* h_cfg);
/* apply_env_overrides (rea.cpp:270-279): ZCOMM_<KEY> environment overrides. */
int zc_apply_env_overrides(zc_arb_config* h_cfg);

/* ---- L0 frame (frame.hpp:38-50) — host-side pure functions ---- */
int zc_write_header(const zc_frame_header* h, uint8_t* h_dst, uint64_t dst_len); /* frame.cpp:35-45 */
int zc_parse_header(const uint8_t* h_src, uint64_t src_len, zc_frame_header* h_out); /* frame.cpp:47-59; ZC_ERR_INVALID_ARGUMENT when src_len < 32 (nullopt) */
int zc_validate_header(const zc_frame_header* h, uint64_t region_bytes); /* frame.cpp:61-69; returns 1/0 */
/* frame_commit_raw (frame.cpp:71-81) on device; *d_total = 0 when the region is too small. */
int zc_frame_commit_raw(const uint8_t* d_raw, uint64_t raw_len, uint8_t* d_region, uint64_t region_len,
                        uint64_t* d_total, void* stream);

/* ---- L1 quantizer (quant.hpp:29-53) ---- */
/* std::mt19937_64(seed) on the device, bit-exact: d_out[i] = the (skip+i)-th draw.  Chunks of the
 * stream are generated in parallel from jump-ahead states (x^(2^j) mod the generator's
 * characteristic polynomial, built once per process). */
int zc_mt19937_64(uint64_t seed, uint64_t skip, uint64_t n, uint64_t* d_out, void* stream);
/* qsgd_quantize_chunk (quant.cpp:64-82) with rng = mt19937_64(seed) after `skip` draws: one draw
 * per element, in order.  Synchronous; non-finite input -> ZC_ERR_INVALID_ARGUMENT. */
int zc_qsgd_quantize_chunk_f32(const float* d_x, uint64_t n, uint32_t levels, double norm, uint64_t seed,
                               uint64_t skip, int32_t* d_sym, void* stream);
/* The reference's norm: sqrt of the SEQUENTIAL double sum of squares (quant.cpp:87-91), one device
 * thread (any parallel order rounds differently); non-finite input sets ZC_DERR_NONFINITE. */
int zc_qsgd_norm_f32(const float* d_x, uint64_t n, double* d_norm, uint32_t* d_err, void* stream);
/* qsgd_quantize (quant.cpp:84-98): symbols into d_sym, *h_scale = norm (1 when the norm is 0). */
int zc_qsgd_quantize_f32(const float* d_x, uint64_t n, uint32_t levels, uint64_t seed, int32_t* d_sym,
                         double* h_scale, void* stream);
/* checked_absmax (quant.cpp:13-20): *d_absmax = max|x| (exact, as f64); non-finite -> ZC_DERR_NONFINITE. */
int zc_absmax_f32(const float* d_x, uint64_t n, double* d_absmax, uint32_t* d_err, void* stream);
int zc_absmax_f64(const double* d_x, uint64_t n, double* d_absmax, uint32_t* d_err, void* stream);
/* eb_quantize_with_scale / eb_quantize_chunk (quant.cpp:43-62): sym = llround(x/scale), half away from
 * zero, bit-exact with the reference fed (double)x.  Host-side argument checks match quant.cpp:44-46. */
int zc_eb_quantize_f32(const float* d_x, uint64_t n, double scale, int32_t* d_sym, uint32_t* d_err,
                       void* stream);
int zc_eb_quantize_f64(const double* d_x, uint64_t n, double scale, int32_t* d_sym, uint32_t* d_err,
                       void* stream);
/* eb_quantize (quant.cpp:30-41): absmax pass, scale = 2*rel*max (1 when max == 0), quantize.  Synchronous
 * (reads the scale back).  *h_scale receives the bin width. */
int zc_eb_quantize_rel_f32(const float* d_x, uint64_t n, double rel, int32_t* d_sym, double* h_scale,
                           void* stream);
/* dequantize_into (quant.cpp:107-127): ErrorBounded scale*s, Qsgd (scale/levels)*s, PreQuantized s.
 * f64 output is bit-exact with the reference; f32 output is that value rounded once to nearest. */
int zc_dequantize_f64(const int32_t* d_sym, uint64_t n, int32_t mode, double scale, uint32_t levels,
                      double* d_out, void* stream);
int zc_dequantize_f32(const int32_t* d_sym, uint64_t n, int32_t mode, double scale, uint32_t levels,
                      float* d_out, void* stream);

/* ---- L2 codecs (fixedlen.hpp:22-42, huffman.hpp:38-70) ---- */
/* fixedlen_encode (fixedlen.cpp:15-37): *d_payload = bytes (0 on empty input or capacity shortfall),
 * *d_width = pack width. */
int zc_fixedlen_encode(const int32_t* d_sym, uint64_t count, uint8_t* d_out, uint64_t out_cap,
                       uint64_t* d_payload, uint32_t* d_width, void* stream);
/* fixedlen_decode_into (fixedlen.cpp:39-65): *d_ok = 1/0; header is host-side. */
int zc_fixedlen_decode(const zc_frame_header* h, const uint8_t* d_payload, uint64_t payload_len,
                       uint8_t* d_dst, uint64_t dst_len, int32_t* d_ok, void* stream);

/* huffman_build_context (huffman.cpp:165-173).  Returns an immutable context whose tables live in
 * device memory (and a host copy); *out is NULL-safe to destroy.  An all-zero histogram yields a
 * context with valid == 0, exactly like the reference. */
int zc_huff_ctx_create(const uint64_t* h_hist256, zc_huff_ctx** out);
/* Communicator::set_shared_huffman_from_bytes (collectives.cpp:99-106): +1 smoothing. Host bytes. */
int zc_huff_ctx_create_from_bytes(const uint8_t* h_sample, uint64_t n, zc_huff_ctx** out);
/* Same, from a device-resident sample (histogram computed on device). */
int zc_huff_ctx_create_from_device_bytes(const uint8_t* d_sample, uint64_t n, zc_huff_ctx** out, void* stream);
/* huffman_context_from_lengths (huffman.cpp:175-180). */
int zc_huff_ctx_from_lengths(const uint8_t* h_lens256, zc_huff_ctx** out);
int zc_huff_ctx_valid(const zc_huff_ctx* ctx);
int zc_huff_ctx_code_lengths(const zc_huff_ctx* ctx, uint8_t* h_lens256);
int zc_huff_ctx_codes(const zc_huff_ctx* ctx, uint32_t* h_code256, uint32_t* h_rev256);
void zc_huff_ctx_destroy(zc_huff_ctx* ctx);
/* huffman_expected_code_len / huffman_self_code_len (huffman.cpp:182-214), host-side; *h_valid 0 = nullopt. */
int zc_huffman_expected_code_len(const zc_huff_ctx* ctx, const uint64_t* h_hist256, double* h_bits,
                                 int32_t* h_valid);
int zc_huffman_self_code_len(const uint64_t* h_hist256, double* h_bits, int32_t* h_valid);
/* huffman_encode (huffman.cpp:216-246), shared-context mode (embed == 0) or embedded codebook
 * (embed == 1).  *d_payload = bytes or 0 on failure.  d_index (optional, may be NULL) receives the
 * companion index: ceil(n / ZC_HUFF_INDEX_GRAIN) u32 bit offsets relative to the code stream start. */
int zc_huffman_encode(const uint8_t* d_raw, uint64_t n, const zc_huff_ctx* ctx, uint8_t* d_out,
                      uint64_t out_cap, int32_t embed, uint64_t* d_payload, uint32_t* d_index, void* stream);
/* huffman_decode_into (huffman.cpp:248-316).  With d_index the decode is chunk-parallel; with
 * d_index == NULL (a frame produced elsewhere, e.g. by the CPU reference) a sequential single-warp
 * decoder is used.  *d_ok = 1/0. */
int zc_huffman_decode(const zc_frame_header* h, const uint8_t* d_payload, uint64_t payload_len,
                      const zc_huff_ctx* shared_ctx, const uint32_t* d_index, uint8_t* d_dst,
                      uint64_t dst_len, int32_t* d_ok, void* stream);

/* ---- L3 runtime entropy arbitration (rea.hpp:114-133) ---- */
/* profile_sample (rea.cpp:93-118) on device; ctx may be NULL. */
int zc_profile_sample(const uint8_t* d_raw, uint64_t n, const zc_huff_ctx* ctx, zc_sample_stats* d_stats,
                      void* stream);
/* predict_payload (rea.cpp:120-143) and arbitrate_plan (rea.cpp:145-176): host-callable builds of the
 * same __host__ __device__ code the device selector runs. */
uint64_t zc_predict_payload(int32_t codec, uint64_t raw_bytes, const zc_sample_stats* h_stats,
                            const zc_arb_config* h_cfg);
int zc_arbitrate_plan(uint64_t raw_bytes, uint64_t payload_cap, const zc_sample_stats* h_stats,
                      const zc_transport_hint* h_hint, const zc_huff_ctx* ctx, const zc_arb_config* h_cfg,
                      zc_arbitration_plan* h_plan);
/* encode_best (rea.cpp:178-238), Algorithm 1, fully on device: profile -> plan -> materialise -> post-check
 * -> raw fallback.  Result in *d_result (no host round-trip). */
int zc_encode_best(const uint8_t* d_raw, uint64_t raw_len, uint8_t* d_stage, uint64_t stage_len,
                   const zc_transport_hint* h_hint, const zc_huff_ctx* ctx, const zc_arb_config* h_cfg,
                   zc_encode_result* d_result, void* stream);

/* ---- batched hot path (RankCtx::send_batch / recv_batch, collectives.cpp:201-348) ----
 * A message of raw_bytes is cut into ceil(raw_bytes / 4 MiB) batches (transport.hpp:137-142); batch b
 * is encoded into stage b at d_stages + b*stage_stride (capacity stage_len, normally
 * ZC_STAGE_BANK_BYTES).  `pin` follows send_batch: AUTO = encode_best, others materialise the pinned
 * codec and fall back to raw only on hard failure.  d_index (Huffman companion index) holds
 * ZC_HUFF_INDEX_ENTRIES u32 per batch and may be NULL when Huffman cannot be chosen. */
int zc_encode_batches_sym(const int32_t* d_sym, uint64_t raw_bytes, uint8_t* d_stages, uint64_t stage_stride,
                          uint64_t stage_len, int32_t pin, const zc_transport_hint* h_hint,
                          const zc_huff_ctx* ctx, const zc_arb_config* h_cfg, zc_encode_result* d_results,
                          uint32_t* d_index, uint32_t* d_err, void* stream);
/* Fused quantize + encode: symbols are produced from fp32 input on the fly (never written to HBM). */
int zc_encode_batches_f32(const float* d_x, uint64_t count, double scale, uint8_t* d_stages,
                          uint64_t stage_stride, uint64_t stage_len, int32_t pin,
                          const zc_transport_hint* h_hint, const zc_huff_ctx* ctx, const zc_arb_config* h_cfg,
                          zc_encode_result* d_results, uint32_t* d_index, uint32_t* d_err, void* stream);
/* recv_batch decode dispatch (collectives.cpp:314-336), including the raw-copy fallback for
 * unintelligible frames.  d_sent (optional) holds each frame's committed size — the received
 * region that validate_header checks against (collectives.cpp:313); NULL means stage_len.
 * d_codec_out (optional) receives the codec decoded per batch, 0xFFFFFFFF for the raw fallback.
 * Output either raw symbols (int32), fused dequantized fp32, or (add_sym) the reduce-scatter
 * sink: decoded symbols added into d_acc with the int32 overflow check (ZC_DERR_OVERFLOW). */
int zc_decode_batches_sym(const uint8_t* d_stages, uint64_t stage_stride, uint64_t stage_len,
                          const zc_encode_result* d_sent, uint64_t raw_bytes, const zc_huff_ctx* ctx,
                          const uint32_t* d_index, int32_t* d_sym, uint32_t* d_codec_out, void* stream);
int zc_decode_batches_f32(const uint8_t* d_stages, uint64_t stage_stride, uint64_t stage_len,
                          const zc_encode_result* d_sent, uint64_t count, double scale, const zc_huff_ctx* ctx,
                          const uint32_t* d_index, float* d_out, uint32_t* d_codec_out, void* stream);
int zc_decode_batches_add_sym(const uint8_t* d_stages, uint64_t stage_stride, uint64_t stage_len,
                              const zc_encode_result* d_sent, uint64_t raw_bytes, const zc_huff_ctx* ctx,
                              const uint32_t* d_index, int32_t* d_acc, uint32_t* d_err, void* stream);
/* Host-buffer codec round trip: the reference's per-batch send_encoded -> recv_decoded over a message
 * (collectives.cpp:201-348 with quantize / dequantize, quant.cpp:43-62 and 107-127), the call that
 * RankCtx::send_encoded + recv_decoded make on host spans.  h_x (host fp32; pinned for overlap) -> H2D ->
 * fused quantize+encode (frames land in d_stages / d_results / d_index exactly as zc_encode_batches_f32
 * writes them) -> decode+dequantize -> D2H -> h_y.  Pipelined in groups of `group_batches` 4 MiB batches
 * (0 = 4) over internal H2D / kernel / D2H streams so both copy directions and the kernels overlap; ordered after earlier work on `stream`,
 * and later work on `stream` waits for it.  d_work: count floats of device scratch (16-byte aligned). */
int zc_codec_roundtrip_host_f32(const float* h_x, uint64_t count, double scale, float* d_work, uint8_t* d_stages,
                                uint64_t stage_stride, uint64_t stage_len, int32_t pin,
                                const zc_transport_hint* h_hint, const zc_huff_ctx* ctx, const zc_arb_config* h_cfg,
                                zc_encode_result* d_results, uint32_t* d_index, uint32_t* d_err, float* h_y,
                                uint32_t group_batches, void* stream);

/* ---- L6 collectives (collectives.hpp:48-153) ----
 * One zc_comm per rank.  Multi-process: each rank calls zc_comm_create, exchanges the opaque
 * zc_comm_export() blob with its peers through any bootstrap (torch.distributed here), then calls
 * zc_comm_connect() with all ranks' blobs (rank order).  Single-process groups (several ranks on one
 * or more local devices, the analogue of the reference's thread-per-rank Communicator::run) use
 * zc_comm_create_group() and the zc_group_* calls, which enqueue every rank's kernels before
 * waiting on any (ranks' kernels must run concurrently, exactly like the reference's rank threads).
 * Each zc_comm_* collective runs on the rank's internal stream and returns when it has completed
 * (the `stream` argument is reserved); a failure on any rank is broadcast to every rank's error
 * word (the reference's link poisoning, transport.cpp:90-95) and reported with the root cause's
 * status, and the communicator then needs zc_comm_reset() (after a barrier, multi-process) to open
 * a clean epoch (transport.cpp:97-105) — group calls reset automatically. */
int zc_comm_create(int rank, int nranks, int device, const zc_collective_config* h_cfg, zc_comm** out);
int zc_comm_export_size(void);
int zc_comm_export(zc_comm* comm, uint8_t* h_blob);
int zc_comm_connect(zc_comm* comm, const uint8_t* h_blobs /* nranks * zc_comm_export_size() */);
int zc_comm_create_group(int nranks, const int* h_devices, const zc_collective_config* h_cfg,
                         zc_comm** out /* array of nranks */);
void zc_comm_destroy(zc_comm* comm);
int zc_comm_rank(const zc_comm* comm);
int zc_comm_nranks(const zc_comm* comm);
/* Communicator::set_shared_huffman[_from_bytes] (collectives.cpp:92-106); ctx is copied. */
int zc_comm_set_shared_huffman(zc_comm* comm, const zc_huff_ctx* ctx);
/* RankCtx::allreduce (collectives.cpp:423-503) on device-resident symbols, in place.  The meta ring
 * and scale reconciliation (:428-458) run first; *h_scale is in/out. */
int zc_comm_allreduce_sym(zc_comm* comm, int32_t* d_sym, uint64_t count, int32_t mode, double* h_scale,
                          uint32_t levels, void* stream);
/* RankCtx::allreduce_eb (collectives.cpp:505-516): global abs-max, quantize with the shared scale
 * (device-resident, no host round-trip), ring RS+AG, dequantize into d_out (fp32, or fp64 when
 * out_f64). */
int zc_comm_allreduce_eb_f32(zc_comm* comm, const float* d_x, void* d_out, int32_t out_f64, uint64_t count,
                             double rel, void* stream);
/* Reduce-scatter phase of allreduce alone: afterwards rank r owns fully reduced chunk (r+1) mod n,
 * chunk bounds c*count/n (collectives.cpp:465-467).  d_sym is in/out (whole buffer). */
int zc_comm_reduce_scatter_sym(zc_comm* comm, int32_t* d_sym, uint64_t count, void* stream);
/* RankCtx::allgather (collectives.cpp:525-544): d_all has nranks*block symbols; this rank's block
 * must already be at d_all + rank*block. */
int zc_comm_allgather_sym(zc_comm* comm, int32_t* d_all, uint64_t block, void* stream);
/* RankCtx::allreduce_max (collectives.cpp:398-421). */
int zc_comm_allreduce_max(zc_comm* comm, double v, double* h_out, void* stream);
/* RankCtx::allreduce_qsgd (collectives.cpp:518-523): qsgd_quantize on the device (sequential norm,
 * bit-exact mt19937_64 draws), the compressed ring allreduce in QSGD mode (scale reconciliation as
 * the reference's), dequantize (scale/levels)*sym into d_out (fp32, or fp64 when out_f64). */
int zc_comm_allreduce_qsgd_f32(zc_comm* comm, const float* d_x, void* d_out, int32_t out_f64, uint64_t count,
                               uint32_t levels, uint64_t seed, void* stream);
/* RankCtx::alltoall (collectives.cpp:546-567): d_send / d_recv hold nranks*block symbols; block j of
 * d_send goes to rank j, block j of d_recv comes from rank j (zc_comm_alltoall_sym copies the own
 * block).  Frames use cfg.pin. */
int zc_comm_alltoall_sym(zc_comm* comm, const int32_t* d_send, int32_t* d_recv, uint64_t block, void* stream);
/* RankCtx::broadcast (collectives.cpp:569-591): root's d_data to every rank along the ring, in place;
 * a root outside [0, nranks) is ZC_ERR_INVALID_ARGUMENT. */
int zc_comm_broadcast_sym(zc_comm* comm, int32_t* d_data, uint64_t count, int32_t root, void* stream);
/* CollectiveRequest / group_execute (collectives.hpp:94-105, collectives.cpp:593-616): requests run
 * in order as one submission (one host wait at the end).  AllReduce: sym/count in place with
 * mode/scale(in-out)/levels; AllGather: sym = this rank's block of `count`, recv = nranks*count;
 * AllToAll: sym = nranks*count send symbols (count = block), recv = nranks*count; Broadcast:
 * sym/count in place from root.  A request missing its buffer is ZC_ERR_INVALID_ARGUMENT (the reference's
 * "request needs an output"). */
enum { ZC_COLL_ALLREDUCE = 0, ZC_COLL_ALLGATHER = 1, ZC_COLL_ALLTOALL = 2, ZC_COLL_BROADCAST = 3 };
typedef struct zc_coll_request {
  int32_t op;
  int32_t root;
  int32_t mode;
  uint32_t levels;
  int32_t* sym;
  int32_t* recv;
  uint64_t count;
  double scale;
} zc_coll_request;
int zc_comm_group_execute(zc_comm* comm, zc_coll_request* reqs, int32_t nreqs, void* stream);
/* Measured send/receive timeline of the staged ring path (the B200 counterpart of the modelled
 * BatchTimelineRow / write_timeline_csv, pipeline.hpp:32-46, pipeline.cpp:160-170): CUDA events on
 * the communicator stream around every piece.  Send rows (kind 0) are per 4 MiB batch: the piece's
 * encode, whose stores ARE the NVLink transfer, from launch to publication (start/end), with the
 * frame's codec and total bytes.  Receive rows (kind 1) are per piece: wait start, frame arrival
 * (ready) and decode end.  Times are seconds since zc_comm_timeline_enable.  max_pieces = 0
 * disables; rows beyond the capacity are dropped. */
typedef struct zc_timeline_row {
  uint64_t seq;       /* piece sequence number (the receiver's count; sender and receiver agree) */
  int32_t kind;       /* 0 send, 1 receive */
  int32_t peer;       /* rank sent to / received from (-1: any) */
  uint32_t batch;     /* batch within the piece (send rows) */
  uint32_t codec;     /* ZC_CODEC_* of the frame (send rows); 0xFF for receive rows */
  uint64_t raw_bytes;
  uint64_t total_bytes; /* frame bytes (send rows); 0 for receive rows */
  double start_sec, ready_sec, end_sec;
} zc_timeline_row;
int zc_comm_timeline_enable(zc_comm* comm, int32_t max_pieces);
/* Rows recorded so far (waits for the rank's queued work): *n_rows = the row count, at most cap
 * of them written to rows (rows may be NULL with cap 0). */
int zc_comm_timeline_rows(zc_comm* comm, zc_timeline_row* rows, int32_t cap, int32_t* n_rows);
/* Seconds from a's timeline origin to b's (both enabled on the same device). */
int zc_comm_timeline_origin_delta(zc_comm* a, zc_comm* b, double* sec);
/* Waits for the rank's queued work, checks its device error word, and maps it to a status. */
int zc_comm_sync(zc_comm* comm);
/* Clean epoch after an aborted collective (Connection::reset_sim, transport.cpp:97-105). */
int zc_comm_reset(zc_comm* comm);
/* RankCtx::send_encoded / recv_decoded (collectives.cpp:350-364): point-to-point, any pair of ranks.
 * The message is cut into batches (4 MiB, or ZC_SLOT_BYTES under per-slot framing), each framed by
 * send_batch's dispatch (cfg.pin) straight into the pair's channel in the receiver's memory and
 * counted in the sender's WireStats; the receiver decodes each frame (recv_batch, raw-copy
 * fallback included).  A send returns once its frames are written, which needs the receiver to
 * have consumed all but the last two pieces (the credit window); a receive returns with the data
 * in d_dst. */
int zc_comm_send_encoded(zc_comm* comm, int32_t peer, const void* d_raw, uint64_t raw_bytes, void* stream);
int zc_comm_recv_decoded(zc_comm* comm, int32_t peer, void* d_dst, uint64_t dst_bytes, void* stream);
/* Link poisoning from the host (Communicator::run when one rank's body throws, transport.cpp:90-95):
 * every rank's pending and next collective fails with ZC_ERR_PEER until zc_comm_reset. */
int zc_comm_abort(zc_comm* comm);
/* Communicator::wire_stats / reset_stats (collectives.cpp:175-190). */
int zc_comm_wire_stats(zc_comm* comm, zc_wire_stats* h_out);
int zc_comm_reset_stats(zc_comm* comm);

/* Single-process groups (Communicator::run over all ranks): arrays are indexed by rank. */
int zc_group_allreduce_sym(zc_comm* const* comms, int nranks, int32_t* const* d_syms, uint64_t count,
                           int32_t mode, double* h_scales, uint32_t levels);
int zc_group_allreduce_eb_f32(zc_comm* const* comms, int nranks, const float* const* d_xs, void* const* d_outs,
                              int32_t out_f64, uint64_t count, double rel);
int zc_group_reduce_scatter_sym(zc_comm* const* comms, int nranks, int32_t* const* d_syms, uint64_t count);
int zc_group_allgather_sym(zc_comm* const* comms, int nranks, int32_t* const* d_alls, uint64_t block);
int zc_group_allreduce_max(zc_comm* const* comms, int nranks, const double* h_vs, double* h_outs);
int zc_group_alltoall_sym(zc_comm* const* comms, int nranks, const int32_t* const* d_sends, int32_t* const* d_recvs,
                          uint64_t block);
int zc_group_broadcast_sym(zc_comm* const* comms, int nranks, int32_t* const* d_datas, uint64_t count, int32_t root);
/* group_execute on every rank (reqs[r] = rank r's request list, same ops in the same order). */
int zc_group_execute(zc_comm* const* comms, int nranks, zc_coll_request* const* reqs, int32_t nreqs);

#ifdef __cplusplus
}
#endif
#endif /* ZCOMM_B200_H */
