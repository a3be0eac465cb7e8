// zc_kernels.h — host launchers of the sm_100a kernels (internal to libzcomm_b200.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <utility>

#include "zc_common.cuh"

namespace zc {

enum SrcKind : int { SRC_BYTES = 0, SRC_F32 = 1, SRC_F64 = 2 };
// OUT_ADD_Q: the reduce-scatter sink of allreduce_eb — the local fp32 chunk (DecParams::acc_f32) is
// quantized on the fly and added to the decoded symbols; the int32 sum goes to `out`.
enum OutKind : int { OUT_BYTES = 0, OUT_F32 = 1, OUT_F64 = 2, OUT_ADD_I32 = 3, OUT_ADD_Q = 4 };

// Encode modes.
enum EncMode : int {
  ENC_SEND = 0,     // send_batch semantics: pin dispatch, raw fallback, capacity error bit
  ENC_BEST = 1,     // encode_best semantics (result {0,0,0} instead of an error bit)
  ENC_BARE_FL = 2,  // fixedlen_encode: bare payload, no header, 0 on capacity shortfall
  ENC_BARE_HF = 3,  // huffman_encode: bare payload (+ codebook when embed), 0 on failure
  ENC_PROFILE = 4,  // profile_sample only
};

// One rank's view of its two ring links (collectives.cpp:76-84 links, transport.hpp:106-134
// staging banks).  Receive banks live in the RECEIVER's HBM; the sender's kernel stores the
// frame straight into them over NVLink (or same-device memory in loopback groups) and publishes
// {length, sequence} with a system-scope release; the receiver's kernel acquires the sequence,
// consumes the frame and returns the bank with a release on the sender's credit word.
struct Link {
  uint8_t* tx_banks;               // successor's receive banks (peer-mapped)
  unsigned long long* tx_ready;    // successor's ready words [nbanks]
  unsigned long long* tx_len;      // successor's frame-length words [nbanks]
  unsigned long long* tx_credit;   // our credit words [nbanks], written by the successor
  const uint8_t* rx_banks;         // our receive banks
  unsigned long long* rx_ready;    // our ready words
  unsigned long long* rx_len;      // our frame-length words
  unsigned long long* rx_credit;   // predecessor's credit words (peer-mapped)
  uint64_t bank_stride;            // bytes per bank (frame region + companion index)
  uint64_t idx_off;                // companion index offset inside a bank
  uint32_t nbanks;
  uint32_t nranks;
  uint64_t tx_seq0, rx_seq0;       // frames already sent / received on this link
  uint32_t* err_self;              // our error word
  uint32_t* const* err_all;        // every rank's error word (device array of peer pointers)
  unsigned long long timeout_ns;
  zc_wire_stats* wire;             // device-side WireStats accumulation (own memory)
  int max_clusters;                // residency cap for this launch (loopback groups share a GPU)
};

struct EncParams {
  const void* src;
  int src_kind;
  int mode;
  int pin;
  int embed;           // bare huffman: prepend codebook
  double scale, rcp;   // float sources
  const double* dscale;  // or, when set, {scale, 1/scale} in device memory (allreduce_eb's agreed scale)
  const uint32_t* maxzz_in;  // SRC_BYTES: each unit's max zig-zag, known from the producer (or null)
  int no_spec;               // fp32: take the two-read FixedLen path (heavy-tailed data defeats the guess)
  uint64_t total_bytes;
  uint64_t unit_bytes;
  uint32_t nunits;
  uint32_t _pad;
  uint8_t* stages;
  uint64_t stride;
  uint64_t stage_len;  // bytes available at each stage (header included unless bare)
  zc_transport_hint hint;
  zc_arb_config cfg;
  const DevHuff* ctx;  // may be null
  zc_encode_result* results;
  uint32_t* index;     // companion index, index_stride u32 per unit (may be null)
  uint64_t index_stride;
  uint32_t* err;
  zc_sample_stats* stats;  // per-unit stats (may be null)
  uint64_t* bare_payload;  // bare modes: payload bytes
  uint32_t* bare_width;    // bare fixedlen: width
  // ring mode (fused reduce-scatter step): frames go to the successor's banks; with rx_add the
  // predecessor's frame for the same unit is first decoded and added into `src` (the local
  // chunk), and the sum is what gets encoded — decode -> reduce -> re-encode in one kernel.
  int link_tx;
  int link_rx_add;  // receive part enabled (the reduce-scatter sink adds)
  int rx_store;     // receive sink stores the decoded symbols instead of adding (all-gather step)
  void* rx_dst;     // incoming chunk (local symbols)
  uint64_t rx_total_bytes;
  uint32_t rx_nunits;
  Link L;
};

struct DecParams {
  const uint8_t* stages;
  uint64_t stride;
  uint64_t region;         // bytes of each received region when frame_len is null
  const zc_encode_result* frame_len;  // per-unit committed frame (total_bytes) or null
  uint64_t total_bytes;    // raw bytes of the message
  uint64_t unit_bytes;
  uint32_t nunits;
  int out_kind;
  void* out;
  double scale;            // dequantization factor for OUT_F32 / OUT_F64
  const double* dscale;    // or, when set, {scale, 1/scale} in device memory
  const float* acc_f32;    // OUT_ADD_Q: the local fp32 chunk quantized into the sums
  uint32_t* maxzz_out;     // OUT_ADD_*: per unit, atomicMax of the sums' zig-zag (or null)
  const DevHuff* ctx;
  const uint32_t* index;   // may be null
  uint64_t index_stride;
  uint32_t* codec_out;     // per unit decoded codec, or 0xFFFFFFFF for the raw fallback (may be null)
  uint32_t* flags;         // per unit scratch: 1 = needs sequential Huffman decode (device, >= nunits)
  uint32_t* err;
  int bare;                // bare decode: `stages` is one payload and `hdr` describes it
  zc_frame_header hdr;
  int32_t* ok_out;         // bare decode result
  int fast;                // zc_fixed.cu's decoder has handled the valid FixedLen / RAW units
  int own_frames;          // the frames come from this library's batched encoder without a Huffman
                           // context: all valid FixedLen / RAW, so the general kernels are skipped
  int huff_lane;           // (set by launch_decode) Huffman grains on the per-lane decoder only
};

// Quantizer bin width of a float source / dequantization factor: the host value, or the device
// pair {scale, 1/scale} (allreduce_eb: agreed on the device, never seen by the host).
__device__ __forceinline__ double enc_scale(const EncParams& p) { return p.dscale ? p.dscale[0] : p.scale; }
__device__ __forceinline__ double enc_rcp(const EncParams& p) { return p.dscale ? p.dscale[1] : p.rcp; }
__device__ __forceinline__ double dec_scale(const DecParams& p) { return p.dscale ? p.dscale[0] : p.scale; }

// One piece of a ring step fused with the next step's send of the same chunk (zc_fixed.cu):
// decode the predecessor's FixedLen / RAW frames -> reduce into the local chunk (int32 add, or the
// local fp32 quantized on the fly) -> per unit: range and window range -> decide -> pack the sums
// into the successor's region.  FixedLen / RAW only (no Huffman context, no embedded codebooks).
struct FusedParams {
  const uint8_t* in_stages;  // this rank's received piece region
  uint64_t in_stride;
  const zc_encode_result* in_res;
  int sink;                  // OUT_ADD_I32 (sums in place) or OUT_ADD_Q (sum = q(x) + decoded)
  int32_t* sum;              // local chunk piece (int32)
  const float* x;            // OUT_ADD_Q: local fp32 chunk piece
  const double* dscale;      // OUT_ADD_Q: {scale, 1/scale}
  EncParams enc;             // the successor's frames: src = sum (SRC_BYTES), stages / results there
  uint32_t* err;
};
cudaError_t launch_ring_fused(const FusedParams& f, void* scratch, cudaStream_t s);
size_t ring_fused_scratch_bytes(uint32_t nunits);

// Programmatic dependent launch: the kernel may begin while the previous kernel on the stream drains
// (its CTAs are placed as the previous ones retire); it executes griddepcontrol.wait before it reads
// anything the previous kernels wrote, so stream semantics are unchanged.  Used along the codec
// step's chain of mostly-empty kernels (redo emit, Huffman side, general decoder), whose launch and
// placement latency would otherwise add to the step.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  return cudaLaunchKernelEx(&lc, kernel, std::forward<Args>(args)...);
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// Every kernel launch of the library bumps one process-wide counter (zc_launch_count), so callers
// can state how many of OUR kernels a region launched.
void note_launch();
void note_launches(uint64_t k);  // a replayed graph's launches
// Function attributes (cudaFuncSetAttribute) are per device: true the first time the current
// device is seen by the caller's `mask`.
inline bool first_on_device(std::atomic<uint64_t>& mask) {
  int d = 0;
  cudaGetDevice(&d);
  const uint64_t bit = 1ull << (d & 63);
  return (mask.fetch_or(bit) & bit) == 0;
}

cudaError_t launch_encode(const EncParams& p, cudaStream_t s);
// The default batched send path: profile -> scan -> emit streaming kernels (zc_batch.cu).
cudaError_t launch_encode_batch(const EncParams& p, void* scratch, cudaStream_t s);
size_t batch_scratch_bytes(uint32_t nunits);
void preload_batch_kernels();
// zc_fixed.cu: the fp32 FixedLen / RAW units of the batched path (TMA-pipelined).
bool fixed_path_ok(const EncParams& p);
cudaError_t launch_fixed_range(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                               cudaStream_t s);
cudaError_t launch_fixed_emit(const EncParams& p, void* scratch, uint64_t total_slices, uint32_t s_full, int sms,
                              cudaStream_t s);
bool fixed_decode_ok(const DecParams& p);
cudaError_t launch_fixed_decode(const DecParams& p, cudaStream_t s);
void preload_fixed_kernels();
int encode_max_clusters();
// Force module loading of every kernel (lazy loading may otherwise stall a launch behind a
// running peer-waiting kernel).
void preload_encode_kernels();
void preload_decode_kernels();
void preload_quant_kernels();
cudaError_t launch_decode(const DecParams& p, cudaStream_t s);
cudaError_t launch_absmax(const void* x, int src_kind, uint64_t n, double* out, uint32_t* err, cudaStream_t s);
cudaError_t launch_quantize(const void* x, int src_kind, uint64_t n, double scale, int32_t* sym, uint32_t* err,
                            cudaStream_t s);
cudaError_t launch_dequantize(const int32_t* sym, uint64_t n, double k, int prequant, void* out, int out_f64,
                              cudaStream_t s);
cudaError_t launch_commit_raw(const uint8_t* raw, uint64_t n, uint8_t* region, uint64_t cap, uint64_t* total,
                              cudaStream_t s);
cudaError_t launch_hist(const uint8_t* d, uint64_t n, uint64_t* hist, cudaStream_t s);

}  // namespace zc
