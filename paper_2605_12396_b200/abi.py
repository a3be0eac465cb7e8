"""ctypes declarations mirroring ``include/zcomm_b200.h`` (types and constants only).

These are the POD structs of the C-ABI boundary; each mirrors a reference struct
(paths relative to /root/reference/proj/core/).  No compute lives here.
"""
import ctypes as C

HEADER_BYTES = 32                       # frame.hpp:15
FRAME_MAGIC = 0x464D435A                # frame.hpp:13
FRAME_VERSION = 1                       # frame.hpp:14
FLAG_EMBEDDED_CODEBOOK = 0x0001         # frame.hpp:16
SLOT_BYTES = 512 * 1024                 # transport.hpp:17
SLOTS_PER_CHANNEL = 8                   # transport.hpp:18
BATCH_RAW_BYTES = SLOT_BYTES * SLOTS_PER_CHANNEL   # transport.hpp:20
STAGE_BANK_BYTES = HEADER_BYTES + BATCH_RAW_BYTES  # transport.hpp:22
SAMPLE_WINDOW_BYTES = 64 * 1024         # rea.hpp:16
HUFF_MAX_CODE_LEN = 32                  # huffman.hpp:13
HUFF_CODEBOOK_BYTES = 256               # huffman.hpp:14
HUFF_ROOT_BITS = 12                     # huffman.hpp:15
HUFF_INDEX_GRAIN = 1024
HUFF_INDEX_ENTRIES = BATCH_RAW_BYTES // HUFF_INDEX_GRAIN

OK, ERR_INVALID_ARGUMENT, ERR_OVERFLOW, ERR_RUNTIME, ERR_LOGIC, ERR_CUDA, ERR_PEER = range(7)
DERR_NONFINITE, DERR_RANGE, DERR_OVERFLOW, DERR_CAPACITY = 0x1, 0x2, 0x4, 0x8
DERR_TIMEOUT, DERR_ABORT, DERR_MISMATCH = 0x10, 0x20, 0x40

CODEC_RAW, CODEC_FIXEDLEN, CODEC_HUFFMAN = 0, 1, 2
PIN_AUTO, PIN_RAW, PIN_FIXEDLEN, PIN_HUFFMAN = 0, 1, 2, 3
QUANT_ERROR_BOUNDED, QUANT_QSGD, QUANT_PREQUANTIZED = 0, 1, 2
REGIME_INTRA, REGIME_INTER = 0, 1
CODEC_NAMES = {CODEC_RAW: "raw", CODEC_FIXEDLEN: "fixedlen", CODEC_HUFFMAN: "huffman"}
PIN_NAMES = {PIN_AUTO: "auto", PIN_RAW: "raw", PIN_FIXEDLEN: "fixedlen", PIN_HUFFMAN: "huffman"}


class FrameHeader(C.Structure):          # frame.hpp:28-36
    _fields_ = [("magic", C.c_uint32), ("version", C.c_uint8), ("codec", C.c_uint8),
                ("flags", C.c_uint16), ("raw_bytes", C.c_uint64), ("payload_bytes", C.c_uint64),
                ("params", C.c_uint64)]


class CodecCost(C.Structure):            # rea.hpp:44-48
    _fields_ = [("alpha_sec", C.c_double), ("enc_bytes_per_sec", C.c_double),
                ("dec_bytes_per_sec", C.c_double)]


class CostModel(C.Structure):            # rea.hpp:50-53
    _fields_ = [("raw", CodecCost), ("fixedlen", CodecCost), ("huffman", CodecCost)]


class ArbConfig(C.Structure):            # rea.hpp:64-79
    _fields_ = [("small_batch_threshold_bytes", C.c_uint64), ("huffman_min_raw_bytes", C.c_uint64),
                ("min_gain_permil", C.c_uint32), ("embed_codebook", C.c_uint32),
                ("lam_enc", C.c_double), ("lam_dec", C.c_double), ("cost", CostModel)]


class TransportHint(C.Structure):        # rea.hpp:33-36
    _fields_ = [("regime", C.c_int32), ("_pad", C.c_int32), ("beta_eff_bytes_per_sec", C.c_double)]


class SampleStats(C.Structure):          # rea.hpp:18-29
    _fields_ = [("sampled_bytes", C.c_uint64), ("hist", C.c_uint64 * 256), ("max_zigzag", C.c_uint64),
                ("ctx_code_len_bits", C.c_double), ("self_code_len_bits", C.c_double),
                ("ctx_code_len_valid", C.c_uint32), ("self_code_len_valid", C.c_uint32)]


class CodecEstimate(C.Structure):        # rea.hpp:81-88
    _fields_ = [("codec", C.c_uint32), ("admissible", C.c_uint32), ("predicted_payload", C.c_uint64),
                ("enc_sec", C.c_double), ("dec_sec", C.c_double), ("predicted_sec", C.c_double)]


class ArbitrationPlan(C.Structure):      # rea.hpp:90-103
    _fields_ = [("choice", C.c_uint32), ("_pad", C.c_uint32), ("raw", CodecEstimate),
                ("fixedlen", CodecEstimate), ("huffman", CodecEstimate)]


class EncodeResult(C.Structure):         # rea.hpp:105-111
    _fields_ = [("codec", C.c_uint32), ("_pad", C.c_uint32), ("payload_bytes", C.c_uint64),
                ("total_bytes", C.c_uint64)]


class WireStats(C.Structure):            # collectives.hpp:36-43
    _fields_ = [("frames_by_codec", C.c_uint64 * 3), ("raw_bytes", C.c_uint64),
                ("payload_bytes", C.c_uint64), ("total_bytes", C.c_uint64), ("index_bytes", C.c_uint64),
                ("wall_codec_sec", C.c_double)]


COLL_ALLREDUCE, COLL_ALLGATHER, COLL_ALLTOALL, COLL_BROADCAST = 0, 1, 2, 3  # CollOp, collectives.hpp:17


class CollRequest(C.Structure):          # CollectiveRequest, collectives.hpp:94-101
    _fields_ = [("op", C.c_int32), ("root", C.c_int32), ("mode", C.c_int32), ("levels", C.c_uint32),
                ("sym", C.c_void_p), ("recv", C.c_void_p), ("count", C.c_uint64), ("scale", C.c_double)]


class TimelineRow(C.Structure):          # zc_timeline_row (measured BatchTimelineRow, pipeline.hpp:32-46)
    _fields_ = [("seq", C.c_uint64), ("kind", C.c_int32), ("peer", C.c_int32), ("batch", C.c_uint32),
                ("codec", C.c_uint32), ("raw_bytes", C.c_uint64), ("total_bytes", C.c_uint64),
                ("start_sec", C.c_double), ("ready_sec", C.c_double), ("end_sec", C.c_double)]


class CollectiveConfig(C.Structure):     # collectives.hpp:24-34
    _fields_ = [("arb", ArbConfig), ("hint", TransportHint), ("pin", C.c_int32),
                ("serialized", C.c_int32), ("fused_codec_min_msg_bytes", C.c_uint64),
                ("per_slot_framing", C.c_int32), ("_pad", C.c_int32)]


def default_arb_config() -> ArbConfig:
    """ArbitrationConfig{} defaults (rea.hpp:50-53, 64-79)."""
    c = ArbConfig()
    c.small_batch_threshold_bytes = 4096
    c.huffman_min_raw_bytes = 65536
    c.min_gain_permil = 50
    c.embed_codebook = 0
    c.lam_enc = 0.25
    c.lam_dec = 0.25
    c.cost.fixedlen.alpha_sec, c.cost.fixedlen.enc_bytes_per_sec, c.cost.fixedlen.dec_bytes_per_sec = 1.0e-6, 250.0e9, 300.0e9
    c.cost.huffman.alpha_sec, c.cost.huffman.enc_bytes_per_sec, c.cost.huffman.dec_bytes_per_sec = 1.5e-6, 120.0e9, 150.0e9
    return c


def make_hint(beta: float = 10.0 * 1073741824.0, regime: int = REGIME_INTER) -> TransportHint:
    """TransportHint{} defaults: inter-node, 10 GiB/s (rea.hpp:33-36, transport.hpp:33-35)."""
    h = TransportHint()
    h.regime = regime
    h.beta_eff_bytes_per_sec = beta
    return h


def default_collective_config(pin: int = PIN_AUTO) -> CollectiveConfig:
    """CollectiveConfig{} defaults (collectives.hpp:24-34)."""
    c = CollectiveConfig()
    c.arb = default_arb_config()
    c.hint = make_hint()
    c.pin = pin
    c.serialized = 0
    c.fused_codec_min_msg_bytes = BATCH_RAW_BYTES
    return c
