"""CPU: the product library's C-ABI boundary without a GPU.

* libzcomm_b200.so loads and exports every function include/zcomm_b200.h declares;
* the host-side pure functions of the boundary (frame header codec, selector, Huffman context
  builder, config parsing) match the reference (golden fixtures from oracle/_ref) — these are the
  same __host__ __device__ code paths the kernels run;
* no compute entry point is called (no CUDA device here).
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2605_12396_b200 import abi, zcomm

from golden_data import GOLDEN, arrays

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "zcomm_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(zc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = zcomm.lib()
    names = declared_functions()
    assert len(names) >= 60
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_version_and_error_strings():
    L = zcomm.lib()
    assert L.zc_version().decode().startswith("zcomm-b200")
    assert isinstance(L.zc_last_error(), (bytes, type(None)))


def test_defaults_match_reference_structs():
    """ArbitrationConfig{} / TransportHint{} / CollectiveConfig{} (rea.hpp:33-79, collectives.hpp:24-34)."""
    a, b = zcomm.default_arb_config(), abi.default_arb_config()
    assert bytes(a) == bytes(b)
    h = abi.TransportHint()
    zcomm.lib().zc_default_transport_hint(C.byref(h))
    assert (h.regime, h.beta_eff_bytes_per_sec) == (abi.REGIME_INTER, 10.0 * 2**30)
    c = abi.CollectiveConfig()
    zcomm.lib().zc_default_collective_config(C.byref(c))
    assert bytes(c) == bytes(abi.default_collective_config())


# ------------------------------------------------------------------ frame (frame.cpp:35-81)
def test_header_round_trip_matches_port(port):
    """200 random headers (test_frame.cpp:13-34): zc_write_header bytes == the oracle's; parse inverts."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        h = abi.FrameHeader()
        h.magic, h.version = abi.FRAME_MAGIC, abi.FRAME_VERSION
        h.codec = int(rng.integers(0, 3))
        h.flags = abi.FLAG_EMBEDDED_CODEBOOK if (h.codec == 2 and rng.integers(0, 2)) else 0
        h.raw_bytes = int(rng.integers(1, 1 << 40))
        h.payload_bytes = int(rng.integers(1, 1 << 40))
        h.params = int(rng.integers(0, 2**63))
        b = zcomm.write_header(h)
        ob = np.zeros(32, np.uint8)
        port.lib.zo_write_header(C.byref(h), ob)
        assert b == bytes(ob)
        p = zcomm.parse_header(b)
        assert bytes(p) == bytes(h)


def test_parse_needs_full_header():
    """test_frame.cpp:36-39: 31 bytes -> nullopt (ZC_ERR_INVALID_ARGUMENT at the C-ABI)."""
    buf = (C.c_uint8 * 31)()
    h = abi.FrameHeader()
    assert zcomm.lib().zc_parse_header(C.cast(buf, C.c_void_p), 31, C.byref(h)) == abi.ERR_INVALID_ARGUMENT
    assert zcomm.parse_header(bytes(31)) is None
    with pytest.raises(ValueError):
        zcomm.write_header(abi.FrameHeader(), 16)  # write_header throws below 32 B (frame.cpp:36)


def test_validate_rejects_corrupted_fields():
    """test_frame.cpp:41-76."""
    def hdr(codec, raw, pay):
        h = abi.FrameHeader()
        h.magic, h.version, h.codec, h.raw_bytes, h.payload_bytes = abi.FRAME_MAGIC, 1, codec, raw, pay
        return h
    region = 32 + 16
    assert zcomm.validate_header(hdr(1, 64, 16), region)
    bad = hdr(1, 64, 16)
    bad.magic ^= 1
    assert not zcomm.validate_header(bad, region)
    bad = hdr(1, 64, 16)
    bad.version = 2
    assert not zcomm.validate_header(bad, region)
    assert not zcomm.validate_header(hdr(3, 64, 16), region)
    assert not zcomm.validate_header(hdr(1, 0, 16), region)
    assert not zcomm.validate_header(hdr(1, 64, region), region)
    assert zcomm.validate_header(hdr(0, 64, 64), 32 + 64)
    assert not zcomm.validate_header(hdr(0, 64, 32), 32 + 64)


# ------------------------------------------------------------------ selector (rea.cpp:120-176), host build
def test_selector_host_build_matches_reference(port):
    """zc_arbitrate_plan / zc_predict_payload (the same code the device selector runs) against the
    reference's decisions over the golden beta sweep."""
    ctxs = {}
    for e in GOLDEN["known"]["selector"]:
        raw = arrays()[f"raw/{e['case']}"]
        if e["case"] not in ctxs:
            ctxs[e["case"]] = zcomm.HuffmanContext.from_bytes(raw.tobytes())
        ctx = ctxs[e["case"]]
        st = port.profile(raw, port.huff_from_bytes(raw))  # stats (device-computed on the GPU path)
        plan = zcomm.arbitrate_plan(e["raw_bytes"], abi.BATCH_RAW_BYTES, st, abi.make_hint(e["beta"]), ctx)
        assert plan.choice == e["choice"], e
        assert [plan.raw.predicted_payload, plan.fixedlen.predicted_payload, plan.huffman.predicted_payload] == e["pred"]
        assert [plan.raw.predicted_sec, plan.fixedlen.predicted_sec, plan.huffman.predicted_sec] == e["sec"]
        assert [zcomm.predict_payload(c, e["raw_bytes"], st) for c in (0, 1)] == e["pred"][:2]


# ------------------------------------------------------------------ Huffman context (huffman.cpp:23-214), host build
@pytest.mark.parametrize("nm", ["single42", "two_equal", "geometric8", "fibonacci60"] + [f"random{i}" for i in range(6)])
def test_huffman_context_host_build_matches_reference(nm):
    k = GOLDEN["known"][f"huff_{nm}"]
    ctx = zcomm.HuffmanContext.from_hist(k["hist"])
    assert ctx.valid == bool(k["valid"])
    assert ctx.code_lengths == k["lens"]
    code, rev = ctx.codes()
    assert code == k["code"] and rev == k["rev"]
    assert ctx.expected_code_len(k["hist"]) == k["expected_len"]
    assert zcomm.huffman_self_code_len(k["hist"]) == k["expected_len"]  # own tree == own ctx (test_huffman.cpp:100-110)


@pytest.mark.parametrize("name", sorted(GOLDEN["codec"]))
def test_shared_context_from_bytes_matches_reference(name):
    """set_shared_huffman_from_bytes (collectives.cpp:99-106): +1-smoothed histogram of the sample."""
    raw = arrays()[f"raw/{name}"]
    ctx = zcomm.HuffmanContext.from_bytes(raw[: abi.BATCH_RAW_BYTES].tobytes())
    assert ctx.code_lengths == arrays()[f"ctxlens/{name}"].tolist()


def test_invalid_contexts():
    assert not zcomm.HuffmanContext.from_hist([0] * 256).valid  # test_huffman.cpp:90-94
    assert zcomm.huffman_self_code_len([0] * 256) is None
    assert zcomm.HuffmanContext.from_lengths([1, 1, 1] + [0] * 253) is None  # Kraft sum > 1
    assert zcomm.HuffmanContext.from_lengths([40] + [0] * 255) is None       # over the 32-bit cap


# ------------------------------------------------------------------ config (rea.cpp:240-279)
def test_config_parsing():
    """test_rea.cpp:356-380."""
    cfg = zcomm.load_arbitration_config(
        "# comment line\n\nmin_gain_permil = 75   # trailing comment\n  lam_enc=0.5\n"
        "embed_codebook = true\nhuffman_enc_bps = 2e11\n")
    assert cfg.min_gain_permil == 75 and cfg.lam_enc == 0.5 and cfg.embed_codebook == 1
    assert cfg.cost.huffman.enc_bytes_per_sec == 2e11
    for bad in ("vibe = 9\n", "min_gain_permil\n", "embed_codebook = maybe\n"):
        with pytest.raises(ValueError):
            zcomm.load_arbitration_config(bad)
    with pytest.raises(ValueError, match="line 1"):
        zcomm.load_arbitration_config("vibe = 9\n")


def test_env_overrides(monkeypatch):
    """test_rea.cpp:382-398."""
    monkeypatch.setenv("ZCOMM_MIN_GAIN_PERMIL", "120")
    monkeypatch.setenv("ZCOMM_FIXEDLEN_DEC_BPS", "5e10")
    cfg = zcomm.apply_env_overrides(zcomm.default_arb_config())
    assert cfg.min_gain_permil == 120 and cfg.cost.fixedlen.dec_bytes_per_sec == 5e10
    assert cfg.small_batch_threshold_bytes == 4096 and cfg.lam_enc == 0.25


def test_compute_entry_points_fail_loudly_without_device():
    """No CPU fallback: a compute call without a CUDA device returns ZC_ERR_CUDA, never a result."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    n = C.c_int(-1)
    rc = zcomm.lib().zc_device_count(C.byref(n))
    assert rc == abi.ERR_CUDA or n.value == 0
