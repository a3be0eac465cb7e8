"""GPU parity against the REFERENCE's own outputs (tests/golden/, generated from the compiled
reference by tests/golden/make_golden.py): the sm_100a path through the C-ABI must reproduce the
reference's frames, payloads, profiles, selector choices and collective results bit-for-bit."""
import numpy as np
import pytest
import torch

from paper_2605_12396_b200 import abi

from golden_data import GOLDEN, arrays, frame_of, ring_input, sha

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]
DEV = "cuda"
HINTS = {"inter10g": abi.make_hint(), "nvlink900g": abi.make_hint(900e9, abi.REGIME_INTRA),
         "thin1g": abi.make_hint(1e9)}
CASES = sorted(GOLDEN["codec"])


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def _ctx(zc, raw):
    return zc.HuffmanContext.from_bytes(raw[: abi.BATCH_RAW_BYTES].tobytes())


@pytest.mark.parametrize("name", CASES)
def test_encode_best_frames_equal_reference(zc, name):
    """zc_encode_best == reference encode_best (rea.cpp:178-238), every hint, with/without ctx."""
    raw = arrays()[f"raw/{name}"]
    ctx = _ctx(zc, raw)
    assert ctx.code_lengths == arrays()[f"ctxlens/{name}"].tolist()
    for key, want in GOLDEN["codec"][name]["frames"].items():
        hname, c = key.split("/")
        r, frame = zc.encode_best(t(raw), hint=HINTS[hname], ctx=ctx if c == "ctx" else None)
        assert (r.codec, r.payload_bytes, r.total_bytes) == (want["codec"], want["payload_bytes"], want["total_bytes"]), key
        assert sha(frame.cpu().numpy()) == want["sha256"], key


@pytest.mark.parametrize("name", CASES)
def test_batched_send_path_equals_reference(zc, name):
    """zc_encode_batches_sym (send_batch, Auto pin -> encode_best) on a one-batch message: the
    persistent task kernel emits the reference's frame; the batched decoder restores the input."""
    raw = arrays()[f"raw/{name}"]
    ctx = _ctx(zc, raw)
    for c in ("noctx", "ctx"):
        fr = zc.encode_batches(t(raw), abi.PIN_AUTO, hint=HINTS["inter10g"], ctx=ctx if c == "ctx" else None)
        assert sha(fr.frame(0).cpu().numpy()) == GOLDEN["codec"][name]["frames"][f"inter10g/{c}"]["sha256"], c
        if len(raw) % 4 == 0:
            back = zc.decode_batches(fr, ctx=ctx)
            assert bytes(back.cpu().numpy().view(np.uint8)[: len(raw)]) == bytes(raw)


@pytest.mark.parametrize("name", CASES)
def test_bare_codecs_equal_reference(zc, name):
    """zc_fixedlen_encode / zc_huffman_encode payloads == fixedlen.cpp:15-37 / huffman.cpp:216-246."""
    g = GOLDEN["codec"][name]
    raw = arrays()[f"raw/{name}"]
    if "fixedlen_width" in g:
        pay, w = zc.fixedlen_encode(t(raw.view(np.int32)), len(raw) + 64)
        assert w == g["fixedlen_width"]
        assert bytes(pay.cpu().numpy()) == bytes(arrays()[f"fixedlen/{name}"])
    out = zc.huffman_encode(t(raw), _ctx(zc, raw), 4 * len(raw) + 512)
    pay = out[0] if isinstance(out, tuple) else out
    assert bytes(pay.cpu().numpy()) == bytes(arrays()[f"huffman/{name}"])


@pytest.mark.parametrize("name", CASES)
def test_device_profile_equals_reference(zc, name):
    """zc_profile_sample (device histogram) == profile_sample (rea.cpp:93-118)."""
    g = GOLDEN["codec"][name]["profile"]
    raw = arrays()[f"raw/{name}"]
    st = zc.profile_sample(t(raw), _ctx(zc, raw))
    assert st.sampled_bytes == g["sampled_bytes"] and st.max_zigzag == g["max_zigzag"]
    assert sha(np.array(st.hist, np.uint64)) == g["hist_sha256"]
    assert st.ctx_code_len_valid == g["ctx_code_len_valid"] and st.ctx_code_len_bits == g["ctx_code_len_bits"]


@pytest.mark.parametrize("n", [2, 3, 4])
@pytest.mark.parametrize("pin", ["auto", "raw", "fixedlen", "huffman"])
def test_ring_allreduce_equals_reference(zc, n, pin):
    """Fused compressed ring RS + AG on one GPU (loopback group of n ranks) == the reference
    Communicator's allreduce: output symbols and summed WireStats."""
    k = GOLDEN["collectives"][f"ring{n}_{pin}"]
    base = ring_input(n)
    g = zc.Group(n, cfg=zc.collective_config(k["pin"]))
    g.set_shared_huffman_from_bytes(base[0].view(np.uint8)[: abi.BATCH_RAW_BYTES].tobytes())
    syms = [t(base[r]) for r in range(n)]
    g.reset_stats()
    g.allreduce(syms, [2e-4] * n)
    for s in syms:
        assert sha(s.cpu().numpy()) == k["out_sha256"]
    w = g.wire_stats()
    assert list(w.frames_by_codec) == k["wire"]["frames_by_codec"]
    assert (w.raw_bytes, w.payload_bytes, w.total_bytes) == (k["wire"]["raw_bytes"], k["wire"]["payload_bytes"],
                                                              k["wire"]["total_bytes"])
    g.close()


@pytest.mark.parametrize("n", [2, 3, 4])
def test_ring_allgather_equals_reference(zc, n):
    k = GOLDEN["collectives"][f"allgather{n}"]
    blk = ring_input(n)[:, : k["block"]]
    g = zc.Group(n)
    g.reset_stats()
    outs = g.allgather([t(blk[r]) for r in range(n)])
    for o in outs:
        assert sha(o.cpu().numpy()) == k["out_sha256"]
    w = g.wire_stats()
    assert list(w.frames_by_codec) == k["wire"]["frames_by_codec"] and w.payload_bytes == k["wire"]["payload_bytes"]
    g.close()


def test_hand_vectors(zc):
    """test_collectives.cpp:83-118 through the group C-ABI."""
    for nm in ("symsum4", "reconcile2"):
        k = GOLDEN["collectives"][nm]
        g = zc.Group(len(k["in"]))
        syms = [t(np.array(s, np.int32)) for s in k["in"]]
        assert g.allreduce(syms, k["scales_in"]) == k["scales_out"]
        assert [s.cpu().numpy().tolist() for s in syms] == k["out"]
        g.close()
