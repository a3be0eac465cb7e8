"""Loader for the golden fixtures in tests/golden/ (generated from the compiled reference by
tests/golden/make_golden.py).  Test infrastructure only; no reference files are read at run time."""
import functools
import hashlib
import json
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(GOLDEN_DIR, "golden.json")) as _f:
    GOLDEN = json.load(_f)

RING_COUNT = 1_500_001  # 6 MiB per rank: > fused_codec_min_msg_bytes, ragged chunks and batches


@functools.lru_cache(maxsize=1)
def arrays() -> dict:
    with np.load(os.path.join(GOLDEN_DIR, "codec.npz")) as z:
        return {k: z[k] for k in z.files}


def sha(b) -> str:
    return hashlib.sha256(np.ascontiguousarray(b).view(np.uint8).tobytes()).hexdigest()


def frame_of(case: str, key: str) -> np.ndarray:
    """The reference's encode_best frame for `case` under `key` ("<hint>/<ctx|noctx>")."""
    return arrays()["frame/" + GOLDEN["codec"][case]["frames"][key]["sha256"]]


def ring_input(n: int, count: int = RING_COUNT) -> np.ndarray:
    """Per-rank int32 symbols for the ring fixtures (numpy PCG64, fixed seed per n)."""
    rng = np.random.default_rng(7 + n)
    mag = rng.geometric(0.02, (n, count)).astype(np.int32)
    return mag * rng.choice(np.array([-1, 1], np.int32), (n, count))
