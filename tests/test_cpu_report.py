"""Report emitters: the reference's 26-column CSV (bench.cpp:551-565) and Markdown
pivot (bench.cpp:620-671) written by paper_2605_12396_b200/report.py, byte-compared with the
compiled reference's own emitters over the same rows."""
import numpy as np
import pytest

import oracle
from paper_2605_12396_b200 import report

REF = oracle.ref()
pytestmark = pytest.mark.skipif(REF is None, reason="oracle/_ref (compiled reference) not built")


def _rows(seed=3, n=24):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        r = report.ReportRow(collective=int(rng.integers(0, 4)), ranks=int(rng.integers(1, 9)),
                             msg_bytes=int(2 ** rng.integers(10, 31)) + int(rng.integers(0, 3)),
                             codec=int(rng.integers(0, 4)), quant=int(rng.integers(0, 3)), dist=int(rng.integers(0, 4)),
                             seed=int(rng.integers(0, 1 << 40)), overlap=int(rng.integers(0, 2)),
                             regime=int(rng.integers(0, 2)))
        r.bw_bytes_per_sec = float(10 ** rng.uniform(8, 12))
        r.latency_sec = float(rng.uniform(0, 1e-4))
        r.sim_time_sec = float(10 ** rng.uniform(-6, 0))
        r.wall_time_sec = float(rng.uniform(0, 2))
        r.wire_raw_bytes = int(rng.integers(0, 1 << 40))
        r.wire_payload_bytes = int(rng.integers(0, 1 << 40))
        r.wire_total_bytes = r.wire_payload_bytes + 32 * int(rng.integers(0, 1000))
        r.frames_raw, r.frames_fixedlen, r.frames_huffman = (int(x) for x in rng.integers(0, 5000, 3))
        r.cr_quant = 1.0
        r.cr_final = float(rng.uniform(0.5, 9))
        r.fill_bandwidths(r.msg_bytes)
        r.speedup_vs_raw = float(rng.uniform(0.1, 4))
        r.exposed_codec_sim_sec = 0.0 if i % 2 else float(rng.uniform(0, 1e-3))
        r.wall_codec_sec = float(rng.uniform(0, 1e-2))
        rows.append(r)
    return rows


def test_csv_header_matches_reference():
    assert REF.emit_csv([]) == report.CSV_HEADER + "\n" == report.emit_csv([])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_csv_bytes_equal_reference(seed):
    rows = _rows(seed)
    assert report.emit_csv(rows) == REF.emit_csv(rows)


@pytest.mark.parametrize("seed", [4, 5])
def test_markdown_bytes_equal_reference(seed):
    rows = _rows(seed)
    assert report.emit_markdown(rows) == REF.emit_markdown(rows)


def test_pretty_bytes_known():
    assert report.pretty_bytes(1 << 20) == "1 MiB"
    assert report.pretty_bytes(3 * (1 << 29)) == "1.5 GiB"
    assert report.pretty_bytes(1000) == "1000 B"


def test_timeline_csv_format():
    """write_timeline_csv (pipeline.cpp:160-170): the reference's header, codec names and
    setprecision(9) times."""
    from paper_2605_12396_b200 import report
    assert report.TIMELINE_HEADER == ("batch,codec,raw_bytes,total_bytes,enc_start_sec,enc_end_sec,"
                                      "xfer_start_sec,xfer_end_sec,dec_start_sec,dec_end_sec")
    row = dict(codec=1, raw_bytes=4194304, total_bytes=1572896, enc_start_sec=1.0 / 3, enc_end_sec=2e-5,
               xfer_start_sec=0.0, xfer_end_sec=1e-9, dec_start_sec=12.5, dec_end_sec=123456789.123)
    lines = report.emit_timeline_csv([row]).splitlines()
    assert lines[1] == "0,fixedlen,4194304,1572896,0.333333333,2e-05,0,1e-09,12.5,123456789"
