"""Run reports in the reference's formats, filled from B200 measurements.

The reference writes one CSV row per experiment (``ReportRow``, bench.hpp:42-69; ``emit_csv``,
bench.cpp:551-565, header bench.cpp:331-337) and a Markdown pivot of compression ratio and speed-up
by message size (``emit_markdown``, bench.cpp:620-671).  This module emits the same 26 columns and
the same Markdown, byte for byte (tests/test_cpu_report.py checks it against the compiled
reference), so sweeps on B200 drop into the reference's tooling.  Column meanings on B200:

* ``sim_time_sec`` — the collective's device time from CUDA events (max over ranks).  The
  reference fills it from its analytic network clock; on B200 the time is measured, not modelled.
* ``wall_time_sec`` — host wall clock around the same calls.
* ``speedup_vs_raw`` — device time of the paired RAW-pinned run / this run (bench.cpp:266-272).
* ``exposed_codec_sim_sec`` / ``wall_codec_sec`` — 0: codec work runs inside the fused step
  kernels, there is no separately timed codec phase to report.
"""
from __future__ import annotations

import dataclasses
from typing import Iterable, List, Sequence

COLLECTIVES = ["allreduce", "allgather", "alltoall", "broadcast"]      # CollOp (collectives.hpp:17)
CODECS = ["auto", "raw", "fixedlen", "huffman"]                        # CodecPin (collectives.hpp:22)
QUANTS = ["none", "eb", "qsgd"]                                        # QuantKind (bench.hpp:14)
DISTS = ["uniform", "gaussian", "geometric", "file"]                   # DataDist (bench.hpp:13)
OVERLAPS = ["pipelined", "serialized"]                                 # OverlapMode (pipeline.hpp:15)
REGIMES = ["intranode", "internode"]                                   # Regime (transport.hpp:25)

CSV_HEADER = ("collective,ranks,msg_bytes,codec,quant,dist,seed,overlap,regime,"
              "bw_bytes_per_sec,latency_sec,sim_time_sec,wall_time_sec,"
              "wire_raw_bytes,wire_payload_bytes,wire_total_bytes,"
              "frames_raw,frames_fixedlen,frames_huffman,cr_quant,cr_final,"
              "alg_bw_bytes_per_sec,bus_bw_bytes_per_sec,speedup_vs_raw,"
              "exposed_codec_sim_sec,wall_codec_sec")


@dataclasses.dataclass
class ReportRow:
    """bench.hpp:42-69, field for field (enums as their index)."""
    collective: int = 0
    ranks: int = 0
    msg_bytes: int = 0
    codec: int = 0
    quant: int = 1
    dist: int = 0
    seed: int = 0
    overlap: int = 0
    regime: int = 1
    bw_bytes_per_sec: float = 0.0
    latency_sec: float = 0.0
    sim_time_sec: float = 0.0
    wall_time_sec: float = 0.0
    wire_raw_bytes: int = 0
    wire_payload_bytes: int = 0
    wire_total_bytes: int = 0
    frames_raw: int = 0
    frames_fixedlen: int = 0
    frames_huffman: int = 0
    cr_quant: float = 1.0
    cr_final: float = 1.0
    alg_bw_bytes_per_sec: float = 0.0
    bus_bw_bytes_per_sec: float = 0.0
    speedup_vs_raw: float = 1.0
    exposed_codec_sim_sec: float = 0.0
    wall_codec_sec: float = 0.0

    def fill_bandwidths(self, size_bytes: int) -> None:
        """algBw / busBw from the time and the collective (bench.cpp:299-320)."""
        t, n = self.sim_time_sec, float(self.ranks)
        if t <= 0.0:
            return
        if self.collective == 0:      # allreduce
            self.alg_bw_bytes_per_sec = size_bytes / t
            self.bus_bw_bytes_per_sec = self.alg_bw_bytes_per_sec * 2.0 * (n - 1.0) / n
        elif self.collective == 1:    # allgather
            self.alg_bw_bytes_per_sec = size_bytes * n / t
            self.bus_bw_bytes_per_sec = self.alg_bw_bytes_per_sec * (n - 1.0) / n
        elif self.collective == 2:    # alltoall
            self.alg_bw_bytes_per_sec = size_bytes / t
            self.bus_bw_bytes_per_sec = self.alg_bw_bytes_per_sec * (n - 1.0) / n
        else:                         # broadcast
            self.alg_bw_bytes_per_sec = size_bytes / t
            self.bus_bw_bytes_per_sec = self.alg_bw_bytes_per_sec

    def fill_wire(self, w) -> None:
        """WireStats -> wire / frame columns and cr_final (bench.cpp:290-297)."""
        self.wire_raw_bytes, self.wire_payload_bytes, self.wire_total_bytes = w.raw_bytes, w.payload_bytes, w.total_bytes
        self.frames_raw, self.frames_fixedlen, self.frames_huffman = (w.frames_by_codec[0], w.frames_by_codec[1],
                                                                      w.frames_by_codec[2])
        self.cr_final = w.raw_bytes / w.payload_bytes if w.payload_bytes > 0 else 1.0

    def flat(self) -> List[float]:
        return [float(getattr(self, f.name)) for f in dataclasses.fields(self)]


def _g(v: float, prec: int) -> str:
    """C++ ostream defaultfloat with setprecision(prec) (= printf %.{prec}g)."""
    return format(float(v), f".{prec}g")


def csv_double(v: float) -> str:
    """bench.cpp:325-329: setprecision(17)."""
    return _g(v, 17)


def pretty_bytes(b: int) -> str:
    """bench.cpp:354-365."""
    suffix = ["B", "KiB", "MiB", "GiB", "TiB"]
    v, s = float(b), 0
    while v >= 1024.0 and s < 4:
        v /= 1024.0
        s += 1
    return f"{_g(v, 4)} {suffix[s]}"


def emit_csv(rows: Iterable[ReportRow]) -> str:
    """bench.cpp:551-565: header line, then one line per row."""
    out = [CSV_HEADER + "\n"]
    for r in rows:
        out.append(",".join([
            COLLECTIVES[r.collective], str(r.ranks), str(r.msg_bytes), CODECS[r.codec], QUANTS[r.quant],
            DISTS[r.dist], str(r.seed), OVERLAPS[r.overlap], REGIMES[r.regime],
            csv_double(r.bw_bytes_per_sec), csv_double(r.latency_sec), csv_double(r.sim_time_sec),
            csv_double(r.wall_time_sec), str(r.wire_raw_bytes), str(r.wire_payload_bytes), str(r.wire_total_bytes),
            str(r.frames_raw), str(r.frames_fixedlen), str(r.frames_huffman), csv_double(r.cr_quant),
            csv_double(r.cr_final), csv_double(r.alg_bw_bytes_per_sec), csv_double(r.bus_bw_bytes_per_sec),
            csv_double(r.speedup_vs_raw), csv_double(r.exposed_codec_sim_sec), csv_double(r.wall_codec_sec),
        ]) + "\n")
    return "".join(out)


def emit_markdown(rows: Sequence[ReportRow]) -> str:
    """bench.cpp:620-671: pivot of CR and speed-up per message size and codec, then every run."""
    sizes: List[int] = []
    codecs: List[int] = []
    for r in rows:
        if r.msg_bytes not in sizes:
            sizes.append(r.msg_bytes)
        if r.codec not in codecs:
            codecs.append(r.codec)

    def find(size, c):
        for r in rows:
            if r.msg_bytes == size and r.codec == c:
                return r
        return None

    out = ["## Compression and speedup by message size\n\n", "| message size |"]
    for c in codecs:
        out.append(f" CR {CODECS[c]} | speedup {CODECS[c]} |")
    out.append("\n|---|")
    out.append("---|---|" * len(codecs))
    out.append("\n")
    for size in sizes:
        out.append(f"| {pretty_bytes(size)} |")
        for c in codecs:
            r = find(size, c)
            if r is None:
                out.append(" - | - |")
                continue
            out.append(f" {r.cr_final:.3f} | {r.speedup_vs_raw:.3f} |")
        out.append("\n")
    out.append("\n## Runs\n\n")
    out.append("| collective | ranks | message size | codec | quant | sim time (s) | CR final | bus BW "
               "(B/s) | speedup |\n")
    out.append("|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        out.append(f"| {COLLECTIVES[r.collective]} | {r.ranks} | {pretty_bytes(r.msg_bytes)} | {CODECS[r.codec]} | "
                   f"{QUANTS[r.quant]} | {_g(r.sim_time_sec, 6)} | {r.cr_final:.3f} | "
                   f"{_g(r.bus_bw_bytes_per_sec, 4)} | {r.speedup_vs_raw:.3f} |\n")
    return "".join(out)


TIMELINE_HEADER = ("batch,codec,raw_bytes,total_bytes,enc_start_sec,enc_end_sec,"
                   "xfer_start_sec,xfer_end_sec,dec_start_sec,dec_end_sec")
CODEC_NAMES = {0: "raw", 1: "fixedlen", 2: "huffman"}                   # codec_name (frame.hpp:20-26)


def emit_timeline_csv(rows: Sequence[dict]) -> str:
    """write_timeline_csv (pipeline.cpp:160-170): header, then one line per batch with the times
    at setprecision(9).  Rows come from Group.timeline() — MEASURED with CUDA events on B200, where
    the reference's rows are its modelled schedule; batch ids number the rows in order."""
    out = [TIMELINE_HEADER + "\n"]
    for i, r in enumerate(rows):
        out.append(",".join([str(i), CODEC_NAMES.get(r["codec"], "raw"), str(r["raw_bytes"]), str(r["total_bytes"])] +
                            [_g(r[k], 9) for k in ("enc_start_sec", "enc_end_sec", "xfer_start_sec", "xfer_end_sec",
                                                   "dec_start_sec", "dec_end_sec")]) + "\n")
    return "".join(out)


def overlap_summary(rows: Sequence[dict]) -> dict:
    """How much of the codec work the pipeline hides: the union of all encode intervals and of all
    decode intervals against the collective's span (first encode start to last decode end)."""
    def union(iv):
        iv = sorted(iv)
        tot, cur = 0.0, None
        for a, b in iv:
            if cur is None or a > cur[1]:
                if cur:
                    tot += cur[1] - cur[0]
                cur = [a, b]
            else:
                cur[1] = max(cur[1], b)
        return tot + (cur[1] - cur[0] if cur else 0.0)
    enc = [(r["enc_start_sec"], r["enc_end_sec"]) for r in rows]
    dec = [(r["dec_start_sec"], r["dec_end_sec"]) for r in rows if r["dec_start_sec"] == r["dec_start_sec"]]
    span = max(b for _, b in enc + dec) - min(a for a, _ in enc + dec)
    busy_e, busy_d = union(enc), union(dec)
    both = union(enc + dec)
    return {"span_sec": span, "encode_busy_sec": busy_e, "decode_busy_sec": busy_d,
            "overlap_sec": busy_e + busy_d - both, "serial_sum_sec": busy_e + busy_d}
