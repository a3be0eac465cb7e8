#!/usr/bin/env python
"""Benchmark of the B200 compressed-collectives hot path.

N=1 (default): BASELINE config 0 — single-rank codec round trip on 64 Mi synthetic Gaussian fp32
elements, absolute error bound 1e-4 (bin width 2e-4): fused quantize + 64 KiB histogram + selector
+ encode into 4 MiB-batch frames, then decode + dequantize back to fp32.  One step = one round
trip over the whole array.  value = codec GB/s over raw symbol bytes (4 B/element, the
codec_bench.cpp:49 convention) per round trip.  The selector runs with the reference's default
inter-node hint (10 GiB/s, transport.hpp:33-35), so it picks FixedLen on Gaussian data; the
Huffman-pinned round trip of the same config is reported beside it.

N>1 (torchrun): compressed ring AllReduce (allreduce_eb) of BASELINE config 1 (N=2: 256 MB
Laplacian per rank, abs eb 1e-4) or config 2 (N=4/8: 512^3 smooth field per rank, rel 1e-3);
value = algbw = bytes per rank / time (the max over ranks).

--impl reference: the reference's own CPU implementation of the same round trip (oracle/_ref,
compiled from /root/reference sources) on all host cores, over a bounded sample per step.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

COUNT_C0 = 64 << 20          # config 0: 64 Mi fp32 elements
ABS_EB = 1e-4
SCALE = 2 * ABS_EB           # eb_quantize_with_scale bin width for an absolute bound
BETA = 10.0 * 1073741824.0   # reference default hint (inter-node, 10 GiB/s)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def load_traffic(kernel):
    """dram read+write bytes per launch from the committed ncu capture (profiles/ncu_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d.get(kernel)
    except Exception:
        return None


# ------------------------------------------------------------------------------- synthetic inputs
# Both arms (ours and --impl reference) build their inputs with these host generators, so the two
# JSON lines describe the same data and the same config.
DATA_C0 = "synthetic: numpy default_rng(1).standard_normal fp32 (BASELINE config 0 Gaussian)"
DATA_C1 = "synthetic: Laplacian(0, 1e-2) fp32 per rank, numpy default_rng(100 + rank)"
DATA_C2 = ("synthetic: 512^3 smooth field per rank, sin(2 pi i/512 + 0.37 r) cos(4 pi j/512) + "
           "0.5 sin(6 pi k/512 + 0.37 r), fp32")


def gen_c0(count):
    import numpy as np
    return np.random.default_rng(1).standard_normal(count, dtype=np.float32)


def gen_rank(world, rank, count):
    """Per-rank input of the N>1 workloads: config 1 (N=2) Laplacian gradients, config 2 (N>=4)
    the smooth scientific field (first `count` elements of the 512^3 field)."""
    import numpy as np
    if world == 2:
        return np.random.default_rng(100 + rank).laplace(0.0, 1e-2, count).astype(np.float32)
    n = 512
    slabs = min(n, -(-count // (n * n)))
    out = np.empty(slabs * n * n, np.float32)
    i = np.arange(n, dtype=np.float64)
    ph = 0.37 * rank
    a = np.sin(2 * np.pi * i / n + ph)[:, None] * np.cos(4 * np.pi * i / n)[None, :]   # (i, j)
    b = 0.5 * np.sin(6 * np.pi * i / n + ph)                                             # (k)
    for ii in range(slabs):
        out[ii * n * n:(ii + 1) * n * n] = (a[ii][:, None] + b[None, :]).astype(np.float32).ravel()
    return out[:count]


def workload_config(world, count):
    """The config dict both arms print (identical keys and values)."""
    if world == 1:
        return {"workload": "BASELINE config 0: single-rank codec round trip, 64 Mi Gaussian fp32, abs eb 1e-4",
                "count": count, "raw_bytes": 4 * count, "scale": SCALE, "pin": "auto (encode_best)",
                "hint_beta_bytes_per_sec": BETA, "batches": (4 * count + (4 << 20) - 1) // (4 << 20),
                "batch_bytes": 4 << 20}
    if world == 2:
        wl, q = "BASELINE config 1: ring AllReduce, 256 MB Laplacian per rank, abs eb 1e-4", "abs eb 1e-4"
    else:
        wl, q = "BASELINE config 2: ring RS+AG (allreduce_eb), 512^3 smooth field per rank, rel eb 1e-3", "rel eb 1e-3"
    return {"workload": wl, "count_per_rank": count, "quantizer": q, "pin": "auto (encode_best)",
            "hint_beta_bytes_per_sec": BETA, "shared_huffman": "primed from rank 0's first 1 Mi symbols (bench.cpp:169-204)",
            "parallelism": f"ring{world}"}


def world_count(world, count_arg):
    if count_arg:
        return count_arg
    return COUNT_C0 if world <= 2 else 512 * 512 * 512


def eb_rel(world, xs_absmax):
    """allreduce_eb's rel: config 1 fixes the absolute bound 1e-4 (scale 2e-4 = 2 rel gmax)."""
    return ABS_EB / xs_absmax if world == 2 else 1e-3


# ---------------------------------------------------------------------------------------- N = 1
def codec_bench(args):
    import torch
    from paper_2605_12396_b200 import abi, zcomm

    L = zcomm.lib()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    count = args.count
    raw_bytes = 4 * count
    x = torch.from_numpy(gen_c0(count)).to(dev)
    hint = abi.make_hint(BETA)
    cfg = zcomm.default_arb_config()
    # shared Huffman context primed like prime_shared_huffman (bench.cpp:169-204): rank 0's first
    # <= 1 Mi symbols under the run's scale, +1 smoothing
    prime = zcomm.eb_quantize_with_scale(x[: 1 << 20], SCALE)
    ctx = zcomm.HuffmanContext.from_bytes(prime)
    fr = zcomm.alloc_frames(raw_bytes, dev)
    out = torch.empty(count, dtype=torch.float32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    codecs = torch.zeros(fr.nbatches, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    s = C.c_void_p(stream.cuda_stream)
    P = zcomm._ptr

    def encode(pin, st=s):
        zcomm.check(L.zc_encode_batches_f32(P(x), count, SCALE, P(fr.stages), zcomm.STAGE_STRIDE,
                                            abi.STAGE_BANK_BYTES, pin, C.byref(hint), ctx.handle, C.byref(cfg),
                                            P(fr.results), P(fr.index), P(err), st))

    def decode(dst, st=s):
        zcomm.check(L.zc_decode_batches_f32(P(fr.stages), zcomm.STAGE_STRIDE, abi.STAGE_BANK_BYTES,
                                            P(fr.results), count, SCALE, ctx.handle, P(fr.index), P(dst),
                                            P(codecs), st))

    def graph_run(pin, steps, warmup, parts=("enc", "dec")):
        """The same step (encode call + decode call, every kernel and the scratch memset) captured
        once as a CUDA graph and replayed: the launch path B200 deployments use for a fixed-shape
        step.  Returns ms per step (CUDA events around `steps` replays) or None if capture fails."""
        try:
            side = torch.cuda.Stream()
            ss = C.c_void_p(side.cuda_stream)
            with torch.cuda.stream(side):
                for _ in range(max(1, warmup)):  # per-stream scratch exists before capture
                    encode(pin, ss)
                    decode(out, ss)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                if "enc" in parts:
                    encode(pin, ss)
                if "dec" in parts:
                    decode(out, ss)
            for _ in range(warmup):
                g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(steps):
                g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            if int(err.item()):
                raise RuntimeError(f"device error word 0x{int(err.item()):x}")
            return a.elapsed_time(b) / steps
        except Exception as e:  # noqa: BLE001
            print(f"bench: CUDA graph capture unavailable ({e}); eager timing reported", file=sys.stderr)
            return None

    def run(pin, steps, warmup, with_clocks=False):
        for _ in range(warmup):
            encode(pin)
            decode(out)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
               torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = Clocks(0)
        if with_clocks:
            clk.__enter__()
            time.sleep(0.3)
        torch.cuda.synchronize()
        n0 = zcomm.launch_count()
        start.record(stream)
        for i in range(steps):
            ev[i][0].record(stream)
            encode(pin)
            ev[i][1].record(stream)
            decode(out)
            ev[i][2].record(stream)
        end.record(stream)
        launches = zcomm.launch_count() - n0
        torch.cuda.synchronize()
        if with_clocks:
            clk.__exit__()
        total = start.elapsed_time(end) / steps
        enc = statistics.mean(a.elapsed_time(b) for a, b, _ in ev)
        dec = statistics.mean(b.elapsed_time(c) for _, b, c in ev)
        res = fr.encode_results()
        payload = sum(r.payload_bytes for r in res)
        frames = [0, 0, 0]
        for r in res:
            frames[r.codec] += 1
        e = int(err.item())
        if e:
            raise RuntimeError(f"device error word 0x{e:x}")
        return {"ms": total, "enc_ms": enc, "dec_ms": dec, "payload": payload, "frames": frames,
                "clocks": clk.summary() if with_clocks else None, "launches": launches}

    auto = run(abi.PIN_AUTO, args.steps, args.warmup, with_clocks=True)
    # correctness guard on the measured output: the eb bound plus the one fp32 rounding of the output
    y = out
    maxerr = float((y.double() - x.double()).abs().max().item())
    bound = ABS_EB * (1 + 1e-9) + float(x.abs().max().item()) * 2.0 ** -24
    if not maxerr <= bound:
        raise RuntimeError(f"round trip exceeds the error bound: {maxerr} > {bound}")
    huff = run(abi.PIN_HUFFMAN, max(3, args.steps // 2), args.warmup)
    graph_ms = graph_run(abi.PIN_AUTO, args.steps, args.warmup)
    graph_enc_ms = graph_run(abi.PIN_AUTO, args.steps, args.warmup, ("enc",)) if graph_ms is not None else None
    graph_dec_ms = graph_run(abi.PIN_AUTO, args.steps, args.warmup, ("dec",)) if graph_ms is not None else None
    if graph_ms is not None:
        yg = out.clone()
        encode(abi.PIN_AUTO)
        decode(out)
        torch.cuda.synchronize()
        if not torch.equal(yg, out):
            raise RuntimeError("graph-replayed round trip differs from the eager one")

    # e2e: the public C-ABI host-buffer call (zc_codec_roundtrip_host_f32: pinned host fp32 in ->
    # frames -> pinned host fp32 out), H2D / kernels / D2H pipelined over 8 MiB groups inside the
    # library; every byte of input and output crosses PCIe inside the timed region
    hx = torch.empty(count, dtype=torch.float32, pin_memory=True)
    hx.copy_(x.cpu())
    hy = torch.empty(count, dtype=torch.float32, pin_memory=True)
    work = torch.empty_like(x)

    def e2e_step():
        zcomm.check(L.zc_codec_roundtrip_host_f32(hx.data_ptr(), count, SCALE, P(work), P(fr.stages),
                                                  zcomm.STAGE_STRIDE, abi.STAGE_BANK_BYTES, abi.PIN_AUTO,
                                                  C.byref(hint), ctx.handle, C.byref(cfg), P(fr.results),
                                                  P(fr.index), P(err), hy.data_ptr(), 8, s))

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = t0.elapsed_time(t1) / args.steps
    if int(err.item()):
        raise RuntimeError(f"device error word 0x{int(err.item()):x} in the e2e run")
    if not torch.equal(hy, y.cpu()):
        raise RuntimeError("e2e output differs from the device-resident run")

    loop = loopback_allreduce(args) if not args.no_loopback else None

    peak, peak_kind = peaks()
    gbs = lambda ms: raw_bytes / (ms * 1e-3) / 1e9  # noqa: E731
    step_ms = graph_ms if graph_ms is not None else auto["ms"]
    P_auto, F = auto["payload"], fr.nbatches
    enc_bytes = 4 * count + P_auto + 32 * F     # fp32 read + frames written
    dec_bytes = P_auto + 32 * F + 4 * count     # frames read + fp32 written
    enc_ms = graph_enc_ms if graph_enc_ms is not None else auto["enc_ms"]
    dec_ms = graph_dec_ms if graph_dec_ms is not None else auto["dec_ms"]
    dom = "encode" if enc_ms >= dec_ms else "decode"
    dom_ms = max(enc_ms, dec_ms)
    dom_bytes = enc_bytes if dom == "encode" else dec_bytes
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = load_traffic("zc_encode_f32" if dom == "encode" else "zc_decode")
    line = {
        "metric": "codec GB/s (quantize+histogram+select+encode+decode+dequantize round trip, raw symbol bytes)",
        "value": round(gbs(step_ms), 2),
        "unit": "GB/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(step_ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32->int32 (fp64 quantizer arithmetic)",
        "data": DATA_C0,
        "config": workload_config(1, count),
        "l2": "inputs (256 MiB fp32) exceed the 126 MB L2; no flush needed",
        "launch": "cuda_graph (one captured step replayed)" if graph_ms is not None else "eager",
        "eager_ms_per_step": round(auto["ms"], 4),
        "compression_ratio": round(raw_bytes / P_auto, 4),
        "frames_by_codec": {"raw": auto["frames"][0], "fixedlen": auto["frames"][1], "huffman": auto["frames"][2]},
        "encode_ms": round(enc_ms, 4), "decode_ms": round(dec_ms, 4),
        "encode_gbs": round(gbs(enc_ms), 2), "decode_gbs": round(gbs(dec_ms), 2),
        "huffman_pinned": {
            "value": round(gbs(huff["ms"]), 2), "unit": "GB/s", "ms_per_step": round(huff["ms"], 4),
            "compression_ratio": round(raw_bytes / huff["payload"], 4),
            "encode_gbs": round(gbs(huff["enc_ms"]), 2), "decode_gbs": round(gbs(huff["dec_ms"]), 2),
            "frames_by_codec": {"raw": huff["frames"][0], "fixedlen": huff["frames"][1], "huffman": huff["frames"][2]},
        },
        "roofline": {
            "bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
            "algorithmic_bytes_per_launch": dom_bytes,
            "roundtrip_frac": round((enc_bytes + dec_bytes) / (step_ms * 1e-3) / 1e9 / peak, 4),
        },
        "e2e": {"value": round(gbs(e2e_ms), 2), "unit": "GB/s", "ms_per_step": round(e2e_ms, 3),
                "h2d_bytes_per_step": 4 * count, "d2h_bytes_per_step": 4 * count},
        "gpu_launches": auto["launches"],
        "clocks": auto["clocks"],
    }
    if loop is not None:
        line["collective_loopback"] = loop
    if not args.no_cpu_baseline:
        # the reference on all host cores over the SAME 64 Mi workload, repeated so the timed CPU work
        # is ~10+ core-seconds; value = mean throughput of the repetitions
        line["cpu_baseline"] = cpu_baseline(x[: args.cpu_sample].cpu().numpy(), prime.cpu().numpy(), 0,
                                            reps=args.cpu_reps)
    return line


def loopback_allreduce(args):
    """BASELINE config 1's compressed AllReduce (2 ranks x 64 Mi Laplacian fp32, abs eb 1e-4) as a
    loopback group on this one GPU: both ranks' ring kernels share cuda:0, frames move through
    device memory instead of NVLink.  Device-timed with CUDA events; context, not the headline."""
    import torch
    from paper_2605_12396_b200 import zcomm
    n, count = 2, COUNT_C0
    xs = []
    for r in range(n):
        g = torch.Generator(device="cuda")
        g.manual_seed(100 + r)
        u = torch.rand(count, generator=g, device="cuda", dtype=torch.float64) - 0.5
        xs.append((-1e-2 * torch.sign(u) * torch.log1p(-2 * u.abs())).float())
        del u
    grp = zcomm.Group(n)
    rel = ABS_EB / max(float(x.abs().max().item()) for x in xs)
    outs = [torch.empty_like(x) for x in xs]
    for _ in range(args.warmup):
        grp.allreduce_eb(xs, rel, outs=outs)
    torch.cuda.synchronize()
    grp.reset_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = max(3, args.steps // 2)
    a.record()
    for _ in range(steps):
        grp.allreduce_eb(xs, rel, outs=outs)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    exact = xs[0].double() + xs[1].double()
    err = float((outs[0].double() - exact).abs().max().item())
    bound = n * ABS_EB * (1 + 1e-9) + float(exact.abs().max().item()) * 2.0 ** -24
    if not err <= bound:
        raise RuntimeError(f"loopback allreduce exceeds the error bound: {err} > {bound}")
    w = grp.wire_stats()
    grp.close()
    return {"workload": "BASELINE config 1 on one GPU: 2-rank loopback group, 64 Mi Laplacian fp32 per rank, abs eb 1e-4",
            "ms_per_step": round(ms, 3), "algbw_gbs": round(4 * count / (ms * 1e-3) / 1e9, 2),
            "compression_ratio": round(w.raw_bytes / max(w.payload_bytes, 1), 4), "max_abs_err": err,
            "note": "both ranks share one B200's HBM and SMs; not an NVLink number"}


# ------------------------------------------------------------------------- CPU baseline / reference
def cpu_baseline(xs, prime_syms, pin, threads=None, reps=1):
    """The reference's codec round trip (oracle/_ref: encode_best / send_batch + decode dispatch +
    dequantize per 4 MiB batch, bench-style) on a thread pool over the host cores."""
    import numpy as np
    import oracle
    from paper_2605_12396_b200 import abi
    ref = oracle.ref()
    kind = "reference"
    if ref is None:
        raise RuntimeError("oracle/_ref is not built; the CPU baseline needs the compiled reference")
    threads = threads or os.cpu_count()
    x = np.ascontiguousarray(xs, np.float32)
    ctx = ref.huff_from_bytes(np.ascontiguousarray(prime_syms).view(np.uint8))
    cfg = abi.default_arb_config()
    pay = C.c_uint64()
    frames = np.zeros(3, np.uint64)
    wall = C.c_double()
    total = 0.0
    for _ in range(reps):
        rc = ref.lib.zr_codec_roundtrip_mt(x, len(x), SCALE, pin, ctx, C.byref(cfg), abi.REGIME_INTER, BETA, threads,
                                           None, C.byref(pay), frames, C.byref(wall))
        if rc:
            raise RuntimeError(ref.error())
        total += wall.value
    ref.lib.zr_huff_ctx_free(ctx)
    return {"value": round(reps * 4 * len(x) / total / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"{reps} x {len(x)} fp32 elements ({len(x) * 4 >> 20} MiB, {int(frames.sum())} batches each) "
                      f"of the same workload, {'auto' if pin == 0 else 'pinned'} codec, compiled reference "
                      f"(oracle/_ref) on a {threads}-thread pool",
            "compression_ratio": round(4 * len(x) / max(pay.value, 1), 4), "seconds": round(total, 3),
            "core_seconds": round(total * threads, 1)}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    if world > 1:
        return reference_collective_arm(args, world)
    n = args.cpu_sample
    x = gen_c0(n)
    prime = np.clip(np.round(x[: 1 << 20].astype(np.float64) / SCALE), -2**31, 2**31 - 1).astype(np.int32)
    for _ in range(args.warmup):
        cpu_baseline(x[: min(n, 4 << 20)], prime, 0)
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(x, prime, 0))
    t_all = time.perf_counter() - t_all
    v = statistics.mean(r["value"] for r in vals)
    cb = dict(vals[-1])
    cb["value"] = round(v, 3)
    return {
        "metric": "codec GB/s (quantize+histogram+select+encode+decode+dequantize round trip, raw symbol bytes)",
        "value": round(v, 3), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t_all / args.steps, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32->int32 (fp64 quantizer arithmetic)",
        "data": DATA_C0, "impl": "reference",
        "config": workload_config(1, n),
        "cpu_baseline": cb,
        "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


_XS_CACHE = {}


def collective_cpu_baseline(world, count, sample_count, reps=1):
    """The reference's own collective runtime: Communicator(world, cfg).run with one host thread per
    rank, each calling RankCtx::allreduce_eb on its rank's input (bench.cpp:206-289 times
    Communicator::run by wall clock).  Shared Huffman context primed like prime_shared_huffman.
    Bounded sample: the first `sample_count` elements of every rank's input."""
    import oracle
    from paper_2605_12396_b200 import abi
    ref = oracle.ref()
    if ref is None:
        raise RuntimeError("oracle/_ref is not built; the CPU baseline needs the compiled reference")
    m = min(count, sample_count)
    key = (world, m)
    if key not in _XS_CACHE:
        _XS_CACHE.clear()
        _XS_CACHE[key] = np.stack([gen_rank(world, r, m) for r in range(world)]).astype(np.float64)
    xs = _XS_CACHE[key]
    gmax = float(np.abs(xs).max())
    rel = eb_rel(world, gmax)
    scale = 2.0 * rel * gmax
    prime = np.clip(np.round(xs[0, : 1 << 20] / scale), -2**31, 2**31 - 1).astype(np.int32).view(np.uint8)
    cfg = abi.default_collective_config(abi.PIN_AUTO)
    cfg.hint = abi.make_hint(BETA)
    out = np.zeros_like(xs)
    w = abi.WireStats()
    wall = C.c_double()
    total = 0.0
    for _ in range(reps):
        rc = ref.lib.zr_allreduce_eb(world, C.byref(cfg), np.ascontiguousarray(xs).ravel(), m, rel, prime.ctypes.data, len(prime),
                                     out.ravel(), C.byref(w), C.byref(wall))
        if rc:
            raise RuntimeError(ref.error())
        total += wall.value
    return {"value": round(reps * 4 * m / total / 1e9, 4), "unit": "GB/s", "cores": world, "kind": "reference",
            "sample": f"{reps} x allreduce_eb of {m} fp32 elements per rank ({4 * m >> 20} MiB; the first {m} of the "
                      f"{count}-element workload), {world} rank threads of the compiled reference's Communicator::run",
            "compression_ratio": round(w.raw_bytes / max(w.payload_bytes, 1), 4), "seconds": round(total, 3)}


def reference_collective_arm(args, world):
    count = world_count(world, args.count)
    for _ in range(max(0, min(args.warmup, 1))):
        collective_cpu_baseline(world, count, min(args.ref_sample, 1 << 20))
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        vals.append(collective_cpu_baseline(world, count, args.ref_sample))
    t_all = time.perf_counter() - t_all
    v = statistics.mean(r["value"] for r in vals)
    cb = dict(vals[-1])
    cb["value"] = round(v, 4)
    return {
        "metric": "compressed AllReduce algbw GB/s", "value": round(v, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_all / args.steps, 2),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32->int32 symbols (int32 sum)",
        "data": DATA_C1 if world == 2 else DATA_C2, "impl": "reference",
        "config": workload_config(world, count), "cpu_baseline": cb,
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


# ---------------------------------------------------------------------------------------- N > 1
def max_over_ranks(v: float) -> float:
    """Max of a per-rank scalar over the job (torch.distributed must be initialised)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v)], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_bench(args):
    """Compressed ring AllReduce (allreduce_eb: quantize -> fused compressed RS -> AG -> dequantize),
    one process per GPU; device-timed with CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2605_12396_b200 import zcomm

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ndev = torch.cuda.device_count()
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    use_nccl = ndev >= world and os.environ.get("ZC_BENCH_GLOO") is None
    dist.init_process_group("nccl" if use_nccl else "gloo",
                            **({"device_id": torch.device("cuda", dev_index)} if use_nccl else {}))
    dev = torch.device("cuda", dev_index)
    count = world_count(world, args.count)
    xh = gen_rank(world, rank, count)
    x = torch.from_numpy(xh).to(dev)
    comm = zcomm.Communicator(rank, world, dev_index)
    gmax = max_over_ranks(float(np.abs(xh).max()))
    rel = eb_rel(world, gmax)
    # shared Huffman context primed like prime_shared_huffman (bench.cpp:169-204): rank 0's first
    # 1 Mi symbols at the run's global scale, broadcast so every rank holds the same table
    prime = torch.zeros(1 << 20, dtype=torch.int32)
    if rank == 0:
        prime = torch.from_numpy(np.clip(np.round(xh[: 1 << 20].astype(np.float64) / (2.0 * rel * gmax)),
                                         -2**31, 2**31 - 1).astype(np.int32))
    pt = prime.to(dev) if dist.get_backend() == "nccl" else prime
    dist.broadcast(pt, 0)
    comm.set_shared_huffman_from_bytes(pt.cpu().numpy().tobytes())
    out = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        comm.allreduce_eb(x, rel, out)
    torch.cuda.synchronize()
    zcomm.lib().zc_comm_reset_stats(comm._h)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    n0 = zcomm.launch_count()
    clk = Clocks(dev_index)
    with clk:
        time.sleep(0.2)
        t0.record(stream)
        for _ in range(args.steps):
            comm.allreduce_eb(x, rel, out)
        t1.record(stream)
        torch.cuda.synchronize()
    launches = zcomm.launch_count() - n0
    dist.barrier()
    dt = max_over_ranks(t0.elapsed_time(t1) / 1e3 / args.steps)
    w = comm.wire_stats()

    # e2e through the public API: pinned host input -> device -> allreduce_eb -> pinned host output
    hx = torch.empty(count, dtype=torch.float32, pin_memory=True)
    hx.copy_(x.cpu())
    hy = torch.empty(count, dtype=torch.float32, pin_memory=True)
    dx = torch.empty_like(x)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        dx.copy_(hx, non_blocking=True)
        comm.allreduce_eb(dx, rel, out)
        hy.copy_(out, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    dt_e2e = max_over_ranks(e0.elapsed_time(e1) / 1e3 / args.steps)

    # context: plain uncompressed NCCL AllReduce of the same fp32 buffer
    nccl_algbw = None
    if use_nccl:
        y = x.clone()
        for _ in range(3):
            dist.all_reduce(y)
        torch.cuda.synchronize()
        dist.barrier()
        n0e, n1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0e.record(stream)
        for _ in range(args.steps):
            dist.all_reduce(y)
        n1e.record(stream)
        torch.cuda.synchronize()
        nccl_algbw = round(4 * count / max_over_ranks(n0e.elapsed_time(n1e) / 1e3 / args.steps) / 1e9, 2)
        del y

    line = None
    if rank == 0:
        S = 4 * count
        cr = w.raw_bytes / max(w.payload_bytes, 1)
        algbw = S / dt / 1e9
        per_gpu_sent = w.total_bytes / max(args.steps, 1)  # this rank's frames (wire stats are per rank)
        line = {
            "metric": "compressed AllReduce algbw GB/s", "value": round(algbw, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32->int32 symbols (int32 sum)",
            "data": "synthetic (generated on device)",
            "config": {"workload": workload, "count_per_rank": count, "pin": "auto",
                       "hint_beta_bytes_per_sec": BETA, "parallelism": f"ring{world}",
                       "l2": "per-rank input exceeds L2"},
            "compression_ratio": round(cr, 4), "busbw": round(algbw * 2 * (world - 1) / world, 2),
            "frames_by_codec": list(w.frames_by_codec),
            "roofline": {"bound": "nvlink", "achieved": round(per_gpu_sent / dt / 1e9, 2), "peak": 900.0,
                         "unit": "GB/s", "frac": round(per_gpu_sent / dt / 1e9 / 900.0, 4), "traffic": None},
            "nccl_uncompressed_algbw": nccl_algbw,
            "e2e": {"value": round(S / dt_e2e / 1e9, 2), "unit": "GB/s", "ms_per_step": round(dt_e2e * 1e3, 3),
                    "h2d_bytes_per_step": S, "d2h_bytes_per_step": S},
            "gpu_launches": launches, "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = collective_cpu_baseline(world, count, args.ref_sample)
    comm.close()
    dist.destroy_process_group()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--count", type=int, default=0)
    ap.add_argument("--cpu-sample", type=int, default=COUNT_C0)
    ap.add_argument("--cpu-reps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-loopback", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=16 << 20,
                    help="elements per rank of the collective CPU baseline's bounded sample")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torchrun (what the driver does itself)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        line = reference_arm(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1:
        line = allreduce_bench(args)
    else:
        args.count = args.count or COUNT_C0
        line = codec_bench(args)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
