#!/usr/bin/env python
"""bench.py — throughput of the arXiv 2212.00404 hot path on B200.

Headline workload ("configs4-sweep", BASELINE.json configs[4]; SURVEY.md
§8(d)-(e)): the multi-channel layer 14x14, C = 512, M = 4096, K = 3 (Eq. 1,
PAPER.md P:92-98) in its three variants FP32 (KM-SIMT), TF32 and BF16
(tcgen05).  One step = that layer once per precision.  Metric: GFLOP/s
(direct-conv count 2*M*C*K*K*Ho*Wo summed over the step).

Multi-GPU (torchrun, one rank per GPU): the filters are sharded by index m
(Fig. 2(c), lifted from SMs to GPUs).  Rank r computes
O[r*M/N : (r+1)*M/N] from its contiguous F slice; I is broadcast once at setup
(NCCL).  Total work is fixed as N grows ("scaling": "strong"); the headline is
the units of all ranks / the max-over-ranks device time, so the driver's per-N
values give T_1 / max_r T_N directly.  The path's only
collective, the all-gather of O, is timed separately (`allgather_us`); at
N > 1 rank 0 also times the full-M layer alone (`t1_us`) in the same run.

Timing: W warm-up steps, then EXACTLY K steps between a barrier + synchronize
on both sides; device time from CUDA events on the launching stream; max over
ranks.  A step is one CUDA graph (the three precision calls, 6 kernels,
PDL-chained).  Each kernel's share of the step is what the step loses without
it (full-step graph vs step-minus-precision graphs, replayed interleaved right
after the timed region), scaled to the timed region.  Two buffer sets
(F, O) alternate between steps: 2 x (75.5 + 75.5 + 37.7) MB of filters pass
through between re-reads of a set, > 3x the 126 MB L2 ("inputs larger than
L2").  NVML samples SM clocks and throttle reasons every ~1 ms during the
timed region.

Secondary results (earlier stdout lines + gpurun_out/bench_detail_n<N>.json;
the LAST stdout line is the compact headline): the 104-call layer suite of
configs[1..4] (+ the 28x28x256 target layer) with per-precision values
(`suite`), per-layer back-to-back latencies, cuDNN on the same shapes, batched
/ padded / strided calls, cold (L2-flushed) call times, the empty-kernel
launch floor.

`--impl reference` times the CPU oracle (oracle/, fp64 C) on a bounded sample
of the same workload on the host cores; it never imports the product package.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "GFLOP/s & % of HBM/tensor-pipe roofline per layer at 1/2/4/8 B200 vs cuDNN"
UNIT = "GFLOP/s"
WORKLOAD = "configs4-sweep"
PRECS = ("fp32", "tf32", "bf16")
FP32_LANES_PER_SM = 128
L2_BYTES = 126 * 2 ** 20


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "sm_max_mhz": float(p.get("sm_max_mhz", 1965.0)), "source": "MEASURED_PEAKS.json"}
    except Exception:
        # B200_PROFILING.md fallback figures
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0, "source": "B200_PROFILING.md fallback"}


def fp32_peak_tflops(pk, sms):
    """FP32 FMA pipe: SMs x 128 lanes x 2 FLOP x max SM clock."""
    return sms * FP32_LANES_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12


def layer_geom(c):
    c = dict(c)
    c["Ho"], c["Wo"] = c["Wy"] - c["K"] + 1, c["Wx"] - c["K"] + 1
    c["flop"] = 2.0 * c["M"] * c["C"] * c["K"] ** 2 * c["Ho"] * c["Wo"]
    return c


def bytes_alg(c, prec):
    """e_in*(C*Wx*Wy + M*C*K^2) + 4*M*Ho*Wo, each tensor once."""
    e = 2 if prec == "bf16" else 4
    return e * (c["C"] * c["Wx"] * c["Wy"] + c["M"] * c["C"] * c["K"] ** 2) + 4 * c["M"] * c["Ho"] * c["Wo"]


def roof(c, prec, kernel, pk, sms):
    """(bound, peak, unit, algorithmic amount in peak units x s) of one call."""
    by = bytes_alg(c, prec)
    t_hbm = by / (pk["hbm_gbs"] * 1e9)
    if kernel.startswith("KS") or prec == "fp32":
        pf = fp32_peak_tflops(pk, sms)
        if kernel.startswith("KS") and t_hbm >= c["flop"] / (pf * 1e12):
            return "hbm", pk["hbm_gbs"], "GB/s", by / 1e9
        return "alu", pf, "TFLOP/s", c["flop"] / 1e12
    tc = pk["bf16_tflops"] * (0.5 if prec == "tf32" else 1.0)        # tf32 = bf16/2 (guide ratio)
    if t_hbm >= c["flop"] / (tc * 1e12):
        return "hbm", pk["hbm_gbs"], "GB/s", by / 1e9
    return "tensor", tc, "TFLOP/s", c["flop"] / 1e12


KERNEL_NAMES = {0: "KS", 1: "KM-SIMT", 2: "KM-TC", 3: "KM-TC/G", 4: "KS-C3"}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons polled through NVML every ~1 ms in a thread
    (nvidia-smi -lms 10 if NVML is unavailable); only samples taken between
    mark_start() and mark_end() are summarised."""

    def __init__(self, cuda_index: int):
        self.cuda_index = cuda_index
        self.samples, self.stop = [], threading.Event()
        self.t_start = self.t_end = None
        self.max_mhz, self.source = None, None

    def __enter__(self):
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            try:
                idx = torch.cuda._get_nvml_device_index(self.cuda_index)
            except Exception:
                idx = self.cuda_index
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                    "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

            def poll():
                while not self.stop.is_set():
                    try:
                        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.time(), mhz, [n for n, b in bits.items() if r & b]))
                    except Exception:
                        pass
                    time.sleep(0.001)
            self.source = "nvml ~1 ms"
        except Exception:
            poll = self._smi
            self.source = "nvidia-smi -lms 10"
        self.th = threading.Thread(target=poll, daemon=True)
        self.th.start()
        t = time.time() + 5
        while not self.samples and time.time() < t:
            time.sleep(0.002)
        return self

    def _smi(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            p = subprocess.Popen(["nvidia-smi", "-i", str(self.cuda_index), f"--query-gpu={q}",
                                  "--format=csv,noheader,nounits", "-lms", "10"],
                                 stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            return
        for line in p.stdout:
            if self.stop.is_set():
                break
            f = [x.strip() for x in line.split(",")]
            try:
                self.max_mhz = float(f[1])
                self.samples.append((time.time(), float(f[0]),
                                     [n for n, v in zip(names, f[2:6]) if v.lower().startswith("active")]))
            except (ValueError, IndexError):
                continue
        p.terminate()

    def mark_start(self):
        self.t_start = time.time()

    def mark_end(self):
        self.t_end = time.time()

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=2)

    def summary(self):
        inside = [(m, r) for ts, m, r in self.samples
                  if self.t_start is not None and self.t_start <= ts <= (self.t_end or ts)]
        sm = [m for m, _ in inside]
        reasons = sorted({x for _, r in inside for x in r})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": self.source,
                "window_s": round((self.t_end or 0) - (self.t_start or 0), 4)}


# ----------------------------------------------------------------------------- helpers
def _ev():
    import torch
    return torch.cuda.Event(enable_timing=True)


def _capture(stream, fn):
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        stream.synchronize()
        g.capture_begin()
        fn()
        g.capture_end()
    return g


def _max_over_ranks(vals, dev, world):
    if world == 1:
        return list(vals)
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(vals), device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def _flush_l2(buf):
    buf.add_(1.0)              # writes > 2x L2 (evicts every layer's buffers)


def _r(x, n=3):
    return None if x is None else round(float(x), n)


# ----------------------------------------------------------------------------- headline
def headline(args, conv, dev, stream, world, rank, pk, sms):
    """configs[4] in FP32 / TF32 / BF16, M split over the ranks (strong)."""
    import torch
    import torch.distributed as dist
    c = layer_geom(synth.SHARD_SWEEP)
    C, Wx, Wy, K, M, Ho, Wo = (c[k] for k in ("C", "Wx", "Wy", "K", "M", "Ho", "Wo"))
    if M % world:
        raise SystemExit(f"M={M} not divisible by world={world}")
    Ml = M // world
    m0 = rank * Ml
    I32 = torch.from_numpy(synth.uniform01(synth.SEED_I, (C, Wy, Wx))).to(dev)
    if world > 1:
        from paper_2212_00404_b200.shard import broadcast_input
        broadcast_input(I32, src=0)                       # G0: once, untimed
    Fglob = synth.uniform_pm1(synth.SEED_F + 104, (M, C, K, K))
    Floc = torch.from_numpy(np.ascontiguousarray(Fglob[m0:m0 + Ml])).to(dev)
    del Fglob
    NSET = 2
    bufs = {}
    for p in args.precs:
        dt = torch.bfloat16 if p == "bf16" else torch.float32
        I = I32.to(dt).contiguous()
        Fs = [Floc.to(dt).contiguous() if j == 0 else Floc.to(dt).contiguous().clone() for j in range(NSET)]
        Os = [torch.empty((Ml, Ho, Wo), device=dev) for _ in range(NSET)]
        bufs[p] = (I, Fs, Os)
    plans = {p: conv.plan_multi(C, Wx, Wy, K, Ml, p) for p in args.precs}
    sh = stream.cuda_stream

    def call(p, j):
        I, Fs, Os = bufs[p]
        conv.conv_multi_ex(I, C, Wx, Wy, Fs[j], K, Ml, Os[j], p, sh)

    with torch.cuda.stream(stream):
        for j in range(NSET):
            for p in args.precs:
                call(p, j)
    stream.synchronize()
    # the step = one CUDA graph per buffer set: the precision calls PDL-chained
    # (each call's prologue overlaps the previous one's tail; no graph or
    # event boundary inside the step)
    step_g = [_capture(stream, lambda j=j: [call(p, j) for p in args.precs]) for j in range(NSET)]
    graphs = {(p, j): _capture(stream, lambda p=p, j=j: call(p, j)) for p in args.precs for j in range(NSET)}
    with torch.cuda.stream(stream):
        for s in range(args.warmup):
            step_g[s % NSET].replay()
    stream.synchronize()

    # ---- timed region: exactly K steps
    P = len(args.precs)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = _ev(), _ev()
    with ClockSampler(dev.index) as clk, torch.cuda.stream(stream):
        clk.mark_start()
        t0.record(stream)
        for s in range(args.steps):
            step_g[s % NSET].replay()
        t1.record(stream)
        stream.synchronize()
        clk.mark_end()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = _max_over_ranks([t0.elapsed_time(t1)], dev, world)[0]
    ms_step = total_ms / args.steps
    # ---- each kernel's live share of the PDL-chained step (outside the timed
    # region): what the step loses without it — R replays of the full step and
    # of each step-minus-precision graph, interleaved over 4 rounds
    minus = [_capture(stream, lambda i=i: [call(q, 0) for q in args.precs if q != args.precs[i]]) for i in range(P)]
    R = 50

    def _rep_ms(g):
        a, b = _ev(), _ev()
        a.record(stream)
        for _ in range(R):
            g.replay()
        b.record(stream)
        stream.synchronize()
        return a.elapsed_time(b) / R
    full_s, minus_s = [], [[] for _ in range(P)]
    with torch.cuda.stream(stream):
        for _ in range(4):
            full_s.append(_rep_ms(step_g[0]))
            for i in range(P):
                minus_s[i].append(_rep_ms(minus[i]))
    full = statistics.median(full_s)
    per_p_ms = [max(full - statistics.median(minus_s[i]), 1e-4) * args.steps for i in range(P)]
    scale = total_ms / max(sum(per_p_ms), 1e-9)               # shares of the timed region
    per_p_ms = _max_over_ranks([x * scale for x in per_p_ms], dev, world)
    flop_p = c["flop"]                                    # whole layer (all ranks)
    value = P * flop_p / (ms_step * 1e-3) / 1e9

    byp, kern = {}, {}
    for i, p in enumerate(args.precs):
        us = 1e3 * per_p_ms[i] / args.steps
        kname = KERNEL_NAMES.get(plans[p]["kernel"], "?") + ("" if p == "fp32" else f"-{p}")
        cl = dict(c, M=Ml, flop=c["flop"] / world)
        b, peak, unit, amount = roof(cl, p, kname, pk, sms)
        achieved = amount / (us * 1e-6)
        byp[p] = {"gflops": round(flop_p / (us * 1e-6) / 1e9, 1), "us": round(us, 2),
                  "bound": b, "frac": round(achieved / peak, 4)}
        kern[p] = {"kernel": kname, "bound": b, "achieved": round(achieved, 2), "peak": round(peak, 2),
                   "unit": unit, "frac": round(achieved / peak, 4), "avg_launch_us": round(us, 3),
                   "launches_per_call": plans[p]["launches"], "share": round(per_p_ms[i] / total_ms, 3),
                   "plan": plans[p]}
    dom = max(args.precs, key=lambda p: kern[p]["avg_launch_us"])
    d = kern[dom]
    traffic = _traffic_lookup(d["kernel"], world)
    roofline = {"bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"], "unit": d["unit"],
                "frac": d["frac"], "traffic": traffic, "kernel": d["kernel"], "share": d["share"],
                "peak_src": ("SMs*128*2*sm_max_mhz" if d["unit"] == "TFLOP/s" and dom == "fp32"
                             else pk["source"] + (" x0.5 (tf32)" if dom == "tf32" and d["bound"] == "tensor" else ""))}
    out = {"value": value, "ms_per_step": ms_step, "by_precision": byp, "kernels": kern, "roofline": roofline,
           "clocks": clk.summary(), "gpu_launches": args.steps * sum(plans[p]["launches"] for p in args.precs),
           "l2": f"inputs larger than L2: {NSET} F/O sets alternate, "
                 f"{sum(bufs[p][1][0].numel() * bufs[p][1][0].element_size() for p in args.precs) * NSET / 1e6:.0f} MB",
           "units": f"M={M} filters x {P} precisions; {Ml} per rank"}

    # ---- cold single calls (L2 flushed by writing 2x L2 before each), per precision
    flush = torch.empty(2 * L2_BYTES // 4, device=dev)
    cold = {}
    with torch.cuda.stream(stream):
        for p in args.precs:
            ts = []
            for _ in range(5):
                _flush_l2(flush)
                a, b = _ev(), _ev()
                a.record(stream)
                graphs[(p, 0)].replay()
                b.record(stream)
                stream.synchronize()
                ts.append(1e3 * a.elapsed_time(b))
            cold[p] = round(statistics.median(ts), 2)
    out["t_cold_us"] = cold
    del flush

    # ---- N > 1: T_1 on rank 0 alone (full M), and the O all-gather (G2)
    if world > 1:
        out["sweep_strong"] = _strong_extras(args, conv, dev, stream, world, rank, c, bufs, Ml, byp)
    out["_bufs"] = (bufs, plans, I32)
    return out


def _strong_extras(args, conv, dev, stream, world, rank, c, bufs, Ml, byp):
    import torch
    import torch.distributed as dist
    from paper_2212_00404_b200.shard import allgather_output
    C, Wx, Wy, K, M, Ho, Wo = (c[k] for k in ("C", "Wx", "Wy", "K", "M", "Ho", "Wo"))
    res = {}
    reps = 20
    for p in args.precs:
        t1 = None
        dist.barrier()
        if rank == 0:
            dt = torch.bfloat16 if p == "bf16" else torch.float32
            Ff = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + 104, (M, C, K, K))).to(dev).to(dt)
            Of = torch.empty((M, Ho, Wo), device=dev)
            I = bufs[p][0]
            g = _capture(stream, lambda: conv.conv_multi_ex(I, C, Wx, Wy, Ff, K, M, Of, p, stream.cuda_stream))
            with torch.cuda.stream(stream):
                g.replay()
                a, b = _ev(), _ev()
                a.record(stream)
                for _ in range(reps):
                    g.replay()
                b.record(stream)
            stream.synchronize()
            t1 = 1e3 * a.elapsed_time(b) / reps
            del g, Ff, Of
        dist.barrier()
        O = bufs[p][2][0]
        with torch.cuda.stream(stream):
            for _ in range(3):
                allgather_output(O, M)
            dist.barrier()
            stream.synchronize()
            a, b = _ev(), _ev()
            a.record(stream)
            for _ in range(reps):
                allgather_output(O, M)
            b.record(stream)
            stream.synchronize()
        ag = _max_over_ranks([1e3 * a.elapsed_time(b) / reps], dev, world)[0]
        t1b = torch.tensor([t1 or 0.0], device=dev, dtype=torch.float64)
        dist.broadcast(t1b, src=0)
        t1 = float(t1b.item())
        res[p] = {"t1_us": round(t1, 2), "tN_us": byp[p]["us"], "speedup": round(t1 / byp[p]["us"], 2),
                  "allgather_us": round(ag, 2), "allgather_recv_bytes": int(4 * (M - Ml) * Ho * Wo)}
        res[p].update(_fused_allgather(conv, dev, stream, world, rank, c, bufs[p], Ml, p, reps))
    return res


_SYMM = {}


def _fused_allgather(conv, dev, stream, world, rank, c, buf, Ml, prec, reps):
    """NEXT-2: conv with the all-gather fused into the epilogue
    (conv_multi_allgather_ex) into a torch symmetric-memory O: every rank's
    kernels store their rows straight into all ranks' O over NVLink (one
    multimem.st per value when the NVSwitch multicast object exists).  Device
    time per call, max over ranks; the barrier that publishes the rows is
    timed with it."""
    import torch
    import torch.distributed as dist
    try:
        import torch.distributed._symmetric_memory as symm
        C, Wx, Wy, K, M, Ho, Wo = (c[k] for k in ("C", "Wx", "Wy", "K", "M", "Ho", "Wo"))
        if "O" not in _SYMM:
            O = symm.empty((M, Ho, Wo), dtype=torch.float32, device=dev)
            hdl = symm.rendezvous(O, dist.group.WORLD)
            off = O.data_ptr() - hdl.buffer_ptrs[rank]
            peers = [hdl.buffer_ptrs[(rank + r) % world] + off for r in range(world)]
            mc = int(getattr(hdl, "multicast_ptr", 0) or 0)
            _SYMM.update(O=O, hdl=hdl, peers=peers, mc=(mc + off) if mc else None)
        I, Fs, _ = buf
        m0 = rank * Ml

        def call():
            conv.conv_multi_allgather_ex(I, C, Wx, Wy, Fs[0], K, Ml, m0, M, _SYMM["peers"], _SYMM["mc"], prec,
                                         stream.cuda_stream)
        with torch.cuda.stream(stream):
            for _ in range(3):
                call()
            stream.synchronize()
            dist.barrier()
            a, b = _ev(), _ev()
            a.record(stream)
            for _ in range(reps):
                call()
            b.record(stream)
            stream.synchronize()
        us = _max_over_ranks([1e3 * a.elapsed_time(b) / reps], dev, world)[0]
        return {"fused_allgather_us": round(us, 2), "fused_path": "multimem" if _SYMM["mc"] else "peer stores"}
    except Exception as exc:                       # reported, never fatal for the bench line
        return {"fused_allgather_error": repr(exc)[:120]}


def _traffic_lookup(kernel, world):
    """DRAM bytes per launch of the dominant kernel (ncu --set full, committed)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh)
        v = t.get(f"configs4/{kernel}/n{world}")
        return v if isinstance(v, (int, float)) else None
    except Exception:
        return None


# ----------------------------------------------------------------------------- e2e
def e2e(args, conv, dev, stream, world, rank, hb):
    """The headline step through the public host-buffer API: per precision
    conv_multi_host_async (pinned I and this rank's F slice H2D, kernels, O
    slice D2H), one stream per precision, one host synchronisation per step."""
    import torch
    import torch.distributed as dist
    bufs, _plans, _ = hb
    c = layer_geom(synth.SHARD_SWEEP)
    C, Wx, Wy, K, M = (c[k] for k in ("C", "Wx", "Wy", "K", "M"))
    Ml = M // world
    host = {}
    for p in args.precs:
        I, Fs, Os = bufs[p]
        host[p] = (I.cpu().pin_memory(), Fs[0].cpu().pin_memory(),
                   torch.empty(tuple(Os[0].shape), dtype=torch.float32).pin_memory())
    h2d = sum(a.numel() * a.element_size() + b.numel() * b.element_size() for a, b, _ in host.values())
    d2h = sum(o.numel() * 4 for _, _, o in host.values())
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(len(args.precs) - 1)]
    done = [torch.cuda.Event() for _ in streams]

    def one_step():
        for i, p in enumerate(args.precs):
            Ih, Fh, Oh = host[p]
            conv.conv_multi_host_async(Ih, C, Wx, Wy, Fh, K, Ml, Oh, p, streams[i].cuda_stream)
        for st, ev in zip(streams[1:], done[1:]):
            ev.record(st)
            stream.wait_event(ev)

    one_step()
    stream.synchronize()
    steps = max(1, min(args.steps, args.e2e_steps))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = _ev(), _ev()
    a.record(stream)
    for _ in range(steps):
        one_step()
        stream.synchronize()                     # results on the host once per step
    b.record(stream)
    b.synchronize()
    ms = _max_over_ranks([a.elapsed_time(b) / steps], dev, world)[0]
    flop = len(args.precs) * c["flop"]
    return {"value": round(flop / (ms * 1e-3) / 1e9, 1), "unit": UNIT, "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
            "api": "conv_multi_host_async (pinned)"}


# ----------------------------------------------------------------------------- suite (secondary)
def suite_calls(world, rank):
    calls = []
    for i, c in enumerate(synth.SINGLE_SWEEP):
        calls.append(dict(layer_geom(c), kind="single", prec="fp32", cfg_index=i))
    multi = list(synth.MULTI_LAYERS) + [synth.SHARD_SWEEP]
    for prec in PRECS:
        for j, c in enumerate(multi):
            calls.append(dict(layer_geom(c), kind="multi", prec=prec, cfg_index=100 + j))
    for c in calls:
        c["label"] = f"{c['name']}:{c['prec']}"
    return calls


def suite(args, conv, dev, stream, world, rank, pk, sms):
    """The 104-call layer suite (configs[1..4] + the 28x28x256 target layer);
    at N > 1 every rank runs a full-size filter slice (weak scaling)."""
    import torch
    import torch.distributed as dist
    calls = suite_calls(world, rank)
    cacheI = {}
    for c in calls:
        key = (c["C"], c["Wx"], c["Wy"])
        if key not in cacheI:
            cacheI[key] = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev)
        Fh = synth.uniform_pm1(synth.SEED_F + c["cfg_index"] + 7919 * rank, (c["M"], c["C"], c["K"], c["K"]))
        dt = torch.bfloat16 if c["prec"] == "bf16" else torch.float32
        c["I"] = cacheI[key].to(dt).contiguous()
        c["F"] = torch.from_numpy(Fh).to(dev).to(dt).contiguous()
        if c["kind"] == "single":
            c["I"] = c["I"][0].contiguous()
            c["F"] = c["F"][:, 0].contiguous()
        c["O"] = torch.empty((c["M"], c["Ho"], c["Wo"]), device=dev, dtype=torch.float32)
        c["plan"] = (conv.plan_single(c["Wx"], c["Wy"], c["K"], c["M"]) if c["kind"] == "single"
                     else conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], c["prec"]))
        k = KERNEL_NAMES.get(c["plan"]["kernel"], "?")
        c["kernel"] = k if (c["prec"] == "fp32" or k.startswith("KS")) and k != "KS-C3" else f"{k}-{c['prec']}"
    sh = stream.cuda_stream

    def launch(c):
        if c["kind"] == "single":
            conv.conv_single_ex(c["I"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"], sh)
        else:
            conv.conv_multi_ex(c["I"], c["C"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"], c["prec"], sh)

    with torch.cuda.stream(stream):
        for c in calls:
            launch(c)
    stream.synchronize()
    classes = [("single_fp32", [c for c in calls if c["kind"] == "single"])] + \
              [(f"multi_{p}", [c for c in calls if c["kind"] == "multi" and c["prec"] == p]) for p in PRECS]
    graphs = [_capture(stream, lambda cs=cs: [launch(c) for c in cs]) for _n, cs in classes]
    steps = max(3, min(args.steps, args.suite_steps))
    with torch.cuda.stream(stream):
        for g in graphs:
            g.replay()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[_ev() for _ in range(len(graphs) + 1)] for _ in range(steps)]
    with torch.cuda.stream(stream):
        for s in range(steps):
            evs[s][0].record(stream)
            for i, g in enumerate(graphs):
                g.replay()
                evs[s][i + 1].record(stream)
    stream.synchronize()
    tot = evs[0][0].elapsed_time(evs[-1][-1]) / steps
    per = [sum(evs[s][i].elapsed_time(evs[s][i + 1]) for s in range(steps)) / steps for i in range(len(graphs))]
    tot, *per = _max_over_ranks([tot] + per, dev, world)
    res = {"layers": len(calls), "ms_per_step": round(tot, 4),
           "value": round(world * sum(c["flop"] for c in calls) / (tot * 1e-3) / 1e9, 1),
           "scaling": "weak" if world > 1 else None}
    for (name, cs), ms in zip(classes, per):
        res[name] = {"gflops": round(world * sum(c["flop"] for c in cs) / (ms * 1e-3) / 1e9, 1),
                     "us": round(1e3 * ms, 2)}
    return res, calls, launch


def layer_b2b(calls, launch_fn, stream, pk, sms, reps=12):
    """Each layer alone: `reps` launches back to back in a graph, rotating F/O
    copies so its working set exceeds 3x L2."""
    import torch
    out = {}
    for c in calls:
        per = c["O"].numel() * 4 + c["F"].numel() * c["F"].element_size()
        nrot = max(1, min(12, math.ceil(3 * L2_BYTES / per)))
        vs = []
        for i in range(nrot):
            v = dict(c)
            if i:
                v["F"], v["O"] = c["F"].clone(), torch.empty_like(c["O"])
            vs.append(v)
        for v in vs:
            launch_fn(v)
        g = _capture(stream, lambda: [launch_fn(vs[i % nrot]) for i in range(reps)])
        with torch.cuda.stream(stream):
            g.replay()
            a, b = _ev(), _ev()
            a.record(stream)
            g.replay()
            b.record(stream)
        stream.synchronize()
        us = 1e3 * a.elapsed_time(b) / reps
        bound, peak, unit, amount = roof(c, c["prec"], c.get("kernel", "KS"), pk, sms)
        out[c["label"]] = {"us": round(us, 3), "gflops": round(c["flop"] / (us * 1e-6) / 1e9, 1),
                           "bound": bound, "frac": round(amount / (us * 1e-6) / peak, 4)}
        del g, vs
    return out


def cudnn_context(calls, stream, pk, sms):
    import torch
    torch.backends.cudnn.benchmark = True

    def fn(c):
        torch.backends.cudnn.allow_tf32 = c["prec"] == "tf32"
        I = c["I"][None] if c["kind"] == "multi" else c["I"][None, None]
        F = c["F"] if c["kind"] == "multi" else c["F"][:, None]
        return torch.nn.functional.conv2d(I, F)

    with torch.cuda.stream(stream):
        for c in calls:
            fn(c)
        stream.synchronize()
        lay = layer_b2b(calls, fn, stream, pk, sms)
    torch.backends.cudnn.allow_tf32 = True
    tot_us = sum(v["us"] for v in lay.values())
    return {"engine": f"torch conv2d -> cuDNN {torch.backends.cudnn.version()}, benchmark=True, "
                      "fp32 layers allow_tf32=False",
            "value": round(sum(c["flop"] for c in calls) / (tot_us * 1e-6) / 1e9, 1),
            "ms_sum_of_layers": round(tot_us / 1e3, 4), "layers_us": {k: v["us"] for k, v in lay.items()}}


def launch_floor(conv, stream):
    """Empty-kernel floor: one library no-op launch, back to back in a graph."""
    import torch
    reps = 200
    g = _capture(stream, lambda: [conv.diag_nop(stream.cuda_stream) for _ in range(reps)])
    with torch.cuda.stream(stream):
        g.replay()
        a, b = _ev(), _ev()
        a.record(stream)
        g.replay()
        b.record(stream)
    stream.synchronize()
    return round(1e3 * a.elapsed_time(b) / reps, 3)


def batched(args, conv, dev, stream, pk):
    """28x28x256 as CNNs run it (NEXT-1 batch, NEXT-3 padding / stride)."""
    import torch
    out = {}

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        g = _capture(stream, lambda: [fn() for _ in range(reps)])
        with torch.cuda.stream(stream):
            g.replay()
            a, b = _ev(), _ev()
            a.record(stream)
            g.replay()
            b.record(stream)
        stream.synchronize()
        return 1e3 * a.elapsed_time(b) / reps

    C, W, K, M = 256, 28, 3, 256
    sh = stream.cuda_stream
    for prec in PRECS:
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        peak = fp32_peak_tflops(pk, 148) if prec == "fp32" else pk["bf16_tflops"] * (0.5 if prec == "tf32" else 1)
        for N, pad in ((8, 0), (32, 0), (64, 0), (1, 1), (32, 1)):
            if prec == "fp32" and N == 64:
                continue
            I = torch.from_numpy(synth.uniform01(synth.SEED_I + N, (N, C, W, W))).to(dev, dt)
            F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + N, (M, C, K, K))).to(dev, dt)
            Ho = W + 2 * pad - K + 1
            Os = [torch.empty((N, M, Ho, Ho), device=dev) for _ in range(3)]
            it = iter(range(10 ** 9))
            us = timeit(lambda: conv.conv_multi_pad_ex(I, N, C, W, W, F, K, M, pad, Os[next(it) % 3], prec, sh))
            tf = 2.0 * N * M * C * K * K * Ho * Ho / (us * 1e-6) / 1e12
            out[f"{prec}_n{N}" + ("_pad1" if pad else "")] = {"us": round(us, 2), "tflops": round(tf, 1),
                                                              "frac": round(tf / peak, 4)}
    C2, W2, K2, M2, P2, S2 = 64, 56, 3, 128, 1, 2
    Ho2 = (W2 + 2 * P2 - K2) // S2 + 1
    for prec in PRECS:
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        for N in (1, 8):
            I = torch.from_numpy(synth.uniform01(synth.SEED_I + 11 * N, (N, C2, W2, W2))).to(dev, dt)
            F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + 11 * N, (M2, C2, K2, K2))).to(dev, dt)
            Os = [torch.empty((N, M2, Ho2, Ho2), device=dev) for _ in range(3)]
            it = iter(range(10 ** 9))
            us = timeit(lambda: conv.conv_multi_strided_ex(I, N, C2, W2, W2, F, K2, M2, P2, S2, Os[next(it) % 3],
                                                           prec, sh))
            out[f"{prec}_n{N}_s2"] = {"us": round(us, 2),
                                      "tflops": round(2.0 * N * M2 * C2 * 9 * Ho2 * Ho2 / (us * 1e-6) / 1e12, 1)}
    return out


# ----------------------------------------------------------------------------- CPU oracle
def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_sample(budget_s, threads, precs):
    """The oracle (fp64 C) on the headline step, bounded: the first m_s filters
    of the configs[4] layer, once per precision, m_s sized for ~budget_s.
    Returns (flop, seconds, sample description, threads used)."""
    import oracle
    used = oracle.set_threads(threads)
    c = layer_geom(synth.SHARD_SWEEP)
    I = synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))
    Fcal = synth.uniform_pm1(synth.SEED_F + 104, (max(used, 8), c["C"], c["K"], c["K"]))
    t = time.perf_counter()
    oracle.conv_multi(I, Fcal)
    s_per_filter = (time.perf_counter() - t) / Fcal.shape[0]
    ms = int(max(1, min(c["M"], budget_s / max(1e-9, s_per_filter * len(precs)))))
    if ms >= used:
        ms -= ms % used                                   # whole OpenMP rounds (threads over m)
    F = synth.uniform_pm1(synth.SEED_F + 104, (ms, c["C"], c["K"], c["K"]))
    flop, secs = 0.0, 0.0
    for _ in precs:
        t = time.perf_counter()
        oracle.conv_multi(I, F)
        secs += time.perf_counter() - t
        flop += 2.0 * ms * c["C"] * c["K"] ** 2 * c["Ho"] * c["Wo"]
    desc = f"configs[4], {ms}/{c['M']} filters x{len(precs)} precs ({flop / 1e9:.2f} GFLOP)"
    return flop, secs, desc, used


def cpu_baseline(budget_s, precs):
    threads = os.cpu_count() or 1
    flop, secs, desc, used = oracle_sample(budget_s, threads, precs)
    f1, s1, d1, _ = oracle_sample(min(3.0, budget_s / 4), 1, precs[:1])
    return {"value": round(flop / secs / 1e9, 3), "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": desc, "cpu": cpu_model(), "one_thread_gflops": round(f1 / s1 / 1e9, 3)}


def run_reference(args):
    """--impl reference: the oracle as it stands (all host cores), rank 0 only."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    precs = args.precs
    c = layer_geom(synth.SHARD_SWEEP)
    # bound each step so W + K steps take ~args.ref_total_s in all
    per_step = max(0.2, min(args.ref_step_seconds, args.ref_total_s / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(min(per_step, 1.0), os.cpu_count() or 1, precs)
    flops, secs = 0.0, 0.0
    for _ in range(args.steps):
        f, s, desc, used = oracle_sample(per_step, os.cpu_count() or 1, precs)
        flops += f
        secs += s
    value = flops / secs / 1e9
    res = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / args.steps, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "impl": "reference",
           "dtype": "f64 (oracle)", "data": "synthetic (splitmix64 seeded)",
           "config": {"workload": WORKLOAD, "layer": c["name"], "precisions": list(precs)},
           "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": used, "kind": "oracle",
                            "sample": desc, "cpu": cpu_model()},
           "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    backend = os.environ.get("B200CONV_BENCH_BACKEND", "nccl")
    if world > 1 and backend == "nccl":
        # the communicator (size, NVLS / NVLink transport) in the log; rank 0 only
        os.environ.setdefault("NCCL_DEBUG", "INFO" if rank == 0 else "WARN")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import torch
    import torch.distributed as dist
    from paper_2212_00404_b200 import conv

    if backend != "nccl":
        # (gloo + more ranks than GPUs: a functional check of the N > 1 path on
        # one GPU — the ranks share a device; its timings mean nothing)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    conv.load()
    pk = peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    stream = torch.cuda.Stream(device=dev)
    detail = {}

    hl = headline(args, conv, dev, stream, world, rank, pk, sms)
    hb = hl.pop("_bufs")
    detail["headline_kernels"] = hl["kernels"]
    e2e_res = e2e(args, conv, dev, stream, world, rank, hb) if args.e2e else None
    del hb
    torch.cuda.empty_cache()
    floor = launch_floor(conv, stream)

    suite_res, calls, launch = (suite(args, conv, dev, stream, world, rank, pk, sms) if args.suite
                                else (None, None, None))
    if rank == 0 and world == 1:
        if args.layers and calls is not None:
            detail["layers_b2b"] = layer_b2b(calls, launch, stream, pk, sms)
        if args.cudnn and calls is not None:
            detail["cudnn"] = cudnn_context(calls, stream, pk, sms)
        if args.batched:
            detail["batched"] = batched(args, conv, dev, stream, pk)
    cpu = cpu_baseline(args.cpu_seconds, args.precs) if (rank == 0 and world == 1 and args.cpu_seconds > 0) else None

    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    clocks = hl["clocks"]
    res = {
        "metric": METRIC, "value": round(hl["value"], 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(hl["ms_per_step"], 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32+tf32+bf16 (fp32 acc)",
        "data": "synthetic (splitmix64; I~U[0,1), F~U[-1,1))",
        "config": {"workload": WORKLOAD, "layer": "configs[4] 14x14 C=512 M=4096 K=3",
                   "precisions": list(args.precs), "parallelism": f"filters m split over {world} GPU(s)",
                   "l2": hl["l2"]},
        "by_precision": hl["by_precision"],
        "roofline": hl["roofline"],
        "gpu_launches": hl["gpu_launches"],
        "e2e": e2e_res,
        "cpu_baseline": cpu,
        "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons", "samples")},
        "t_cold_us": hl["t_cold_us"],
        "launch_floor_us": floor,
        "suite": ({k: suite_res[k] for k in ("value", "ms_per_step", "single_fp32", "multi_fp32",
                                             "multi_tf32", "multi_bf16")} if suite_res else None),
    }
    if "sweep_strong" in hl:
        detail["sweep_strong"] = hl["sweep_strong"]
        keep = ("t1_us", "tN_us", "speedup", "allgather_us", "fused_allgather_us")
        res["sweep_strong"] = {p: {k: v[k] for k in keep if k in v} for p, v in hl["sweep_strong"].items()}
    detail["suite"] = suite_res
    detail["clocks"] = clocks
    detail["paper_context"] = {"single_vs_cudnn71_avg": 2.6, "multi_vs_cudnn71_avg": 1.39,
                               "hardware": "GTX 1080Ti (Pascal), FP32, cuDNN v7.1 (PAPER.md P:704, P:717)"}
    path = os.path.join(ROOT, "gpurun_out", f"bench_detail_n{world}.json")
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "w") as fh:
            json.dump({"headline": res, **detail}, fh, indent=1)
        res["detail"] = os.path.relpath(path, ROOT)
    except OSError:
        pass
    for k, v in detail.items():                    # detail first (one line each), headline LAST
        print(json.dumps({"detail": k, "data": v}), flush=True)
    line = json.dumps(res, separators=(",", ":"))
    if len(line) > 2000:                            # keep the headline parseable from a stdout tail
        res.pop("suite", None)
        line = json.dumps(res, separators=(",", ":"))
    print(line, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32,tf32,bf16")
    ap.add_argument("--suite", type=int, default=1)
    ap.add_argument("--suite-steps", type=int, default=200)
    ap.add_argument("--cudnn", type=int, default=1)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--batched", type=int, default=1)
    ap.add_argument("--e2e", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
    ap.add_argument("--ref-step-seconds", type=float, default=8.0)
    ap.add_argument("--ref-total-s", type=float, default=90.0)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    args.precs = tuple(args.precision.split(","))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
