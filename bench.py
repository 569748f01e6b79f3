#!/usr/bin/env python
"""bench.py — throughput of the arXiv 2212.00404 hot path on B200.

One step = one pass of the whole hot path over the BASELINE.json layer suite
("layer-suite"):
  * configs[1]  single-channel sweep, 80 layers (KS, FP32)      Eq. 2
  * configs[2,3] + the 28x28x256 target layer: 7 multi-channel layers
  * configs[4]  14x14 C=512 M=4096 K=3 multi-channel sweep layer
  every multi-channel layer in all three precisions: FP32 (KM-SIMT),
  TF32 and BF16 (KM-TC, tcgen05)                                 Eq. 1
Metric: GFLOP/s (direct-conv count 2*M*C*K*K*Ho*Wo, summed over the step).

Multi-GPU (torchrun, one rank per GPU): every layer's filter set is sharded by
filter index m (Fig. 2(c) P:362-371 lifted to GPUs); rank r owns a
full-size slice of a global problem with N*M filters, so per-GPU work is fixed
("scaling": "weak") and no collective is on the data path (O stays sharded).
I is broadcast once at setup over NCCL.  The strong-scaling numbers of the
configs[4] sweep (M = 4096 split N ways) are reported in "strong_sweep".

Timing: W warm-up steps; the step is captured in ONE CUDA graph (one call per
layer, PDL-chained; the per-group breakdown is the time the step loses
without each group); K steps replayed back to back
between a barrier + synchronize on both sides; device time from CUDA events;
max over ranks.  The step's working set (>1.5 GB) is far larger than the
126 MB L2, so every layer's buffers are evicted by the rest of the step before
they are touched again ("l2": "inputs larger than L2").
`--impl reference` times the CPU oracle (oracle/, fp64) on a bounded sample of
the same workload on the host cores.
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
WORKLOAD = "layer-suite"
NUM_SMS = 148
FP32_LANES_PER_SM = 128


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "sm_max_mhz": float(p.get("sm_max_mhz", 1965.0)), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0, "source": "fallback"}


# ----------------------------------------------------------------------------- workload
def suite(world: int = 1, rank: int = 0, precisions=("fp32", "tf32", "bf16")):
    """List of layer calls of one step for this rank."""
    calls = []
    for i, c in enumerate(synth.SINGLE_SWEEP):
        calls.append(dict(c, kind="single", prec="fp32", cfg_index=i))
    multi = list(synth.MULTI_LAYERS) + [synth.SHARD_SWEEP]
    for prec in precisions:
        for j, c in enumerate(multi):
            calls.append(dict(c, kind="multi", prec=prec, cfg_index=100 + j))
    for c in calls:
        c["Ho"], c["Wo"] = c["Wy"] - c["K"] + 1, c["Wx"] - c["K"] + 1
        c["flop"] = 2.0 * c["M"] * c["C"] * c["K"] ** 2 * c["Ho"] * c["Wo"]
        e = 2 if c["prec"] == "bf16" else 4
        c["bytes_alg"] = e * (c["C"] * c["Wx"] * c["Wy"] + c["M"] * c["C"] * c["K"] ** 2) \
            + 4 * c["M"] * c["Ho"] * c["Wo"]
        c["kernel"] = {"single": "KS"}.get(c["kind"]) or _multi_name(c)
        c["label"] = f"{c['name']}:{c['prec']}"
    return calls


def _multi_name(c):
    """Kernel group of a multi-channel call, as planned: KS-C3 (RGB stems, any
    precision), KM-SIMT (FP32), KM-TC (implicit) or KM-TC/G (im2col + GEMM)."""
    try:
        from paper_2212_00404_b200 import conv
        k = conv.plan_multi(c["C"], c["Wx"], c["Wy"], c["K"], c["M"], c["prec"])["kernel"]
    except Exception:
        k = 1 if c["prec"] == "fp32" else 2
    if k == 4:
        return f"KS-C3-{c['prec']}"
    if c["prec"] == "fp32":
        return "KM-SIMT"
    return f"{'KM-TC/G' if k == 3 else 'KM-TC'}-{c['prec']}"


def roof_for(c, pk):
    """(bound, peak, unit, algorithmic amount per launch) of one call."""
    clk = pk["sm_max_mhz"] * 1e6
    if c["kernel"] == "KS" or c["kernel"].startswith("KS-C3"):
        fp32_peak = NUM_SMS * FP32_LANES_PER_SM * 2 * clk / 1e12         # TFLOP/s
        t_hbm = c["bytes_alg"] / (pk["hbm_gbs"] * 1e9)
        t_alu = c["flop"] / (fp32_peak * 1e12)
        if t_hbm >= t_alu:
            return "hbm", pk["hbm_gbs"], "GB/s", c["bytes_alg"] / 1e9
        return "alu", fp32_peak, "TFLOP/s", c["flop"] / 1e12
    if c["kernel"] == "KM-SIMT":
        return "alu", NUM_SMS * FP32_LANES_PER_SM * 2 * clk / 1e12, "TFLOP/s", c["flop"] / 1e12
    tc_peak = pk["bf16_tflops"] * (0.5 if c["prec"] == "tf32" else 1.0)   # tf32 = bf16/2 (guide ratio)
    t_hbm = c["bytes_alg"] / (pk["hbm_gbs"] * 1e9)
    t_tc = c["flop"] / (tc_peak * 1e12)
    if t_hbm >= t_tc:
        return "hbm", pk["hbm_gbs"], "GB/s", c["bytes_alg"] / 1e9
    return "tensor", tc_peak, "TFLOP/s", c["flop"] / 1e12


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampled every 100 ms in a thread; only samples whose host
    arrival time falls inside [mark_start, mark_end] are summarised."""

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []
        self.t_start = self.t_end = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t = time.time() + 5
            while not self.lines and time.time() < t:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark_start(self):
        self.t_start = time.time()

    def mark_end(self):
        self.t_end = time.time()

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if self.t_start is not None and not (self.t_start <= ts <= (self.t_end or ts) + 0.05):
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_max": max(pw) if pw else None,
                "window_s": round((self.t_end or 0) - (self.t_start or 0), 3)}


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2212_00404_b200 import conv
    from paper_2212_00404_b200.shard import broadcast_input

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # (B200CONV_BENCH_BACKEND=gloo + more ranks than GPUs: a functional check of
    # the N > 1 path on one GPU — ranks share devices; its timings mean nothing)
    backend = os.environ.get("B200CONV_BENCH_BACKEND", "nccl")
    if backend != "nccl":
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
    precisions = tuple(args.precision.split(","))
    calls = suite(world, rank, precisions)

    # ---- inputs: I identical on every rank (broadcast from rank 0 once, untimed);
    # F: this rank's slice of the global N*M filters (seeded per rank)
    torch.manual_seed(0)
    cacheI = {}
    for c in calls:
        key = (c["C"], c["Wx"], c["Wy"])
        if key not in cacheI:
            I = torch.from_numpy(synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))).to(dev)
            broadcast_input(I, src=0)            # once, untimed (NCCL over NVLink)
            cacheI[key] = I
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

    stream = torch.cuda.Stream(device=dev)
    sh = stream.cuda_stream

    def launch(c):
        if c["kind"] == "single":
            conv.conv_single_ex(c["I"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"], sh)
        else:
            conv.conv_multi_ex(c["I"], c["C"], c["Wx"], c["Wy"], c["F"], c["K"], c["M"], c["O"],
                               c["prec"], sh)

    # ---- warm-up (direct launches: first-call attribute setup, caches, clocks)
    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup)):
            for c in calls:
                launch(c)
    stream.synchronize()

    # ---- the step grouped by (kernel, binding roof); each group is timed live
    # as the difference between the step and the step without it (below)
    order = []
    for c in calls:
        c["bound"] = roof_for(c, pk)[0]
        key = (c["kernel"], c["bound"])
        if key not in order:
            order.append(key)
    groups = [(key, [c for c in calls if (c["kernel"], c["bound"]) == key]) for key in order]

    def capture(fn):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            stream.synchronize()
            g.capture_begin()
            fn()
            g.capture_end()
        return g

    # the whole step as ONE graph (every layer PDL-chained to the next) for the
    # timed region; for the per-group breakdown below, the step without each
    # group in turn (a group's time = what removing it saves: its share of the
    # PDL-chained step, with no event or graph boundary around it)
    step_graph = capture(lambda: [launch(c) for _key, cs in groups for c in cs])
    G = len(groups)
    minus_graphs = [capture(lambda gi=gi: [launch(c) for gj, (_key, cs) in enumerate(groups) if gj != gi
                                           for c in cs]) for gi in range(G)]
    with torch.cuda.stream(stream):
        for _ in range(max(1, args.warmup)):
            step_graph.replay()
            for g in minus_graphs:
                g.replay()
    torch.cuda.synchronize()

    # ---- timed region: exactly K steps
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        clk.mark_start()
        t0.record(stream)
        for s in range(args.steps):
            step_graph.replay()
        t1.record(stream)
        stream.synchronize()
        clk.mark_end()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t0.elapsed_time(t1)
    # per-group breakdown (outside the timed region): R replays of the full
    # step and of each step-minus-group graph, interleaved in 4 rounds
    R = max(20, min(args.steps, 100))

    def _replays_us(g):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(R):
            g.replay()
        b.record(stream)
        stream.synchronize()
        return 1e3 * a.elapsed_time(b) / R
    full_s, minus_s = [], [[] for _ in range(G)]
    with torch.cuda.stream(stream):
        for _round in range(4):
            full_s.append(_replays_us(step_graph))
            for gi in range(G):
                minus_s[gi].append(_replays_us(minus_graphs[gi]))
    if world > 1:
        tt = torch.tensor([total_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_per_step = total_ms / args.steps
    flop_rank = sum(c["flop"] for c in calls)
    value = world * flop_rank / (ms_per_step * 1e-3) / 1e9

    # ---- per-group (kernel x roof) live timing -> roofline of the dominant kernel
    full_us = statistics.median(full_s)
    gus = [max(full_us - statistics.median(minus_s[gi]), 1e-3) for gi in range(G)]
    step_us_sum = sum(gus)
    kernels = {}
    for (key, cs), us in zip(groups, gus):
        b, peak, unit, _ = roof_for(cs[0], pk)
        amount = sum(roof_for(c, pk)[3] for c in cs)
        achieved = amount / (us * 1e-6)
        kernels[f"{key[0]}/{key[1]}"] = {
            "kernel": key[0], "bound": b, "launches_per_step": len(cs),
            "kernel_launches_per_step": sum(c["plan"]["launches"] for c in cs), "us_per_step": round(us, 2),
            "avg_launch_us": round(us / len(cs), 3), "share": round(us / step_us_sum, 3),
            "achieved": round(achieved, 2), "peak": round(peak, 2), "unit": unit,
            "frac": round(achieved / peak, 4)}
    dom_key = max(kernels, key=lambda k: kernels[k]["us_per_step"])
    d = kernels[dom_key]
    roofline = {"bound": d["bound"], "achieved": d["achieved"], "peak": d["peak"], "unit": d["unit"],
                "frac": d["frac"], "traffic": _traffic_lookup(dom_key),
                "kernel": dom_key, "share_of_step": d["share"],
                "launches_per_step": d["launches_per_step"], "avg_launch_us": d["avg_launch_us"],
                "kernel_launches_per_step": d["kernel_launches_per_step"],
                "launch_note": "a launch = one call of the hot path; calls whose channel split is reduced "
                               "through the split-K workspace are 2 kernels (main + fixed-order reduce), "
                               "both inside the timed duration",
                "peak_source": pk["source"] + (" x0.5 (tf32 = bf16/2, guide ratio)"
                                               if "tf32" in dom_key and d["bound"] == "tensor" else "")}

    # ---- per-layer latencies: each layer alone, back to back in a graph, with
    # rotating buffers so its working set exceeds L2 (separate from the timed region)
    layers = _layer_b2b(calls, launch, capture, stream, dev, pk) if args.layers else None

    # ---- strong scaling of the configs[4] sweep (M = 4096 split over the N ranks)
    strong = _strong_sweep(args, conv, dev, stream, world, rank, cacheI)

    # ---- batched tensor-core path on the 28x28x256 layer
    batched = _batched(args, conv, dev, stream, pk) if args.batched and rank == 0 else None

    # ---- cuDNN context on the same device / buffers
    cudnn = _cudnn_context(args, calls, dev, stream, capture, pk) if args.cudnn and rank == 0 else None

    # ---- e2e through the public API with host buffers (H2D + kernel + D2H per layer)
    e2e = _e2e(args, conv, calls, stream, world, rank, dev)

    # ---- CPU baseline: the oracle, rank 0 at N=1 only
    cpu = _cpu_baseline(calls, args.cpu_seconds) if (rank == 0 and world == 1 and args.cpu_seconds > 0) else None

    res = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 (KS, KM-SIMT) + tf32 + bf16 (KM-TC); fp32 accumulate",
        "data": "synthetic (splitmix64 seeded; I~U[0,1), F~U[-1,1))",
        "config": {"workload": WORKLOAD, "layers_per_step": len(calls),
                   "single_sweep": "configs[1]: Wx=Wy in {7,14,28,56,224} x K in {1,3,5,7} x M in {32..256}",
                   "multi_layers": [c["name"] for c in synth.MULTI_LAYERS] + [synth.SHARD_SWEEP["name"]],
                   "precisions": list(precisions), "batch": 1,
                   "parallelism": f"filter-sharded m over {world} GPU(s), no data-path collective",
                   "l2": "inputs larger than L2 (step working set %.2f GB >> 126 MB L2)" %
                         (sum(c['O'].numel() * 4 + c['F'].numel() * c['F'].element_size() for c in calls) / 1e9),
                   "timing": "the step as one CUDA graph (PDL-chained launches) replayed K times, CUDA events, max over ranks"},
        "roofline": roofline,
        "kernels": kernels,
        "layers_b2b": layers,
        "gpu_launches": sum(c["plan"]["launches"] for c in calls) * args.steps,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "strong_sweep": strong,
        "batched": batched,
        "cudnn_context": cudnn,
        "clocks": clk.summary(),
        "paper_context": {"single_vs_cudnn71_avg": 2.6, "multi_vs_cudnn71_avg": 1.39,
                          "hardware": "GTX 1080Ti (Pascal), FP32, cuDNN v7.1 (PAPER.md P:704, P:717)"},
    }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(res))


L2_BYTES = 126 * 2 ** 20


def _rotations(c):
    """How many buffer copies make one layer's repeated launches exceed 3x L2."""
    per = c["O"].numel() * 4 + c["F"].numel() * c["F"].element_size()
    return max(1, min(12, math.ceil(3 * L2_BYTES / per)))


def _layer_b2b(calls, launch, capture, stream, dev, pk, reps=12, cudnn_fn=None):
    import torch
    out = {}
    for c in calls:
        nrot = _rotations(c)
        Fs = [c["F"]] + [c["F"].clone() for _ in range(nrot - 1)]
        Os = [c["O"]] + [torch.empty_like(c["O"]) for _ in range(nrot - 1)]
        variants = []
        for i in range(nrot):
            v = dict(c)
            v["F"], v["O"] = Fs[i], Os[i]
            variants.append(v)
        fn = cudnn_fn or launch
        for v in variants:
            fn(v)
        g = capture(lambda: [fn(variants[i % nrot]) for i in range(reps)])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            g.replay()                                    # warm (on the timing stream)
            stream.synchronize()
            e0.record(stream)
            g.replay()
            e1.record(stream)
        stream.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / reps
        bound, peak, unit, amount = roof_for(c, pk)
        out[c["label"]] = {"us": round(us, 3), "gflops": round(c["flop"] / (us * 1e-6) / 1e9, 1),
                           "bound": bound, "frac": round(amount / (us * 1e-6) / peak, 4),
                           "gbs_alg": round(c["bytes_alg"] / (us * 1e-6) / 1e9, 1)}
        del g, Fs, Os, variants
    return out


def _traffic_lookup(kernel):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
        return t.get(kernel)
    except Exception:
        return None


def _batched(args, conv, dev, stream, pk):
    """The north-star tensor-pipe layer (28x28, C = M = 256, K = 3) as CNNs run it:
    a batch of N images in ONE launch (conv_multi_batched_ex), graph replay,
    device events; tensor fraction against the measured peak (TF32 = bf16 / 2)."""
    import torch
    C, W, K, M = 256, 28, 3, 256
    Ho = W - K + 1
    out = {}
    for prec in ("fp32", "tf32", "bf16"):
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        # fp32: the strict-FP32 KM-SIMT path, one launch over the batch (frac of the FMA pipe)
        peak = NUM_SMS * FP32_LANES_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12 if prec == "fp32" \
            else pk["bf16_tflops"] * (0.5 if prec == "tf32" else 1.0)
        for N in ((8, 32) if prec == "fp32" else (8, 32, 64)):
            I = torch.from_numpy(synth.uniform01(synth.SEED_I + N, (N, C, W, W))).to(dev, dt)
            F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + N, (M, C, K, K))).to(dev, dt)
            Os = [torch.empty((N, M, Ho, Ho), device=dev) for _ in range(3)]
            g = torch.cuda.CUDAGraph()
            reps = 10
            with torch.cuda.stream(stream):
                for j in range(3):
                    conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, Os[j % 3], prec, stream.cuda_stream)
                stream.synchronize()
                g.capture_begin()
                for j in range(reps):
                    conv.conv_multi_batched_ex(I, N, C, W, W, F, K, M, Os[j % 3], prec, stream.cuda_stream)
                g.capture_end()
                g.replay()
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                stream.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / reps
            tflops = 2.0 * N * M * C * K * K * Ho * Ho / (us * 1e-6) / 1e12
            out[f"{prec}_n{N}"] = {"us": round(us, 2), "tflops": round(tflops, 1),
                                   ("fma_frac" if prec == "fp32" else "tensor_frac"): round(tflops / peak, 4),
                                   "plan": conv.plan_multi_batched(N, C, W, W, K, M, prec)}
    # the same layer as the networks define it: "same" 3x3 convolution (zero
    # padding 1) — pad pre-pass + the batched kernel
    for prec in ("fp32", "tf32", "bf16"):
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        for N in ((1,) if prec == "fp32" else (1, 32)):
            I = torch.from_numpy(synth.uniform01(synth.SEED_I + 7 * N, (N, C, W, W))).to(dev, dt)
            F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + 7 * N, (M, C, K, K))).to(dev, dt)
            Os = [torch.empty((N, M, W, W), device=dev) for _ in range(3)]
            g = torch.cuda.CUDAGraph()
            reps = 10
            with torch.cuda.stream(stream):
                for j in range(3):
                    conv.conv_multi_pad_ex(I, N, C, W, W, F, K, M, 1, Os[j % 3], prec, stream.cuda_stream)
                stream.synchronize()
                g.capture_begin()
                for j in range(reps):
                    conv.conv_multi_pad_ex(I, N, C, W, W, F, K, M, 1, Os[j % 3], prec, stream.cuda_stream)
                g.capture_end()
                g.replay()
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                stream.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / reps
            tflops = 2.0 * N * M * C * K * K * W * W / (us * 1e-6) / 1e12
            entry = {"us": round(us, 2), "tflops": round(tflops, 1)}
            if prec != "fp32":
                entry["tensor_frac"] = round(tflops / (pk["bf16_tflops"] * (0.5 if prec == "tf32" else 1.0)), 4)
            out[f"{prec}_n{N}_pad1"] = entry
    # stride 2: the ResNet downsampling 3x3 convolution,
    # 56x56x64 -> 28x28x128, pad 1 (conv_multi_strided_ex; per image)
    C2, W2, K2, M2, P2, S2 = 64, 56, 3, 128, 1, 2
    Ho2 = (W2 + 2 * P2 - K2) // S2 + 1
    for prec in ("fp32", "tf32", "bf16"):
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        for N in (1, 8):
            I = torch.from_numpy(synth.uniform01(synth.SEED_I + 11 * N, (N, C2, W2, W2))).to(dev, dt)
            F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + 11 * N, (M2, C2, K2, K2))).to(dev, dt)
            Os = [torch.empty((N, M2, Ho2, Ho2), device=dev) for _ in range(3)]
            g = torch.cuda.CUDAGraph()
            reps = 10
            with torch.cuda.stream(stream):
                for j in range(3):
                    conv.conv_multi_strided_ex(I, N, C2, W2, W2, F, K2, M2, P2, S2, Os[j % 3], prec,
                                               stream.cuda_stream)
                stream.synchronize()
                g.capture_begin()
                for j in range(reps):
                    conv.conv_multi_strided_ex(I, N, C2, W2, W2, F, K2, M2, P2, S2, Os[j % 3], prec,
                                               stream.cuda_stream)
                g.capture_end()
                g.replay()
                stream.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.replay()
                e1.record(stream)
                stream.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / reps
            tflops = 2.0 * N * M2 * C2 * K2 * K2 * Ho2 * Ho2 / (us * 1e-6) / 1e12
            entry = {"us": round(us, 2), "tflops": round(tflops, 1),
                     "layer": "56x56x64 -> 28x28x128, 3x3, stride 2, pad 1",
                     "plan": conv.plan_multi_strided(C2, W2, W2, K2, M2, P2, S2, prec, N)}
            if prec != "fp32":
                entry["tensor_frac"] = round(tflops / (pk["bf16_tflops"] * (0.5 if prec == "tf32" else 1.0)), 4)
            out[f"{prec}_n{N}_s2"] = entry
    return out


def _strong_sweep(args, conv, dev, stream, world, rank, cacheI):
    import torch
    import torch.distributed as dist
    c = synth.SHARD_SWEEP
    out = {}
    for prec in args.precision.split(","):
        Mloc = c["M"] // world
        dt = torch.bfloat16 if prec == "bf16" else torch.float32
        I = cacheI[(c["C"], c["Wx"], c["Wy"])].to(dt).contiguous()
        F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F + 999 + rank, (Mloc, c["C"], c["K"], c["K"]))).to(dev, dt)
        Ho, Wo = c["Wy"] - c["K"] + 1, c["Wx"] - c["K"] + 1
        O = torch.empty((Mloc, Ho, Wo), device=dev)
        reps = 20
        with torch.cuda.stream(stream):
            for _ in range(3):
                conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], F, c["K"], Mloc, O, prec, stream.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            stream.synchronize()
            e0.record(stream)
            for _ in range(reps):
                conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], F, c["K"], Mloc, O, prec, stream.cuda_stream)
            e1.record(stream)
            stream.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / reps
        if world > 1:
            tt = torch.tensor([us], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            us = float(tt.item())
        flop = 2.0 * c["M"] * c["C"] * c["K"] ** 2 * Ho * Wo
        out[prec] = {"us_max_rank": round(us, 3), "gflops_total": round(flop / (us * 1e-6) / 1e9, 1),
                     "filters_per_rank": Mloc}
        if world > 1:
            # G2 of SURVEY §8(a): the path's only collective, the all-gather of
            # the filter-sharded O (NCCL over NVLink), timed with and without
            # the convolution (device events, max over ranks)
            try:
                from paper_2212_00404_b200.shard import allgather_output
                with torch.cuda.stream(stream):
                    for _ in range(3):
                        allgather_output(O, c["M"])
                    dist.barrier()
                    stream.synchronize()
                    e0.record(stream)
                    for _ in range(reps):
                        allgather_output(O, c["M"])
                    e1.record(stream)
                    stream.synchronize()
                    ag = 1e3 * e0.elapsed_time(e1) / reps
                    dist.barrier()
                    stream.synchronize()
                    e0.record(stream)
                    for _ in range(reps):
                        conv.conv_multi_ex(I, c["C"], c["Wx"], c["Wy"], F, c["K"], Mloc, O, prec, stream.cuda_stream)
                        allgather_output(O, c["M"])
                    e1.record(stream)
                    stream.synchronize()
                    both = 1e3 * e0.elapsed_time(e1) / reps
                tt = torch.tensor([ag, both], device=dev)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                out[prec]["allgather_us_max_rank"] = round(float(tt[0]), 3)
                out[prec]["conv_plus_allgather_us_max_rank"] = round(float(tt[1]), 3)
                out[prec]["allgather_bytes_per_rank_recv"] = int(4 * (c["M"] - Mloc) * Ho * Wo)
            except Exception as exc:  # reported, never fatal for the bench line
                out[prec]["allgather_error"] = repr(exc)[:200]
    return out


def _cudnn_context(args, calls, dev, stream, capture, pk):
    """cuDNN (torch conv2d, benchmark=True) on the same shapes and inputs, timed
    with the same per-layer back-to-back graph protocol as layers_b2b."""
    import torch
    torch.backends.cudnn.benchmark = True

    def fn(c):
        torch.backends.cudnn.allow_tf32 = c["prec"] == "tf32"
        I = c["I"][None] if c["kind"] == "multi" else c["I"][None, None]
        F = c["F"] if c["kind"] == "multi" else c["F"][:, None]
        return torch.nn.functional.conv2d(I, F)

    with torch.cuda.stream(stream):
        for c in calls:          # algorithm selection outside capture
            fn(c)
        stream.synchronize()
        lay = _layer_b2b(calls, None, capture, stream, dev, pk, cudnn_fn=fn)
    torch.backends.cudnn.allow_tf32 = True
    tot_us = sum(v["us"] for v in lay.values())
    tot_flop = sum(c["flop"] for c in calls)
    return {"engine": "torch.nn.functional.conv2d -> cuDNN %s, benchmark=True, fp32 layers with "
                      "allow_tf32=False; per-layer back-to-back graph replay (output not rotated)"
                      % torch.backends.cudnn.version(),
            "value": round(tot_flop / (tot_us * 1e-6) / 1e9, 2), "unit": UNIT,
            "ms_per_step_sum_of_layers": round(tot_us / 1e3, 4),
            "layers_us": {k: v["us"] for k, v in lay.items()}}


def _e2e(args, conv, calls, stream, world, rank, dev):
    """Same metric through the public host-buffer API (conv_*_host_async): per
    layer, H2D of I and F from pinned memory, the kernel(s), D2H of O; calls
    round-robin over --e2e-streams streams in an order that interleaves
    output-heavy and input-heavy layers; the host waits once per step."""
    import torch
    import torch.distributed as dist
    steps = max(1, min(args.steps, args.e2e_steps))
    host = []
    for c in calls:
        Ih = c["I"].cpu().pin_memory()
        Fh = c["F"].cpu().pin_memory()
        Oh = torch.empty(tuple(c["O"].shape), dtype=torch.float32).pin_memory()
        host.append((Ih, Fh, Oh))
    h2d = sum(Ih.numel() * Ih.element_size() + Fh.numel() * Fh.element_size() for Ih, Fh, _ in host)
    d2h = sum(Oh.numel() * 4 for _, _, Oh in host)
    # the asynchronous host entry points on --e2e-streams streams (round robin
    # per call): one call's device->host copy overlaps the next calls'
    # host->device copies and kernels (several streams, so a copy queued behind
    # its stream's previous device->host copy does not block the copy engine's
    # queue for the others); one host synchronisation per step
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(args.e2e_streams - 1)]
    done = [torch.cuda.Event() for _ in streams]
    # issue order: the layers of a step are independent problems, so the caller
    # interleaves output-heavy calls (224x224 maps) with input-heavy ones (big
    # filter banks) to keep both PCIe directions busy at once
    net = [Oh.numel() * 4 - Ih.numel() * Ih.element_size() - Fh.numel() * Fh.element_size()
           for Ih, Fh, Oh in host]
    by = sorted(range(len(calls)), key=lambda i: net[i])
    order = []
    lo, hi = 0, len(by) - 1
    while lo <= hi:
        order.append(by[hi]); hi -= 1
        if lo <= hi:
            order.append(by[lo]); lo += 1
    if not args.e2e_interleave:
        order = list(range(len(calls)))

    def one_step():
        for i, j in enumerate(order):
            c, (Ih, Fh, Oh) = calls[j], host[j]
            sh = streams[i % len(streams)].cuda_stream
            if c["kind"] == "single":
                conv.conv_single_host_async(Ih, c["Wx"], c["Wy"], Fh, c["K"], c["M"], Oh, sh)
            else:
                conv.conv_multi_host_async(Ih, c["C"], c["Wx"], c["Wy"], Fh, c["K"], c["M"], Oh, c["prec"], sh)
        for st, ev in zip(streams[1:], done[1:]):
            ev.record(st)
            stream.wait_event(ev)

    one_step()                                   # warm-up (pool, workspaces)
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        one_step()
        stream.synchronize()                     # results on the host once per step
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    flop = world * sum(c["flop"] for c in calls)
    return {"value": round(flop / (ms * 1e-3) / 1e9, 2), "unit": UNIT, "ms_per_step": round(ms, 3),
            "steps": steps, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": f"conv_single_host_async / conv_multi_host_async (pinned host buffers, "
                   f"{len(streams)} streams round robin per call, "
                   f"{'output-/input-heavy calls interleaved' if args.e2e_interleave else 'suite order'}, "
                   f"one host synchronisation per step)"}


# ----------------------------------------------------------------------------- CPU oracle
def _oracle_sample(calls, budget_s, threads):
    """Run the oracle on a bounded sample (the first m_s filters of every layer,
    m_s scaled so the whole sample takes ~budget_s).  Returns (flop, seconds, desc)."""
    import oracle
    used = oracle.set_threads(threads)
    # calibrate: ns per MAC on this host with these threads
    I = synth.uniform01(1, (64, 28, 28))
    F = synth.uniform_pm1(2, (16, 64, 3, 3))
    t = time.perf_counter()
    oracle.conv_multi(I, F)
    dt = time.perf_counter() - t
    ns_per_mac = dt / (16 * 64 * 9 * 26 * 26) * 1e9
    total_mac = sum(c["flop"] / 2 for c in calls)
    frac = min(1.0, budget_s / max(1e-9, total_mac * ns_per_mac * 1e-9))
    flop, secs, nfil = 0.0, 0.0, 0
    cache = {}
    for c in calls:
        ms = max(1, int(round(c["M"] * frac)))
        key = (c["C"], c["Wx"], c["Wy"])
        if key not in cache:
            cache[key] = synth.uniform01(synth.SEED_I, (c["C"], c["Wy"], c["Wx"]))
        Fh = synth.uniform_pm1(synth.SEED_F + c["cfg_index"], (ms, c["C"], c["K"], c["K"]))
        t = time.perf_counter()
        oracle.conv_multi(cache[key], Fh)
        secs += time.perf_counter() - t
        flop += 2.0 * ms * c["C"] * c["K"] ** 2 * c["Ho"] * c["Wo"]
        nfil += ms
    desc = (f"oracle (fp64 C, OpenMP) on the first ceil({frac:.4f}*M) filters of each of the "
            f"{len(calls)} layers of one step ({nfil} filters, {flop / 1e9:.2f} GFLOP)")
    return flop, secs, desc, used


def _cpu_baseline(calls, budget_s):
    threads = os.cpu_count() or 1
    flop, secs, desc, used = _oracle_sample(calls, budget_s, threads)
    return {"value": round(flop / secs / 1e9, 4), "unit": UNIT, "cores": used, "kind": "oracle",
            "sample": desc, "seconds": round(secs, 2)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    precisions = tuple(args.precision.split(","))
    calls = suite(1, 0, precisions)
    budget = max(1.0, args.ref_step_seconds)
    for _ in range(args.warmup):
        _oracle_sample(calls, min(budget, 2.0), os.cpu_count() or 1)
    flops, secs = 0.0, 0.0
    for _ in range(args.steps):
        f, s, desc, used = _oracle_sample(calls, budget, os.cpu_count() or 1)
        flops += f
        secs += s
    value = flops / secs / 1e9
    res = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * secs / args.steps, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "impl": "reference",
           "dtype": "f64 (oracle)", "data": "synthetic (splitmix64 seeded)",
           "config": {"workload": WORKLOAD, "precisions": list(precisions), "batch": 1},
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": used, "kind": "oracle",
                            "sample": desc},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="fp32,tf32,bf16")
    ap.add_argument("--cudnn", type=int, default=1)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-streams", type=int, default=8)
    ap.add_argument("--e2e-interleave", type=int, default=1)
    ap.add_argument("--batched", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=8.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
