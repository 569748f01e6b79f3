"""KM-SIMT configuration sweep on the GPU (calibrates the planner's model).

For each multi-channel bench layer: time the planner's choice and forced
(tile, split, mode) configurations via B200CONV_SIMT_FORCE, 20 launches per
CUDA graph, and check each result against cuDNN fp32 (allow_tf32 off).
usage: simt_sweep.py [layer-substring] [--full]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import torch.nn.functional as Fn

import synth
from paper_2212_00404_b200 import conv

torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False
want = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else ""
full = "--full" in sys.argv
dev = torch.device("cuda", 0)
TILES = [(128, 128), (64, 256), (256, 64), (256, 48), (128, 96), (64, 192), (256, 32), (128, 64), (64, 128)]


STREAM = None


def time_cfg(I, F, O, L, reps=20):
    global STREAM
    STREAM = STREAM or torch.cuda.Stream()
    s = STREAM
    conv.conv_multi_ex(I, L["C"], L["Wx"], L["Wy"], F, L["K"], L["M"], O, "fp32", s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            conv.conv_multi_ex(I, L["C"], L["Wx"], L["Wy"], F, L["K"], L["M"], O, "fp32",
                               torch.cuda.current_stream().cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1000 / reps)
    return best


out = []
# the per-rank shards of the strong-scaled configs[4] sweep (M / G filters, G = 2, 4, 8)
SHARDS = [dict(synth.SHARD_SWEEP, name=f"shard{g}_14x14_c512_m{4096 // g}_k3", M=4096 // g) for g in (2, 4, 8)]
for L in synth.MULTI_LAYERS + [synth.SHARD_SWEEP] + SHARDS:
    if want not in L["name"]:
        continue
    I = torch.from_numpy(synth.uniform01(synth.SEED_I, (L["C"], L["Wy"], L["Wx"]))).to(dev)
    F = torch.from_numpy(synth.uniform_pm1(synth.SEED_F, (L["M"], L["C"], L["K"], L["K"]))).to(dev)
    ref = Fn.conv2d(I[None], F)[0]
    O = torch.empty_like(ref)
    scale = float(ref.abs().max())
    cfgs = [None]
    C = L["C"]
    if "--dense" in sys.argv:
        import simt_model
        for ti, (BM, BN, TN) in enumerate(simt_model.TILES):
            seen = set()
            for S in range(1, min(C, 96) + 1):
                cb, cps = simt_model.split(C, S, BM, BN, L["K"])
                Se = -(-C // cps)
                if Se in seen:
                    continue
                seen.add(Se)
                for ws in (0, 1):
                    if (ws == 0 and Se > 16) or (ws == 1 and Se == 1):
                        continue
                    cfgs.append((ti, S, ws))
    Ss = [] if "--dense" in sys.argv else sorted(
        {s for s in (1, 2, 3, 4, 6, 8, 10, 12, 14, 16, 20, 24, 32, 40, 48, 64, 96) if s <= C})
    for ti in range(len(TILES) if Ss else 0):
        for S in Ss:
            for ws in (0, 1):
                if (ws == 0 and S > 16) or (ws == 1 and S == 1):
                    continue
                if not full and ws == 0 and S not in (1, 4, 8, 16):
                    continue
                cfgs.append((ti, S, ws))
    for cfg in cfgs:
        if cfg is None:
            os.environ.pop("B200CONV_SIMT_FORCE", None)
        else:
            os.environ["B200CONV_SIMT_FORCE"] = "%d,%d,%d" % cfg
        O.fill_(float("nan"))
        try:
            us = time_cfg(I, F, O, L)
        except Exception as e:   # noqa: BLE001
            out.append(dict(layer=L["name"], cfg=cfg, err=str(e)[:80]))
            continue
        conv.conv_multi_ex(I, L["C"], L["Wx"], L["Wy"], F, L["K"], L["M"], O, "fp32", 0)
        torch.cuda.synchronize()
        err = float((O - ref).abs().max()) / scale
        p = conv.plan_multi(L["C"], L["Wx"], L["Wy"], L["K"], L["M"], "fp32")
        rec = dict(layer=L["name"], cfg=cfg, us=round(us, 2), err=err,
                   plan=[p["tile_m"], p["tile_n"], p["grid_x"], p["launches"]])
        out.append(rec)
    os.environ.pop("B200CONV_SIMT_FORCE", None)
    rows = [r for r in out if r["layer"] == L["name"] and "us" in r]
    auto = rows[0]
    best = sorted(rows, key=lambda r: r["us"])[:6]
    print(L["name"], "auto", auto["us"], auto["plan"], "err %.2e" % auto["err"], flush=True)
    for r in best:
        print("    best", r["cfg"], r["us"], r["plan"], "err %.2e" % r["err"], flush=True)
    bad = [r for r in rows if not (r["err"] < 1e-5)]
    if bad:
        print("    BAD", [(r["cfg"], r["err"]) for r in bad][:8], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(os.environ.get("SWEEP_OUT", "gpurun_out/simt_sweep.json"), "w"), indent=0)
