"""Per-layer markdown report (ours vs cuDNN, roofline fraction) from a bench JSON."""
import json, sys
r = json.load(open(sys.argv[1]))
L = r.get("layers_b2b") or {}
cu = (r.get("cudnn_context") or {}).get("layers_us", {})
out = []
out.append(f"# bench report ({sys.argv[1]})\n")
out.append(f"step: {r['ms_per_step']:.4f} ms, value {r['value']:.0f} {r['unit']}, n_gpus {r['n_gpus']}, clocks {r['clocks']}\n")
out.append(f"roofline (dominant kernel group): {json.dumps(r['roofline'])}\n")
out.append(f"cuDNN context: {json.dumps({k: v for k, v in (r.get('cudnn_context') or {}).items() if k != 'layers_us'})}\n")
out.append(f"cpu_baseline: {json.dumps(r.get('cpu_baseline'))}\n")
out.append(f"e2e: {json.dumps(r.get('e2e'))}\n")
out.append("\n| kernel group | launches | us/step | share | achieved | frac of peak |\n|---|---|---|---|---|---|\n")
for k, v in r["kernels"].items():
    out.append(f"| {k} | {v['launches_per_step']} | {v['us_per_step']:.1f} | {v['share']:.3f} | {v['achieved']} {v['unit']} | {v['frac']:.3f} |\n")
out.append("\n| layer | ours us | GFLOP/s | bound | frac | cuDNN us | speedup |\n|---|---|---|---|---|---|---|\n")
tot_o = tot_c = 0.0
for k, v in L.items():
    c = cu.get(k)
    tot_o += v["us"]
    if c: tot_c += c
    sp = f"{c / v['us']:.2f}x" if c else "-"
    out.append(f"| {k} | {v['us']:.2f} | {v['gflops']:.0f} | {v['bound']} | {v['frac']:.3f} | {c if c else '-'} | {sp} |\n")
out.append(f"\nsum of per-layer times: ours {tot_o / 1e3:.3f} ms, cuDNN {tot_c / 1e3:.3f} ms\n")
open(sys.argv[2], "w").write("".join(out))
print("".join(out[:8]))
