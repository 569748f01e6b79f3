import json, sys
r = json.load(open(sys.argv[1]))
for k in ['value', 'ms_per_step', 'roofline', 'clocks', 'e2e', 'cpu_baseline', 'strong_sweep']:
    print(k, json.dumps(r.get(k))[:600])
for k, v in r['kernels'].items():
    print(f"  {k:22s} {v['us_per_step']:9.1f}us n={v['launches_per_step']:3d} avg={v['avg_launch_us']:8.2f} share={v['share']:.3f} frac={v['frac']:.3f} {v['achieved']} {v['unit']}")
cu = (r.get('cudnn_context') or {}).get('layers_us', {})
print('cudnn', json.dumps({k: v for k, v in (r.get('cudnn_context') or {}).items() if k != 'layers_us'}))
L = r.get('layers_b2b') or {}
print('sum b2b ms', sum(v['us'] for v in L.values()) / 1e3, ' cudnn sum', sum(cu.values()) / 1e3)
filt = sys.argv[2] if len(sys.argv) > 2 else ''
for k, v in L.items():
    if filt and filt not in k: continue
    print(f"{k:42s} {v['us']:9.2f}us {v['gflops']:9.1f}GF/s {v['bound']:6s} frac={v['frac']:.3f}  cudnn={cu.get(k, float('nan')):8.2f}us")
