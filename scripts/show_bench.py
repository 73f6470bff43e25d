import json, sys
for fn in sys.argv[1:]:
    l = [x for x in open(fn) if x.startswith('{')]
    if not l:
        print(fn, "NO JSON"); continue
    d = json.loads(l[-1])
    r = d.get('roofline') or {}
    print(fn, f"value={d['value']:.3e} ms/step={d['ms_per_step']:.3f} stepfrac={r.get('step_frac',0):.3f} dom={r.get('kernel')} frac={r.get('frac',0):.3f}",
          "e2e", d.get('e2e') and f"{d['e2e']['value']:.3e}", "cpu", d.get('cpu_baseline') and f"{d['cpu_baseline']['value']:.3e} ({d['cpu_baseline']['cores']} cores)", d.get('clocks'))
    for k, v in (d.get('kernels') or {}).items():
        print("   ", k, f"{v['avg_ms']:.3f} ms", f"frac={v.get('frac', 0):.3f}", f"share={v['share_of_step']:.3f}")
