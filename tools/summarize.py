"""Print a compact summary of bench JSON lines found in log files."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        c = d.get("calibration", {})
        print(f"{f}: N={d['n_gpus']} value={d['value']:.3f} ms/step={d['ms_per_step']:.4f} "
              f"a={c.get('a_us', 0):.2f}us b={c.get('b_ps_per_byte', 0):.3f}ps/B e2e={d['e2e']['value']:.2f}")
        for k, v in d.get("strategies", {}).items():
            print(f"   {k:14s} med={v['iter_ms_median']:.4f} p10={v['iter_ms_p10']:.4f} p90={v['iter_ms_p90']:.4f} "
                  f"pred={v['predicted_ms']:.4f} groups={v['groups']}")
        r = d.get("roofline", {})
        if r:
            print(f"   roofline {r['bound']} achieved={r['achieved']:.1f} frac={r['frac']:.4f} "
                  f"kernel_ms/iter={r['kernel_ms_per_iter']:.3f} launches={r['launches_per_iter']}")
        if d.get("bus_gbs"):
            print("   bus", {k: {kk: round(vv, 1) for kk, vv in v.items()} if isinstance(v, dict) else round(v, 1)
                          for k, v in d["bus_gbs"].items()})
        if d.get("cpu_baseline"):
            print("   cpu", d["cpu_baseline"]["value"], d["clocks"])
