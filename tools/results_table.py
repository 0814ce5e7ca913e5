"""Markdown tables of bench results from scale logs (tools only).
usage: python tools/results_table.py LOG_DIR [traces...]"""
import json
import os
import sys

d = sys.argv[1]
traces = sys.argv[2:] or ["googlenet", "resnet50", "resnet152", "densenet201", "inception_v4", "bert_large"]
print("| trace | N | worker-iters/s (e2e) | MG-WFBP ms (pred.) | WFBP ms | single-buffer ms | groups | plan a µs / b ps/B "
      "| tail µs | drain roofline | scaling eff. |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for t in traces:
    base = None
    for n in (1, 2, 4, 8):
        p = os.path.join(d, f"scale_{t}_n{n}.log")
        if not os.path.exists(p):
            continue
        lines = [l for l in open(p) if l.startswith("{")]
        if not lines:
            continue
        r = json.loads(lines[-1])
        s = r["strategies"]
        if n == 1:
            base = r["value"]
        eff = r["value"] / (n * base) if base else float("nan")
        tail = s["mgwfbp"].get("device_tail_us", float("nan"))
        cal = r["calibration"].get("plan_model", r["calibration"])
        roof = r.get("roofline") or {}
        rf = f"{roof['frac']:.2f} of {'HBM' if n == 1 else '900'}" if roof.get("frac") else "-"
        print(f"| {t} | {n} | {r['value']:.2f} ({r['e2e']['value']:.2f}) | {s['mgwfbp']['iter_ms_median']:.3f} "
              f"({s['mgwfbp']['predicted_ms']:.3f}) | "
              f"{s['wfbp']['iter_ms_median']:.3f} | {s['single_buffer']['iter_ms_median']:.3f} | "
              f"{s['mgwfbp']['groups']} | {cal['a_us']:.2f} / {cal['b_ps_per_byte']:.3f} | "
              f"{tail:.1f} | {rf} | {eff:.4f} |")
