"""Summarise an ncu --set full report (tools only): per kernel, duration,
DRAM bytes / throughput, SOL %, issue activity and the top warp-stall
reasons, plus the algorithmic-bytes roofline if ALG_BYTES is given.
usage: python tools/ncu_summary.py report.ncu-rep [alg_bytes_per_launch ...]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
alg = [float(x) for x in sys.argv[2:]]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
col = {name: i for i, name in enumerate(h)}


def get(r, name):
    i = col.get(name)
    return (r[i], units[i]) if i is not None else ("n/a", "")


def num(r, name):
    v, u = get(r, name)
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "usecond": 1e-6, "nsecond": 1e-9,
             "msecond": 1e-3, "us": 1e-6, "ns": 1e-9}.get(u, 1.0)
    return x * scale


stalls = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for k, r in enumerate(data):
    name = get(r, "Kernel Name")[0]
    dur = num(r, "gpu__time_duration.sum")
    rd, wr = num(r, "dram__bytes_read.sum"), num(r, "dram__bytes_write.sum")
    print(f"## kernel: {name[:150]}")
    print(f"grid {get(r, 'launch__grid_size')[0]} x block {get(r, 'launch__block_size')[0]}, "
          f"regs/thread {get(r, 'launch__registers_per_thread')[0]}, "
          f"dyn smem {get(r, 'launch__shared_mem_per_block_dynamic')[0]} {get(r, 'launch__shared_mem_per_block_dynamic')[1]}")
    if dur:
        print(f"duration                     {dur * 1e6:10.2f} us")
    if rd is not None and wr is not None and dur:
        print(f"dram read + write            {(rd + wr) / 1e6:10.2f} MB  ({(rd + wr) / dur / 1e9:.0f} GB/s)")
    if k < len(alg) and dur:
        print(f"algorithmic bytes            {alg[k] / 1e6:10.2f} MB  ({alg[k] / dur / 1e9:.0f} GB/s)")
    for m in ["gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
              "dram__throughput.avg.pct_of_peak_sustained_elapsed",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed",
              "smsp__issue_active.avg.pct_of_peak_sustained_active",
              "sm__warps_active.avg.pct_of_peak_sustained_active",
              "lts__t_sector_hit_rate.pct"]:
        v, u = get(r, m)
        print(f"{m:60s} {v:>10s} {u}")
    top = sorted(((num(r, c) or 0.0, c) for c in stalls), reverse=True)[:5]
    print("top stalls (warps per issue-active cycle): " +
          ", ".join(f"{c.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={v:.2f}"
                    for v, c in top))
    print()
