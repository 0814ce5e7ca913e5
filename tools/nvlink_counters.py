"""NVLink byte counters around the real cross-GPU merged all-reduce (tools only).

torchrun P ranks, one per GPU. For each size S and algorithm, every rank runs
K standalone launches of the fused group kernel (one group of S bytes, real
IPC peers over NVLink) and reads its GPU's NVLink counters (NVML field
values, summed over links) before and after:

  tx, rx bytes per launch per rank  vs  algorithmic bus bytes
     two-shot 2(P-1)/P * S   one-shot (P-1) * S        (per direction)

plus CUDA-event time per launch (max over ranks) -> bus GB/s = 2(P-1)/P*S/t.
Counters: NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX (KiB, payload) and
NVML_FI_DEV_NVLINK_COUNT_XMIT/RCV_BYTES when the driver has them.

env: SIZES_MB (default 16,64,256), ALGOS (twoshot,oneshot), K (20),
     KNOBS "chunk_tiles,min_chunks,small_tile_max_KiB" (library defaults)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml as nv  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1912_09268_b200 import dist as D  # noqa: E402
from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

FIELDS = {
    "data_tx_kib": "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX",
    "data_rx_kib": "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
    "raw_tx_kib": "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX",
    "raw_rx_kib": "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX",
    "xmit_bytes": "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES",
    "rcv_bytes": "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES",
}


DIAG = {}


def read_counters(h, links):
    """Sum of each field over the links (scopeId = link), or the device-wide
    value (scopeId = UINT_MAX) when per-link reads are refused."""
    out = {}
    for key, name in FIELDS.items():
        fid = getattr(nv, name, None)
        if fid is None:
            DIAG[key] = "no constant"
            continue
        total, ok, codes = 0, False, set()
        for scope in list(links) + [0xFFFFFFFF]:
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            except (nv.NVMLError, TypeError) as e:
                codes.add(repr(e)[:60])
                continue
            codes.add(int(v.nvmlReturn))
            if v.nvmlReturn != 0:
                continue
            if scope == 0xFFFFFFFF:
                if not ok:
                    total, ok = v.value.ullVal, True
                break
            total += v.value.ullVal
            ok = True
        DIAG[key] = sorted(map(str, codes))
        if ok:
            out[key] = total
    return out


def smi_counters(idx):
    """`nvidia-smi nvlink -gt d` (per-link data tx/rx KiB) as raw text."""
    import subprocess

    try:
        return subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(idx)], capture_output=True,
                              text=True, timeout=30).stdout
    except Exception as e:  # noqa: BLE001
        return f"unavailable: {e}"


def smi_total(text):
    """Sum of the Tx / Rx KiB numbers in smi_counters() output."""
    import re

    tx = rx = 0
    for line in text.splitlines():
        m = re.search(r"(Tx|Rx)\D*?(\d+)\s*KiB", line)
        if m:
            if m.group(1) == "Tx":
                tx += int(m.group(2))
            else:
                rx += int(m.group(2))
    return tx, rx


def main():
    rank, P, local = D.init("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ
                                      else int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local]))
    links = []
    for link in range(18):
        try:
            if nv.nvmlDeviceGetNvLinkState(h, link) == nv.NVML_FEATURE_ENABLED:
                links.append(link)
        except nv.NVMLError:
            pass
    sizes = [int(s) << 20 for s in os.environ.get("SIZES_MB", "16,64,256").split(",")]
    K = int(os.environ.get("K", "20"))
    comm = rt.Comm(rank, P, local, max(sizes) + (1 << 20))
    if os.environ.get("KNOBS"):
        v = [int(x) for x in os.environ["KNOBS"].split(",")]
        comm.set_chunk_tiles(v[0], v[1])
        comm.set_small_tile_max(v[2] << 10)
    rows = []
    for S in sizes:
        n = S // 4
        g = torch.empty(n, device=dev).uniform_(-1, 1)
        w = torch.zeros(n, device=dev)
        dp = rt.DevicePlan(comm, [g], [w], gs.MergePlan.all_normal(1))
        for algo in os.environ.get("ALGOS", "twoshot,oneshot").split(","):
            for _ in range(3):
                dp.group_allreduce(0, 0.0, rt.SGD, algo)
            torch.cuda.synchronize()
            D.barrier()
            gidx = torch.cuda.current_device() if "CUDA_VISIBLE_DEVICES" not in os.environ else \
                int(os.environ["CUDA_VISIBLE_DEVICES"].split(",")[local])
            s0 = smi_counters(gidx)
            c0 = read_counters(h, links)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
            import time
            h0 = time.perf_counter()
            ev[0].record()
            for k in range(K):
                dp.group_allreduce(0, 0.0, rt.SGD, algo)
                ev[k + 1].record()
            h1 = time.perf_counter()
            ev[K].synchronize()
            c1 = read_counters(h, links)
            s1 = smi_counters(gidx)
            per = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(K))
            t = D.max_over_ranks(per[len(per) // 2] / 1e3, dev)  # median launch
            d = {k: (c1[k] - c0[k]) / K for k in c1 if k in c0}
            algo_bytes = (2 * (P - 1) / P if algo == "twoshot" else (P - 1)) * S
            row = {"rank": rank, "P": P, "bytes": S, "algo": algo, "us": t * 1e6,
                   "bus_gbs": 2 * (P - 1) / P * S / t / 1e9, "algorithmic_bytes_per_dir": algo_bytes,
                   "per_launch": d, "links": len(links), "host_us_per_launch": (h1 - h0) / K * 1e6,
                   "launch_us_min_max": [per[0] * 1e3, per[-1] * 1e3], "nvml": dict(DIAG)}
            (tx0, rx0), (tx1, rx1) = smi_total(s0), smi_total(s1)
            row["smi_tx_bytes_per_launch"] = (tx1 - tx0) * 1024 / K
            row["smi_rx_bytes_per_launch"] = (rx1 - rx0) * 1024 / K
            if rank == 0 and S == sizes[0]:
                row["smi_sample"] = s1[:1500]
            if "data_tx_kib" in d:
                row["tx_over_algorithmic"] = d["data_tx_kib"] * 1024 / algo_bytes
                row["rx_over_algorithmic"] = d["data_rx_kib"] * 1024 / algo_bytes
            rows.append(row)
        dp.close()
        del g, w
    allrows = [None] * P
    dist.all_gather_object(allrows, rows)
    if rank == 0:
        for rr in allrows:
            for r in rr:
                print(json.dumps(r), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
