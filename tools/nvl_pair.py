"""Two-process fused all-reduce WITHOUT torch.distributed / NCCL (tools
only): the CUDA IPC handles and the start barrier go through files, so
rank 0 can run under ncu while rank 1 runs free (no NCCL kernel is ever
serialised against the peer). Used by tools/ncu_nvlink.sh.

usage: python tools/nvl_pair.py RANK DIR [SIZE_MB] [ALGO]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1912_09268_b200 import gradsched as gs  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402


def file_allgather(d, tag, rank, P, data: bytes):
    with open(os.path.join(d, f"{tag}.{rank}.tmp"), "wb") as f:
        f.write(data)
    os.rename(os.path.join(d, f"{tag}.{rank}.tmp"), os.path.join(d, f"{tag}.{rank}"))
    out = []
    for q in range(P):
        p = os.path.join(d, f"{tag}.{q}")
        t0 = time.time()
        while not os.path.exists(p):
            if time.time() - t0 > 120:
                raise TimeoutError(p)
            time.sleep(0.01)
        with open(p, "rb") as f:
            out.append(f.read())
    return out


def main():
    rank, d = int(sys.argv[1]), sys.argv[2]
    S = (int(sys.argv[3]) if len(sys.argv) > 3 else 64) << 20
    algo = sys.argv[4] if len(sys.argv) > 4 else "twoshot"
    P = 2
    os.makedirs(d, exist_ok=True)
    torch.cuda.set_device(rank)
    comm = rt.Comm(rank, P, rank, S + (1 << 20), exchange=lambda b: file_allgather(d, "ipc", rank, P, b))
    g = torch.empty(S // 4, device="cuda").uniform_(-1, 1)
    w = torch.zeros(S // 4, device="cuda")
    dp = rt.DevicePlan(comm, [g], [w], gs.MergePlan.all_normal(1))
    for _ in range(3):
        dp.group_allreduce(0, 0.0, rt.SGD, algo)
    torch.cuda.synchronize()
    file_allgather(d, "go", rank, P, b"1")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dp.group_allreduce(0, 0.0, rt.SGD, algo)  # the 4th launch: profiled on rank 0
    e1.record()
    e1.synchronize()
    print(f"rank {rank}: {S >> 20} MiB {algo} launch {e0.elapsed_time(e1) * 1e3:.1f} us "
          f"(failed={comm.failed()})", flush=True)
    file_allgather(d, "done", rank, P, b"1")
    dp.close()
    comm.close()


if __name__ == "__main__":
    main()
