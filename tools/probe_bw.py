"""Merged all-reduce bus bandwidth probe at P ranks (torchrun, tools only):
fused engine kernel (one-shot / two-shot, CTA counts) vs NCCL, large sizes.

Tool-level env (the library itself reads no environment): SIZES_KB / SIZES_MB,
ALGOS, CTAS, REPS, DTYPE, STANDALONE, PROTOS (stream,chunked), and KNOBS = ";"-separated
"chunk_tiles,min_chunks,small_tile_max_KiB[,ll_max_KiB[,credit_batch,ag_batch]]" configurations set
through the C-ABI setters (default: the library defaults)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1912_09268_b200 import dist as D  # noqa: E402
from paper_1912_09268_b200 import runtime as rt  # noqa: E402

rank, P, local = D.init("nccl")
dev = torch.device("cuda", local)
sizes = ([int(s) << 10 for s in os.environ["SIZES_KB"].split(",")] if "SIZES_KB" in os.environ
         else [int(s) << 20 for s in os.environ.get("SIZES_MB", "1,4,16,64,256").split(",")])
comm = rt.Comm(rank, P, local, max(sizes) + (1 << 20))
f = 2 * (P - 1) / P
out = []
base = comm.tuning()
knobs = [k for k in os.environ.get("KNOBS", "").split(";") if k] or [""]
for knob, proto in [(k, p) for p in os.environ.get("PROTOS", "stream").split(",") for k in knobs]:
    comm.set_protocol(proto)
    tag = f" {proto}"
    if knob:
        v = [int(x) for x in knob.split(",")]
        comm.set_chunk_tiles(v[0], v[1])
        comm.set_small_tile_max(v[2] << 10)
        comm.set_ll_max((v[3] << 10) if len(v) > 3 else base["ll_max"])
        cb, ab = (v[4], v[5]) if len(v) > 5 else (8, 4)
        comm.set_stream_batches(cb, ab)
        tag += f" [ct={v[0]} mc={v[1]} stm={v[2]}K cb={cb} ab={ab}]"
    for algo in os.environ.get("ALGOS", "oneshot,twoshot").split(","):
        for ctas in [int(c) for c in os.environ.get("CTAS", "64,140").split(",")]:
            m = comm.calibrate_engine(sizes, warmup=2, reps=int(os.environ.get("REPS", "10")), algo=algo,
                                      engine_ctas=ctas, dtype=1 if os.environ.get("DTYPE") == "bf16" else 0)
            t = torch.tensor([x.time_sec for x in m], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out.append((f"engine {algo} ctas={ctas}{tag}", [f * s / tt / 1e9 for s, tt in zip(sizes, t.tolist())],
                        [tt * 1e6 for tt in t.tolist()]))
standalone = [a for a in os.environ.get("STANDALONE", "twoshot").split(",") if a]
if "nvls" in standalone:  # NVLS_CHUNKS: tiles per pipelined chunk of the NVLS kernel
    comm.enable_nvls(0, 4)
runs = [(a, c, k) for a in standalone for c in ([int(x) for x in os.environ.get("NVLS_CHUNKS", "4").split(",")]
                                                  if a == "nvls" else [0])
        for k in ([int(x) for x in os.environ.get("NVLS_SKIP", "0").split(",")] if a == "nvls" else [0])]
for algo, chunk, skip in runs:
    if algo == "nvls":
        comm.set_nvls(0, chunk)
        from paper_1912_09268_b200 import _lib
        rt.check(_lib.mgw_comm_set_nvls_skip(comm.handle, skip))
    m = comm.calibrate(sizes, warmup=2, reps=int(os.environ.get("SREPS", "5")), algo=algo)
    t = torch.tensor([x.time_sec for x in m], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    name = f"standalone {algo}" + (f" chunk={chunk} skip={skip}" if algo == "nvls" else " (grid=occ*SMs)")
    out.append((name, [f * s / tt / 1e9 for s, tt in zip(sizes, t.tolist())], [tt * 1e6 for tt in t.tolist()]))
nccl = []
for s in sizes:
    x = torch.ones(s // 4, device=dev)
    for _ in range(3):
        dist.all_reduce(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        dist.all_reduce(x)
    e1.record()
    e1.synchronize()
    tt = torch.tensor([e0.elapsed_time(e1) / 10 / 1e3], dtype=torch.float64, device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    nccl.append(tt.item())
out.append(("nccl", [f * s / tt / 1e9 for s, tt in zip(sizes, nccl)], [tt * 1e6 for tt in nccl]))
if rank == 0:
    print(f"P={P} sizes(KiB)={[s >> 10 for s in sizes]}  bus GB/s (time us)")
    for name, bw, us in out:
        print(f"  {name:44s}", "  ".join(f"{b:7.1f} ({u:8.1f})" for b, u in zip(bw, us)), flush=True)
comm.close()
dist.destroy_process_group()
