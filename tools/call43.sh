# 4-GPU: NVLS multicast probe (P=2,4) + NCCL NVLS check
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ll; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1; nvidia-smi -q | grep -i -A3 "fabric" > $O/fabric.txt 2>&1
for P in 2 4; do timeout 300 ./tools/nvls_probe $P > $O/nvls_p$P.log 2>&1; echo "nvls P=$P rc=$?"; head -8 $O/nvls_p$P.log; grep "size=16384\|size=65536\|size=262144 \|size=1048576 " $O/nvls_p$P.log | head -20; done
cat > /tmp/nccl_ar.py <<'PY'
import os, torch, torch.distributed as dist
dist.init_process_group("nccl"); r = dist.get_rank(); torch.cuda.set_device(r)
for mb in (16, 64, 256):
    x = torch.ones(mb << 18, device="cuda")
    for _ in range(3): dist.all_reduce(x)
    torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record(); [dist.all_reduce(x) for _ in range(20)]; e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e) / 20; P = dist.get_world_size()
    if r == 0: print(f"NCCL P={P} {mb} MiB: {t*1e3:.1f} us bus {2*(P-1)/P*(mb<<20)/t/1e6:.1f} GB/s", flush=True)
dist.destroy_process_group()
PY
for P in 2 4; do NCCL_DEBUG=INFO timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2960$P /tmp/nccl_ar.py > $O/nccl_p$P.log 2>&1; echo "nccl P=$P rc=$?"; grep -i "nvls" $O/nccl_p$P.log | head -5; grep "^NCCL P" $O/nccl_p$P.log; done
true
