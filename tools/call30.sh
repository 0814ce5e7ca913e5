# 4-GPU: chunked-protocol knobs at P=4 (two-shot), 16-256 MiB
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2z; mkdir -p $O
KNOBS="16,1,3072;8,1,3072;32,1,3072;16,2,3072;8,2,3072;16,1,65536" PROTOS=chunked SIZES_KB=16384,65536,131072,262144 ALGOS=twoshot CTAS=140 STANDALONE= timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 tools/probe_bw.py > $O/sweep_p4_knobs.log 2>&1; echo "sweep rc=$?"
grep -v "^W\|^\s*$\|^\*\|OMP\|NCCL version" $O/sweep_p4_knobs.log | tail -9
