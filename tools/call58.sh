# 2-GPU: P=2 one-shot vs two-shot at large sizes (chunked engine) — is the 8 MiB crossover right above 16 MiB?
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ae; mkdir -p $O
SIZES_MB=8,16,32,64,128,256 CTAS=140 ALGOS=oneshot,twoshot PROTOS=chunked STANDALONE= REPS=15 \
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/probe_bw.py > $O/bw_p2.log 2>&1; echo "bw rc=$?"; grep -A6 "^P=" $O/bw_p2.log
