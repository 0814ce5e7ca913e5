#!/bin/bash
# Quick fused-allreduce bandwidth check at P=2 and P=4 (tools/probe_bw.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for P in ${PS:-2 4}; do
  D=$(seq -s, 0 $((P-1)))
  for S in ${SETS:-SIZES_KB=4,64,1024,4096 SIZES_MB=16,64,256}; do
    env $S CUDA_VISIBLE_DEVICES=$D CTAS=${CTAS:-140} ALGOS=${ALGOS:-oneshot,twoshot} STANDALONE=${STANDALONE-twoshot} \
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
      --master-port 29512 tools/probe_bw.py 2>&1 | grep -A8 "^P=\|Error\|error" | head -12
  done
done
