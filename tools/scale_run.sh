#!/bin/bash
# Multi-GPU call: parity at P=2/4/8 (tests/test_gpu_multirank.py) and the
# bench at N=1,2,4,8 for one trace. Logs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export MGW_OUT_DIR=gpurun_out
TRACE="${1:-googlenet}"
STEPS="${2:-20}"
NG=$(nvidia-smi -L | wc -l)
if [[ "${SKIP_TESTS:-0}" != 1 ]]; then
  timeout 300 python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/mr.log 2>&1; echo "multirank rc=$?"
fi
for N in 1 2 4 8; do
  [[ $N -gt $NG ]] && continue
  if [[ $N == 1 ]]; then
    CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps $STEPS --warmup 3 --trace $TRACE --cpu-budget-s 3 > gpurun_out/scale_${TRACE}_n1.log 2>&1
  else
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --steps $STEPS --warmup 3 --trace $TRACE > gpurun_out/scale_${TRACE}_n${N}.log 2>&1
  fi
  echo "bench N=$N rc=$?"
done
