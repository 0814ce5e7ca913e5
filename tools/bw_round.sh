#!/bin/bash
# 2/4-GPU call: GPU tests, bandwidth probe, benches. Logs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export MGW_OUT_DIR=gpurun_out
NG=$(nvidia-smi -L | wc -l)
TAG="${1:-x}"
if [[ "${SKIP_TESTS:-0}" != 1 ]]; then
  timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_$TAG.log
fi
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29512 tools/probe_bw.py > gpurun_out/bw_${TAG}_p$NG.log 2>&1; echo "bw rc=$?"; grep -A8 "^P=" gpurun_out/bw_${TAG}_p$NG.log
if [[ "${BENCH:-1}" == 1 ]]; then
  for N in 1 $NG; do
    if [[ $N == 1 ]]; then
      CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 20 --warmup 3 --cpu-budget-s 3 > gpurun_out/bench_${TAG}_n1.log 2>&1
    else
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_n$N.log 2>&1
    fi
    echo "bench N=$N rc=$?"
  done
fi
