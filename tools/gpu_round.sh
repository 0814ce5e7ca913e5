#!/bin/bash
# One gpurun call: smoke, GPU tests, B200 trace extraction, 1-GPU bench,
# launch list + one ncu capture of the fused kernel. Logs in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export MGW_OUT_DIR=gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/host_cpu.txt 2>&1; nproc >> gpurun_out/host_cpu.txt
STEP="${1:-all}"
if [[ "$STEP" == all || "$STEP" == smoke ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/status.txt
fi
if [[ "$STEP" == all || "$STEP" == tests ]]; then
  timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a gpurun_out/status.txt
fi
if [[ "$STEP" == all || "$STEP" == traces ]]; then
  timeout 900 python tools/extract_traces.py --out gpurun_out/traces > gpurun_out/traces.log 2>&1; echo "traces rc=$?" | tee -a gpurun_out/status.txt
fi
