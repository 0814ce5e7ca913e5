#!/bin/bash
# 1-GPU ncu evidence (never multi-rank under ncu): launch list of the bench in
# per-group-launch mode (the persistent engine waits on a concurrently running
# replay kernel, which ncu's kernel serialisation forbids), then one full
# capture of the fused group kernel on a 16 MiB group (tools/probe.py).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python bench.py --engine-ctas 0 --steps 2 --warmup 1 --no-cpu-baseline --l2-flush-mib 0"
timeout 300 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
REPS=3 timeout 120 python tools/probe.py > gpurun_out/ncu_probe_plain.log 2>&1 && \
  REPS=3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:group_allreduce -s 10 -c 2 -o gpurun_out/prof_group python tools/probe.py > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
