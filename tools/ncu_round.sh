#!/bin/bash
# 1-GPU ncu evidence (never multi-rank under ncu). Each capture only after the
# same command exited 0 without ncu.
#  1. launch list of the bench in per-group-launch mode (the persistent engine
#     waits on a concurrently running replay kernel, which ncu's kernel
#     serialisation forbids)
#  2. --set full of pack, unpack+SGD and the P=1 fused group kernel (256 MiB)
#  3. --set full of the fused two-shot kernel in loopback (P=2 and P=4
#     emulated ranks, 64 MiB per rank, one cooperative launch)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python bench.py --engine-ctas 0 --steps 2 --warmup 3 --no-cpu-baseline --l2-flush-mib 0"
# the ncu run plans with the plain run's calibrated (a, b): same plan, same launches
timeout 300 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
  MODEL=$(python tools/model_from_bench.py gpurun_out/ncu_plain.log) && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches.csv $CMD --model $MODEL > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 120 python tools/probe_pack.py > gpurun_out/probe_pack.log 2>&1 && \
  REPS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_kernel|unpack_sgd|group_allreduce" -c 3 -o gpurun_out/prof_pack python tools/probe_pack.py > gpurun_out/ncu_pack.log 2>&1
echo "pack/unpack rc=$?"
for P in 2 4; do
  P=$P SIZE_MB=64 ALGO=twoshot timeout 120 python tools/probe_loopback.py > gpurun_out/probe_lb$P.log 2>&1 && \
  P=$P SIZE_MB=64 ALGO=twoshot ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:group_allreduce -s 2 -c 1 -o gpurun_out/prof_lb$P python tools/probe_loopback.py > gpurun_out/ncu_lb$P.log 2>&1
  echo "loopback P=$P rc=$?"
done
