#!/bin/bash
# ncu --set full of the fused two-shot group kernel in loopback (P emulated
# ranks on one GPU, one cooperative launch) — single GPU, never multi-rank.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-lb}
P=${P:-2} SIZE_MB=${SIZE_MB:-64} ALGO=${ALGO:-twoshot} timeout 120 python tools/probe_loopback.py && \
P=${P:-2} SIZE_MB=${SIZE_MB:-64} ALGO=${ALGO:-twoshot} ITERS=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:group_allreduce -s 2 -c 1 -o gpurun_out/prof_$TAG python tools/probe_loopback.py > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?"
