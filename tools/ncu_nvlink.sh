#!/bin/bash
# ncu NVLink byte counters of the REAL cross-GPU fused all-reduce at P = 2:
# rank 1 runs free, rank 0 runs under ncu with only single-pass metrics
# (NVLink tx/rx bytes, duration) so the profiled launch is never replayed (a
# replay could not re-synchronise with the unprofiled peer); no NCCL in the
# processes (tools/nvl_pair.py swaps the IPC handles through files).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=${OUT:-gpurun_out/r2}
mkdir -p "$OUT"
for ALGO in ${ALGOS:-twoshot oneshot}; do
for MB in ${SIZES_MB:-16 64 256}; do
  D=$(mktemp -d)
  METRICS=${METRICS:-gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum}
  timeout 300 python tools/nvl_pair.py 1 "$D" $MB $ALGO > "$OUT/ncu_nvl_r1_${ALGO}_${MB}.log" 2>&1 &
  timeout 300 /usr/local/cuda/bin/ncu --metrics "$METRICS" --clock-control none -k regex:group_allreduce \
    --launch-skip 3 --launch-count 1 --csv --log-file "$OUT/ncu_nvlink_P2_${ALGO}_${MB}MiB.csv" \
    python tools/nvl_pair.py 0 "$D" $MB $ALGO > "$OUT/ncu_nvl_r0_${ALGO}_${MB}.log" 2>&1
  echo "== $ALGO $MB MiB rank0 rc=$?"
  wait
  cat "$OUT/ncu_nvl_r0_${ALGO}_${MB}.log" "$OUT/ncu_nvl_r1_${ALGO}_${MB}.log" | grep -v "^==PROF==" | tail -3
  grep -h "nvl\|duration" "$OUT/ncu_nvlink_P2_${ALGO}_${MB}MiB.csv" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  rm -rf "$D"
done
done
