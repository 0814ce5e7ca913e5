#!/bin/bash
# Two-shot / one-shot chunking sweep of the fused engine (tools/probe_bw.py) at
# P = 2 and P = NG: KNOBS = "chunk_tiles,min_chunks,small_tile_max_KiB;..." set
# through the C-ABI setters (mgw_comm_set_chunk_tiles / _set_small_tile_max).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
NG=$(nvidia-smi -L | wc -l)
for P in $(echo 2 $NG | tr ' ' '\n' | sort -u); do
  DEVS=$(seq -s, 0 $((P-1)))
  echo "== P=$P"
  CUDA_VISIBLE_DEVICES=$DEVS KNOBS="${KNOBS:-16,1,3072;16,4,3072;16,4,65536;32,4,65536}" \
    SIZES_KB=${SIZES_KB:-4096,16384,65536,262144} ALGOS=${ALGOS:-twoshot} CTAS=${CTAS:-140} STANDALONE= \
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 \
    --master-port 29512 tools/probe_bw.py 2>&1 | grep -v "^W\|^\s*$" | tail -20
done
