#!/bin/bash
# Chunk-size sweep of the fused two-shot engine (tools/probe_bw.py) at P=2 and P=NG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
NG=$(nvidia-smi -L | wc -l)
for P in 2 $NG; do
  [[ $P == 2 && $NG == 2 ]] && [[ -n "${DONE2:-}" ]] && continue
  DEVS=$(seq -s, 0 $((P-1)))
  for C in ${CHUNKS:-2 4 8 16}; do
    echo "== P=$P chunk=$C"
    CUDA_VISIBLE_DEVICES=$DEVS MGW_CHUNK_TILES=$C SIZES_KB=${SIZES_KB:-16384,65536,92672,185364,262144} ALGOS=${ALGOS:-twoshot} CTAS=140 STANDALONE= \
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 29512 tools/probe_bw.py 2>&1 | grep -A4 "^P=" | grep -v "^P="
  done
  DONE2=1
done
