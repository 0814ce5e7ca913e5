# 4-GPU: NVLS product path — multirank tests (P=2,4: NVLS bit-exact vs the exact-sum oracle) + bandwidth (push two-shot vs NVLS chunks vs NCCL)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2rr; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs -s > $O/mr.log 2>&1; echo "mr rc=$?"; grep -E "MULTIRANK|nvls calibration|passed|failed|Error|error" $O/mr.log | head -20
for P in 2 4; do
D=$(seq -s, 0 $((P-1)))
SIZES_MB=1,4,16,64,128,256 CUDA_VISIBLE_DEVICES=$D CTAS=140 ALGOS=twoshot PROTOS=chunked STANDALONE=twoshot,nvls NVLS_CHUNKS=1,2,4 SREPS=9 \
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2951$P tools/probe_bw.py > $O/bw_p$P.log 2>&1; echo "bw P=$P rc=$?"; grep -A12 "^P=" $O/bw_p$P.log; tail -3 $O/bw_p$P.log
done
