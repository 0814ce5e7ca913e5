# 4-GPU: NVLS phase split (skip pack/unpack, skip reduce) at P=2,4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ss; mkdir -p $O
for P in 2 4; do
D=$(seq -s, 0 $((P-1)))
SIZES_MB=4,16,64,256 CUDA_VISIBLE_DEVICES=$D CTAS=140 ALGOS=twoshot PROTOS=chunked STANDALONE=nvls NVLS_CHUNKS=4 NVLS_SKIP=0,1,2,3 SREPS=9 \
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2951$P tools/probe_bw.py > $O/bw_p$P.log 2>&1; echo "bw P=$P rc=$?"; grep -A12 "^P=" $O/bw_p$P.log; tail -3 $O/bw_p$P.log
done
