# 2-GPU: P=2 streamed-protocol publication batches
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2h; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/dbg_stream.py > $O/dbg.log 2>&1; echo "dbg rc=$?"; grep -c "bad=0 \[\]" $O/dbg.log
KNOBS="16,1,3072,512,8,4;16,1,3072,512,2,4;16,1,3072,512,1,1;16,1,3072,512,4,2;16,1,3072,512,2,8" PROTOS=stream SIZES_KB=4096,16384,65536,262144 ALGOS=twoshot,oneshot CTAS=140 STANDALONE= timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/probe_bw.py > $O/sweep_p2.log 2>&1; echo "sweep rc=$?"
grep -v "^W\|^\s*$\|^\*\|OMP\|NCCL version" $O/sweep_p2.log | tail -16
