# 2-GPU: loopback tests (GPU 0), multirank P=2, P=2 sweep stream vs chunked x tile-size threshold
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2g; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/dbg_stream.py > $O/dbg.log 2>&1; echo "dbg rc=$?"; grep -c "bad=0 \[\]" $O/dbg.log; grep -v "bad=0 \[\]" $O/dbg.log | head
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine_loopback.py -q -p no:faulthandler > $O/gpu.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED" $O/gpu.log | tail -12
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > $O/mr2.log 2>&1; echo "mr rc=$?"; tail -n 2 $O/mr2.log
KNOBS="16,1,3072;16,1,65536;16,1,524288" PROTOS=stream,chunked SIZES_KB=1024,4096,16384,65536,262144 ALGOS=twoshot,oneshot CTAS=140 STANDALONE= timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/probe_bw.py > $O/sweep_p2.log 2>&1; echo "sweep rc=$?"
grep -v "^W\|^\s*$\|^\*\|OMP\|NCCL version" $O/sweep_p2.log | tail -16
