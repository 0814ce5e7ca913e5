# 2-GPU: streamed protocol correctness (1-GPU loopback tests) then P=2 bandwidth stream vs chunked
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2e; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine_loopback.py -q -x -p no:faulthandler > $O/gpu.log 2>&1; echo "gpu tests rc=$?"
tail -n 30 $O/gpu.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > $O/mr2.log 2>&1; echo "mr rc=$?"; tail -n 3 $O/mr2.log
PROTOS=stream,chunked SIZES_KB=256,1024,4096,16384,65536,262144 ALGOS=twoshot,oneshot CTAS=140 STANDALONE= timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/probe_bw.py > $O/sweep_p2.log 2>&1; echo "sweep rc=$?"
grep -v "^W\|^\s*$" $O/sweep_p2.log | tail -12
