cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2c
nvidia-smi topo -m > gpurun_out/r2c/topo2.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multirank.py -q -x > gpurun_out/r2c/mr2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/nvlink_counters.py > gpurun_out/r2c/nvl_counters_p2.log 2>&1
KNOBS=16,1,3072 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 tools/nvlink_counters.py > gpurun_out/r2c/nvl_counters_p2_old.log 2>&1
KNOBS="16,1,3072;16,4,3072;16,4,65536;32,4,65536;16,8,65536" SIZES_KB=4096,16384,65536,262144 ALGOS=twoshot,oneshot CTAS=140 STANDALONE= timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/probe_bw.py > gpurun_out/r2c/sweep_p2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2c/bench_n2.log 2>&1
OUT=gpurun_out/r2c bash tools/ncu_nvlink.sh > gpurun_out/r2c/ncu_nvlink.log 2>&1
tail -n 4 gpurun_out/r2c/mr2.log; cat gpurun_out/r2c/sweep_p2.log | grep -v "^W\|^\s*$" | tail -30; tail -n 12 gpurun_out/r2c/ncu_nvlink.log
