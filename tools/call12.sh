# 2-GPU: CE-mode + stream tests (GPU 0), P=2 sweep, bench N=2 both protocols, real training CE mode
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2j; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_copy_engine.py tests/test_gpu_kernels.py tests/test_gpu_engine_loopback.py -q -p no:faulthandler > $O/gpu.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED|Error" $O/gpu.log | tail -12
PROTOS=stream,chunked SIZES_KB=4096,16384,65536,262144 ALGOS=twoshot,oneshot CTAS=140 STANDALONE= timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 tools/probe_bw.py > $O/sweep_p2.log 2>&1; echo "sweep rc=$?"
grep -v "^W\|^\s*$\|^\*\|OMP\|NCCL version" $O/sweep_p2.log | tail -8
for PR in chunked stream; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 10 --warmup 3 --protocol $PR > $O/bench_n2_$PR.log 2>&1; echo "bench $PR rc=$?"
python - $O/bench_n2_$PR.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['ms_per_step'], {k:r[k] for k in ['achieved','frac','launch_ms_mean']}, {k:(v['iter_ms_median'], v.get('device_tail_us')) for k,v in l['strategies'].items()})
PY
done
for M in bert_large resnet50; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 tools/train_bench.py --model $M --batch 32 --iters 20 --warmup 5 --mode ce --strategies mgwfbp,wfbp,single > $O/train_ce_$M.log 2>&1; echo "train $M rc=$?"; tail -n 1 $O/train_ce_$M.log | cut -c1-1500
done
