# 4-GPU: hybrid (streamed engine + chunked tail launch): tests (GPU 0), multirank, bench N=2/4 both protocols
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2jj; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_engine_loopback.py tests/test_gpu_kernels.py -q -p no:faulthandler -x > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; tail -n 1 $O/gpu.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log
for N in 2 4; do for PR in chunked stream; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 50 --warmup 10 --protocol $PR > $O/bench_n${N}_$PR.log 2>&1; echo "bench N=$N $PR rc=$?"
python - $O/bench_n${N}_$PR.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(round(l['ms_per_step'],4), round(l['e2e']['value'],2), {k:round(r[k],3) for k in ['achieved','frac','launch_ms_mean']}, {k:(round(v['iter_ms_median'],3), round(v.get('device_tail_us',0),1)) for k,v in l['strategies'].items()})
PY
done; done
