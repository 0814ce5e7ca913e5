# 4-GPU: final normal build — GPU suite (GPU 0), smoke, multirank, bench N=1/2/4 defaults
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ah; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -3
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_n1.log 2>&1; echo "bench N=1 rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
done
for N in 1 2 4; do python - $O/bench_n$N.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['n_gpus'], round(l['value'],3), round(l['ms_per_step'],4), round(l['e2e']['value'],2), l['gpu'].get('engine_protocol'), round(r['frac'],3), round(l['iteration_bound']['frac'],4), l['clocks']['sm_mhz'], l['clocks']['reasons'], {k:(round(v['iter_ms_median'],3), round(v.get('device_tail_us',0),1)) for k,v in l['strategies'].items()})
PY
done
