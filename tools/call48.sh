# 4-GPU: round-end validation after NVLS: full GPU suite (GPU 0), smoke, multirank P=2/4 (incl. NVLS), bench N=1/2/4 defaults,
# bench N=4 with NVLS measured (--nvls -1) and used for groups >= 64 MiB (--nvls 64)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2tt; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -5
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_n1.log 2>&1; echo "bench N=1 rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
done
for X in -1 64; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --steps 50 --warmup 10 --nvls $X > $O/bench_n4_nvls$X.log 2>&1; echo "bench N=4 nvls=$X rc=$?"
done
for f in $O/bench_n1.log $O/bench_n2.log $O/bench_n4.log $O/bench_n4_nvls-1.log $O/bench_n4_nvls64.log; do python - $f <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(sys.argv[1].split('/')[-1], l['n_gpus'], round(l['value'],3), round(l['ms_per_step'],4), round(l['e2e']['value'],2), l['gpu'].get('nvls'), {k:round(r[k],3) for k in ['achieved','frac','launch_ms_mean']}, round(l['iteration_bound']['frac'],4), {k:(round(v['iter_ms_median'],3), round(v.get('device_tail_us',0),1)) for k,v in l['strategies'].items()})
b=l.get('bus_gbs',{})
for k in ('16777216','67108864','134217728','268435456','536870912'):
  if k in b: print('   bus', int(k)>>20, 'MiB', {kk:round(vv,1) for kk,vv in b[k].items()})
PY
done
