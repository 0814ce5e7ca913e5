# 4-GPU: protocol AUTO = chunked at P>1 (engine); full GPU suite (GPU 0), multirank, bench N=2/4 defaults (other-protocol drain + bus table)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2xx; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -5
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N > $O/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
python - $O/bench_n$N.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['n_gpus'], round(l['value'],3), round(l['ms_per_step'],4), round(l['e2e']['value'],2), l['gpu'].get('engine_protocol'), {k:round(r[k],3) for k in ['achieved','frac','launch_ms_mean']}, r.get('other_protocol_drain'), round(l['iteration_bound']['frac'],4), {k:(round(v['iter_ms_median'],3), round(v.get('device_tail_us',0),1)) for k,v in l['strategies'].items()})
b=l.get('bus_gbs',{})
for k in ('16777216','67108864','134217728','268435456'):
  if k in b: print('   bus', int(k)>>20, 'MiB', {kk:round(vv,1) for kk,vv in b[k].items()})
PY
done
