# 4-GPU: cross-group pipelining in the chunked engine — loopback + multirank parity, bench N=2/4 (drain), comm-bound BERT/R50
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2zz; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_engine_loopback.py tests/test_gpu_kernels.py -q -x -p no:faulthandler > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; tail -n 2 $O/gpu.log
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 50 --warmup 10 > $O/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
python - $O/bench_n$N.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['n_gpus'], round(l['value'],3), round(l['ms_per_step'],4), l['gpu'].get('engine_protocol'), {k:round(r[k],3) for k in ['achieved','frac','launch_ms_mean']}, {k:round(v,3) if isinstance(v,float) else v for k,v in r.get('other_protocol_drain',{}).items()}, {k:(round(v['iter_ms_median'],3), round(v.get('device_tail_us',0),1)) for k,v in l['strategies'].items()})
PY
done
for spec in "bert_large 0.1" "resnet50 0.03"; do set -- $spec; for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 50 --warmup 10 --trace $1 --tb-scale $2 > $O/tb_$1_$2_n$N.log 2>&1; echo "tb $1 $2 N=$N rc=$?"
python - $O/tb_$1_$2_n$N.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); s=l['strategies']; m=s['mgwfbp']
print(l['config']['workload'], l['config']['tb_scale'], l['n_gpus'], round(m['iter_ms_median'],3), m['groups'], round(s['wfbp']['iter_ms_median'],3), round(s['single_buffer']['iter_ms_median'],3))
PY
done; done
