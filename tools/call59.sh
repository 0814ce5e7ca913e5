# 4-GPU: final-code sanity on LL/one-shot-heavy plans (GoogLeNet, ResNet-152) at N=4 vs the r2_scale table
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2af; mkdir -p $O
for T in googlenet resnet152; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --trace $T --steps 50 --warmup 10 > $O/bench_${T}_n4.log 2>&1; echo "$T rc=$?"
python - $O/bench_${T}_n4.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['config']['workload'], l['n_gpus'], round(l['value'],3), round(l['ms_per_step'],4), l['gpu'].get('engine_protocol'), round(r['frac'],3), {k:round(v,3) if isinstance(v,float) else v for k,v in r.get('other_protocol_drain',{}).items()}, {k:(round(v['iter_ms_median'],3), round(v.get('device_tail_us',0),1)) for k,v in l['strategies'].items()})
PY
done
