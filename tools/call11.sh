# 2-GPU: bench N=2 (bert_large) chunked vs stream protocol
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2i; mkdir -p $O
for PR in chunked stream; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --steps 10 --warmup 3 --protocol $PR > $O/bench_n2_$PR.log 2>&1; echo "bench $PR rc=$?"
python - $O/bench_n2_$PR.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['ms_per_step'], {k:r[k] for k in ['achieved','frac','launch_ms_mean']}, {k:v['iter_ms_median'] for k,v in l['strategies'].items()})
PY
done
