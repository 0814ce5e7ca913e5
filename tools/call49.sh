# 4-GPU: comm-bound regime refresh with the round-2 engine (protocol AUTO): bench --tb-scale at N=2,4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2uu; mkdir -p $O
for spec in "bert_large 0.1" "resnet50 0.03" "resnet50 0.1" "googlenet 0.03" "googlenet 0.1"; do
set -- $spec
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 50 --warmup 10 --trace $1 --tb-scale $2 > $O/tb_$1_$2_n$N.log 2>&1; echo "tb $1 $2 N=$N rc=$?"
tail -n 1 $O/tb_$1_$2_n$N.log >> $O/tbscale.jsonl
done; done
python - $O/tbscale.jsonl <<'PY'
import json,sys
for ln in open(sys.argv[1]):
    try: l=json.loads(ln)
    except Exception: continue
    s=l['strategies']; m=s['mgwfbp']
    print(l['config']['workload'], l['config']['tb_scale'], l['n_gpus'], round(m['iter_ms_median'],3), round(m['predicted_ms'],3), m['groups'], round(s['wfbp']['iter_ms_median'],3), round(s['single_buffer']['iter_ms_median'],3), round(s['wfbp']['iter_ms_median']/m['iter_ms_median'],2), round(s['single_buffer']['iter_ms_median']/m['iter_ms_median'],2))
PY
