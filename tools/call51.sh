# 4-GPU: comm-bound regime, engine protocol chunked vs stream (AUTO results: call50 / r2uu)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ww; mkdir -p $O
for PR in chunked stream; do
for spec in "bert_large 0.1" "resnet50 0.03" "resnet50 0.1" "googlenet 0.03"; do
set -- $spec
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N bench.py --gpus $N --steps 50 --warmup 10 --trace $1 --tb-scale $2 --protocol $PR > $O/tb_$1_$2_n${N}_$PR.log 2>&1; echo "tb $1 $2 N=$N $PR rc=$?"
tail -n 1 $O/tb_$1_$2_n${N}_$PR.log >> $O/tbscale_$PR.jsonl
done; done; done
for PR in chunked stream; do echo "== $PR"; python - $O/tbscale_$PR.jsonl <<'PY'
import json,sys
for ln in open(sys.argv[1]):
    try: l=json.loads(ln)
    except Exception: continue
    s=l['strategies']; m=s['mgwfbp']
    print(l['config']['workload'], l['config']['tb_scale'], l['n_gpus'], round(m['iter_ms_median'],3), round(m['predicted_ms'],3), m['groups'], round(s['wfbp']['iter_ms_median'],3), round(s['single_buffer']['iter_ms_median'],3), round(s['wfbp']['iter_ms_median']/m['iter_ms_median'],2), round(s['single_buffer']['iter_ms_median']/m['iter_ms_median'],2))
PY
done
