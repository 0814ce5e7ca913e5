# 2-GPU: BERT-large real training at N=2, copy-engine mode, longer runs (100 timed iterations) to separate noise from the strategy gap
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ac; mkdir -p $O
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','bwd_ms','post_bwd_ms','groups','autotune') if q in v}) for k,v in d['results'].items()]"; }
for rep in 1 2; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29565 tools/train_bench.py --model bert_large --batch 32 --iters 100 --warmup 10 --mode ce --tail-groups 1 --strategies single,mgwfbp,mgwfbp@30,tuned > $O/bert_n2_rep$rep.log 2>&1; echo "rep $rep rc=$?"; show $O/bert_n2_rep$rep.log
done
