# 4-GPU: real training at N=4, CE mode (daemon) vs single buffer vs engine mode
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2o; mkdir -p $O
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','host_ms','fwd_ms','bwd_ms','post_bwd_ms','groups') if q in v}) for k,v in d['results'].items()]"; }
for M in bert_large resnet50 resnet152; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29547 tools/train_bench.py --model $M --batch 32 --iters 40 --warmup 5 --mode ce --tail-groups 1 --strategies ddp,single,mgwfbp,wfbp,mgwfbp@100 > $O/${M}_ce_n4.log 2>&1; echo "$M rc=$?"; show $O/${M}_ce_n4.log
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29548 tools/train_bench.py --model bert_large --batch 32 --iters 40 --warmup 5 --mode engine --tail-groups 1 --strategies mgwfbp > $O/bert_large_engine_n4.log 2>&1; echo "engine rc=$?"; show $O/bert_large_engine_n4.log
