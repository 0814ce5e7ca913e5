# 4-GPU: real training, copy-engine mode: single buffer vs calibrated MG-WFBP vs in-situ tuned plan
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ff; mkdir -p $O
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','bwd_ms','post_bwd_ms','groups','autotune') if q in v}) for k,v in d['results'].items()]"; }
for M in bert_large resnet50; do for N in 4 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N tools/train_bench.py --model $M --batch 32 --iters 40 --warmup 5 --mode ce --tail-groups 1 --strategies single,mgwfbp,tuned > $O/${M}_n$N.log 2>&1; echo "$M N=$N rc=$?"; show $O/${M}_n$N.log
done; done
