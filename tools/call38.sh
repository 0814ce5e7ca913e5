cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2gg; mkdir -p $O
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','bwd_ms','post_bwd_ms','groups','autotune') if q in v}) for k,v in d['results'].items()]"; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29564 tools/train_bench.py --model bert_large --batch 32 --iters 20 --warmup 5 --mode ce --tail-groups 1 --strategies single --debug > $O/bert_single_n4.log 2>&1; echo "single rc=$?"; grep -h "debug step\|Error" $O/bert_single_n4.log | head; show $O/bert_single_n4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29565 tools/train_bench.py --model bert_large --batch 32 --iters 40 --warmup 5 --mode ce --tail-groups 1 --strategies ddp,single,mgwfbp,tuned > $O/bert_n4.log 2>&1; echo "all rc=$?"; show $O/bert_n4.log
