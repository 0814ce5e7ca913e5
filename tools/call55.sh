# 2-GPU: multirank P=2 (NVLS cuDeviceGet change) + real training at N=2 in copy-engine mode (verdict item 7 at N=2)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ab; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','bwd_ms','post_bwd_ms','groups','autotune') if q in v}) for k,v in d['results'].items()]"; }
for M in bert_large resnet50; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29565 tools/train_bench.py --model $M --batch 32 --iters 40 --warmup 5 --mode ce --tail-groups 1 --strategies ddp,single,mgwfbp,wfbp,tuned > $O/${M}_n2.log 2>&1; echo "$M rc=$?"; show $O/${M}_n2.log
done
