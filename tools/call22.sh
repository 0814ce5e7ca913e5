# 4-GPU: multirank parity (P=2,4: CE mode + NVLink ordering stress), Inception-v4 real training N=4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2t; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 3 $O/mr.log; grep -h "MULTIRANK" -r $O/mr.log | head
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','host_ms','fwd_ms','bwd_ms','post_bwd_ms','groups') if q in v}) for k,v in d['results'].items()]"; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29547 tools/train_bench.py --model inception_v4 --batch 128 --iters 20 --warmup 5 --mode ce --tail-groups 1 --strategies ddp,single,mgwfbp,wfbp > $O/inception_v4_ce_n4.log 2>&1; echo "inception rc=$?"; show $O/inception_v4_ce_n4.log
