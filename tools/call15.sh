# 2-GPU: ordering stress tests (GPU 0); BERT real training phase breakdown (CE vs engine)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2m; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_engine_loopback.py -q -p no:faulthandler -k "stress" > $O/stress.log 2>&1; echo "stress rc=$?"; tail -n 3 $O/stress.log
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','host_ms','fwd_ms','bwd_ms','post_bwd_ms','groups') if q in v}) for k,v in d['results'].items()]"; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29545 tools/train_bench.py --model bert_large --batch 32 --iters 20 --warmup 5 --mode ce --tail-groups 1 --strategies mgwfbp,mgwfbp@3,mgwfbp@10,mgwfbp@30,mgwfbp@100,mgwfbp@300,single > $O/bert_ce.log 2>&1; echo "ce rc=$?"; show $O/bert_ce.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29546 tools/train_bench.py --model bert_large --batch 32 --iters 20 --warmup 5 --mode engine --tail-groups 1 --strategies mgwfbp,single > $O/bert_engine.log 2>&1; echo "engine rc=$?"; show $O/bert_engine.log
