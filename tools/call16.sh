# 2-GPU: stress + CE tests (GPU 0); BERT / R50 real training, CE mode with the event-recording daemon
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2n; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_engine_loopback.py tests/test_gpu_copy_engine.py -q -p no:faulthandler -k "stress or copy_engine" -x > $O/stress.log 2>&1; echo "stress+ce rc=$?"; tail -n 5 $O/stress.log
show() { tail -n 1 $1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); [print(' ', k, {q:(round(v[q],3) if isinstance(v[q],float) else v[q]) for q in ('iter_ms','host_ms','fwd_ms','bwd_ms','post_bwd_ms','groups') if q in v}) for k,v in d['results'].items()]"; }
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29545 tools/train_bench.py --model bert_large --batch 32 --iters 40 --warmup 5 --mode ce --tail-groups 1 --strategies single,mgwfbp,mgwfbp@10,mgwfbp@100,mgwfbp@300,single > $O/bert_ce.log 2>&1; echo "ce rc=$?"; show $O/bert_ce.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29546 tools/train_bench.py --model resnet50 --batch 32 --iters 40 --warmup 5 --mode ce --tail-groups 1 --strategies single,mgwfbp,wfbp,mgwfbp@10,single > $O/r50_ce.log 2>&1; echo "r50 rc=$?"; show $O/r50_ce.log
