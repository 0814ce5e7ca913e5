# 4-GPU: CE tests (GPU 0), real training CE mode with the daemon thread, tail 0/1, N=2 and N=4
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2l; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_copy_engine.py -q -p no:faulthandler > $O/gpu.log 2>&1; echo "ce tests rc=$?"; tail -n 3 $O/gpu.log
for N in 2 4; do
for T in 1 0; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N tools/train_bench.py --model bert_large --batch 32 --iters 20 --warmup 5 --mode ce --tail-groups $T --strategies mgwfbp,mgwfbp@10,mgwfbp@100,single > $O/train_ce_bert_n${N}_t$T.log 2>&1; echo "bert N=$N tail=$T rc=$?"; tail -n 1 $O/train_ce_bert_n${N}_t$T.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:(round(v['iter_ms'],3), round(v.get('host_ms',0),3), v.get('groups')) for k,v in d['results'].items()})"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N tools/train_bench.py --model resnet50 --batch 32 --iters 20 --warmup 5 --mode ce --tail-groups 1 --strategies mgwfbp,wfbp,single > $O/train_ce_r50_n$N.log 2>&1; echo "r50 N=$N rc=$?"; tail -n 1 $O/train_ce_r50_n$N.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print({k:(round(v['iter_ms'],3), round(v.get('host_ms',0),3), v.get('groups')) for k,v in d['results'].items()})"
done
