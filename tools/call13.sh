# 4-GPU: multirank P=2/4 (default protocol), bench N=4 both protocols, real training CE mode variants
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2k; mkdir -p $O
nvidia-smi topo -m > $O/topo4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multirank.py -q > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 2 $O/mr.log
for PR in chunked stream; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 10 --warmup 3 --protocol $PR > $O/bench_n4_$PR.log 2>&1; echo "bench $PR rc=$?"
python - $O/bench_n4_$PR.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['ms_per_step'], {k:r[k] for k in ['achieved','frac','launch_ms_mean']}, {k:(v['iter_ms_median'], v.get('device_tail_us')) for k,v in l['strategies'].items()})
PY
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 tools/train_bench.py --model bert_large --batch 32 --iters 20 --warmup 5 --mode ce --strategies mgwfbp,mgwfbp@10,mgwfbp@100,merged,single > $O/train_ce_bert_n4.log 2>&1; echo "train rc=$?"; tail -n 1 $O/train_ce_bert_n4.log | cut -c1-2000
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29536 tools/train_bench.py --model resnet50 --batch 32 --iters 20 --warmup 5 --mode ce --strategies mgwfbp,wfbp,merged,single > $O/train_ce_r50_n4.log 2>&1; echo "train rc=$?"; tail -n 1 $O/train_ce_r50_n4.log | cut -c1-2000
