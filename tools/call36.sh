# 4-GPU: multirank parity with per-CTA schedules, then the N=2/4 scale on every trace
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2scale2; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 2 $O/mr.log
for T in googlenet resnet50 resnet152 densenet201 inception_v4 bert_large; do
  for N in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps 20 --warmup 3 --trace $T > $O/scale_${T}_n${N}.log 2>&1; echo "$T N=$N rc=$?"
  done
done
