# 4-GPU: bench N=2,4 on every trace (chunked default); on-box calibrations saved
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2scale; mkdir -p $O
export MGW_OUT_DIR=$O
for T in googlenet resnet50 resnet152 densenet201 inception_v4 bert_large; do
  for N in 2 4; do
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29600 + N)) bench.py --gpus $N --steps 20 --warmup 3 --trace $T > $O/scale_${T}_n${N}.log 2>&1; echo "$T N=$N rc=$?"
  done
done
