# 1-GPU: bench N=1 on every trace (refresh of the DESIGN table; on-box calibrations saved)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2scale; mkdir -p $O
export MGW_OUT_DIR=$O
for T in googlenet resnet50 resnet152 densenet201 inception_v4 bert_large; do
  timeout 400 python bench.py --steps 20 --warmup 3 --trace $T --no-cpu-baseline > $O/scale_${T}_n1.log 2>&1; echo "$T N=1 rc=$?"
done
python tools/results_table.py $O
