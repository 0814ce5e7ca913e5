# 1-GPU: regression (stream ramp, ld_group) + N=1 drain on many-group traces
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2v; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -x > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -5
for T in googlenet densenet201 bert_large; do
  timeout 400 python bench.py --steps 10 --warmup 3 --trace $T --no-cpu-baseline > $O/scale_${T}_n1.log 2>&1; echo "$T N=1 rc=$?"
done
python tools/results_table.py $O
