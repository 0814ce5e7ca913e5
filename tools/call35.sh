cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ee; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -x > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -5
python tools/drain_probe.py --trace googlenet --P 1 --iters 3 --stamps > $O/drain_gn.log 2>&1; echo "rc=$?"; grep "CTA\|span" $O/drain_gn.log | cut -c1-600; tail -n 1 $O/drain_gn.log | cut -c1-200
for T in googlenet densenet201 resnet50 resnet152 inception_v4 bert_large; do
  timeout 400 python bench.py --steps 20 --warmup 3 --trace $T --no-cpu-baseline > $O/scale_${T}_n1.log 2>&1; echo "$T N=1 rc=$?"
done
python tools/results_table.py $O
