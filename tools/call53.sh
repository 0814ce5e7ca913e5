# 1-GPU: final round-2 check — full GPU suite, smoke, bench N=1 defaults
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2yy; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
timeout 900 python bench.py > $O/bench_n1.log 2>&1; echo "bench N=1 rc=$?"; tail -n 1 $O/bench_n1.log | cut -c1-400
