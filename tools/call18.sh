# 1-GPU: full GPU test suite (P=1 TMA engine path), bench N=1 default, smoke
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2p; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -12
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 2 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
python - $O/bench.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['value'], l['ms_per_step'], l['e2e']['value'], {k:r[k] for k in ['achieved','frac','launch_ms_mean']}, r['largest_group'], l['clocks'])
PY
