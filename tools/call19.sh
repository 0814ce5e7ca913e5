cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2q; mkdir -p $O
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
python - $O/bench.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['value'], l['ms_per_step'], l['e2e']['value'], l['gpu']['tuning'], {k:r[k] for k in ['achieved','frac','launch_ms_mean']}, r['largest_group'], l['clocks'])
PY
timeout 600 python -m pytest tests -m gpu -q -p no:faulthandler -k "p1 or P1 or drain or ddp or pipeline" > $O/gpu.log 2>&1; echo "gpu subset rc=$?"; tail -n 2 $O/gpu.log
