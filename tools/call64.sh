# 1-GPU: final code — smoke + bench N=1 defaults
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ak; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
timeout 900 python bench.py > $O/bench_n1.log 2>&1; echo "bench N=1 rc=$?"
python - $O/bench_n1.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(round(l['value'],3), round(l['ms_per_step'],4), round(l['e2e']['value'],2), round(r['frac'],3), l['clocks'], l['gpu_launches'] if 'gpu_launches' in l else None)
PY
