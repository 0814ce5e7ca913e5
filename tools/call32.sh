cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2bb; mkdir -p $O
S=$SECONDS; timeout 1200 python bench.py > $O/bench.log 2> $O/bench.err; echo "bench rc=$? wall $((SECONDS-S)) s"
python - $O/bench.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(l['value'], l['steps'], l['warmup'], l['ms_per_step'], l['e2e']['value'], l['iteration_bound'], {k:r[k] for k in ['achieved','frac','launch_ms_mean']}, l['clocks'], l['gpu_launches'])
print({k:(v['iter_ms_median'],v['iter_ms_p10'],v['iter_ms_p90']) for k,v in l['strategies'].items()})
PY
S=$SECONDS; timeout 900 python bench.py --impl reference > $O/bench_ref.log 2> $O/bench_ref.err; echo "ref rc=$? wall $((SECONDS-S)) s"; tail -n 1 $O/bench_ref.log | cut -c1-400
