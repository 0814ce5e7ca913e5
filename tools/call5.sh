# 1-GPU batch (round 2 re-entry): GPU tests, smoke, default bench, sanitizers
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2b; mkdir -p $O
nvidia-smi -L > $O/smi.txt 2>&1; nproc >> $O/smi.txt
timeout 900 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.log 2>&1; echo "bench ref rc=$?"
PS="1 2 4 8" TOOLS="memcheck racecheck synccheck" OUT=$O timeout 1500 bash tools/sanitize.sh > $O/sanitize.log 2>&1
tail -n 15 $O/gpu.log; tail -n 3 $O/smoke.log; tail -n 2 $O/bench.log | cut -c1-3000; tail -n 2 $O/bench_ref.log | cut -c1-1500; cat $O/sanitize.log
