# 1-GPU batch: GPU tests, sanitizers, ncu of the roofline kernel (engine drain), launch lists
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:faulthandler > $O/gpu4.log 2>&1; echo "gpu tests rc=$?"
python tools/drain_probe.py --trace bert_large --P 1 --iters 5 > $O/drain_p1.log 2>&1
python tools/drain_probe.py --trace bert_large --P 2 --iters 5 > $O/drain_p2lb.log 2>&1
python tools/drain_probe.py --trace resnet50 --P 1 --iters 5 > $O/drain_r50_p1.log 2>&1
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:engine_kernel --launch-count 1 \
  -o $O/prof_drain_bert_p1 python tools/drain_probe.py --trace bert_large --P 1 --iters 1 > $O/ncu_drain_p1.log 2>&1; echo "ncu drain p1 rc=$?"
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:engine_kernel --launch-count 1 \
  -o $O/prof_drain_bert_p2lb python tools/drain_probe.py --trace bert_large --P 2 --iters 1 > $O/ncu_drain_p2lb.log 2>&1; echo "ncu drain p2lb rc=$?"
timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_drain_p1.csv python tools/drain_probe.py --trace bert_large --P 1 --iters 3 > $O/ncu_launch_drain.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_bench_n1_percall.csv python bench.py --steps 2 --warmup 1 --engine-ctas 0 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1; echo "ncu bench launches rc=$?"
PS="1 2 4 8" TOOLS="memcheck racecheck synccheck" OUT=$O bash tools/sanitize.sh > $O/sanitize.log 2>&1
PS="2" TOOLS="initcheck" OUT=$O bash tools/sanitize.sh >> $O/sanitize.log 2>&1
tail -n 3 $O/gpu4.log; cat $O/drain_p1.log $O/drain_p2lb.log $O/drain_r50_p1.log | cut -c1-400; cat $O/sanitize.log
