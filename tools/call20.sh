# 1-GPU ncu: the TMA-fed P=1 engine drain (BERT-large plan) --set full + the bench launch list
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2r; mkdir -p $O
python tools/drain_probe.py --trace bert_large --P 1 --iters 5 > $O/drain_p1.log 2>&1; echo "drain rc=$?"; tail -n 2 $O/drain_p1.log | cut -c1-600
timeout 600 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:engine_kernel --launch-count 1 \
  -o $O/prof_drain_bert_p1_tma python tools/drain_probe.py --trace bert_large --P 1 --iters 1 > $O/ncu_drain_p1.log 2>&1; echo "ncu drain rc=$?"
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_bench_n1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch_bench.log 2>&1; echo "ncu bench launches rc=$?"
