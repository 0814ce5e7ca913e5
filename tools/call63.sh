# 4-GPU: calibration replay gated on the engine's entry barrier (no cross-rank launch skew in T(M)): GPU suite, multirank, small-size engine calibration P=2/4, bench N=2/4 on-box fit
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2aj; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -3
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log
for P in 2 4; do D=$(seq -s, 0 $((P-1)))
SIZES_KB=4,16,64,256,1024,4096 CUDA_VISIBLE_DEVICES=$D CTAS=140 ALGOS=auto PROTOS=chunked STANDALONE= REPS=15 \
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $P --master-addr 127.0.0.1 --master-port 2951$P tools/probe_bw.py > $O/bw_p$P.log 2>&1; echo "bw P=$P rc=$?"; grep -A3 "^P=" $O/bw_p$P.log
done
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N bench.py --gpus $N --steps 50 --warmup 10 > $O/bench_n$N.log 2>&1; echo "bench N=$N rc=$?"
python - $O/bench_n$N.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(l['n_gpus'], round(l['ms_per_step'],4), json.dumps(l.get('calibration',{}).get('onbox', l.get('calibration')))[:400])
PY
done
