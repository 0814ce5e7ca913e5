# 4-GPU: streamed protocol publication batches — single groups (P=4) and the BERT drain / iteration (N=4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2aa; mkdir -p $O
KNOBS="16,1,3072,512,8,4;16,1,3072,512,8,8;16,1,3072,512,8,16;16,1,3072,512,4,16;16,1,3072,512,2,16" PROTOS=stream SIZES_KB=16384,65536,131072,262144 ALGOS=twoshot CTAS=140 STANDALONE= timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 tools/probe_bw.py > $O/sweep_p4_stream.log 2>&1; echo "sweep rc=$?"
grep -v "^W\|^\s*$\|^\*\|OMP\|NCCL version" $O/sweep_p4_stream.log | tail -7
for B in 8,8 8,16 4,16; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 --steps 20 --warmup 3 --protocol stream --stream-batches $B > $O/bench_n4_stream_$B.log 2>&1; echo "bench stream $B rc=$?"
python - $O/bench_n4_stream_$B.log <<'PY'
import json,sys
l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']
print(round(l['ms_per_step'],4), {k:round(r[k],3) for k in ['achieved','frac','launch_ms_mean']}, {k:(round(v['iter_ms_median'],3), round(v.get('device_tail_us',0),1)) for k,v in l['strategies'].items()})
PY
done
