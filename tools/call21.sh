# 1-GPU: measure the Inception-v4 trace on a B200 (tools/inception_v4.py, batch 128)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2s; mkdir -p $O/traces
cp traces/META.json $O/traces/
timeout 900 python tools/extract_traces.py --out $O/traces --models inception_v4 > $O/extract.log 2>&1; echo "extract rc=$?"; tail -n 3 $O/extract.log
