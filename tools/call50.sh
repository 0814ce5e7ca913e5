# 4-GPU: multirank re-check (NVLS plain all-reduce fix) + comm-bound regime refresh (call49)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2vv; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "mr rc=$?"; tail -n 1 $O/mr.log; grep MULTIRANK $O/mr.log | head -3
bash tools/call49.sh
