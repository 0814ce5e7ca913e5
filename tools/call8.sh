cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2f; mkdir -p $O
timeout 600 python tools/dbg_stream.py > $O/dbg.log 2>&1; echo "dbg rc=$?"; cat $O/dbg.log | tail -40
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine_loopback.py -q -p no:faulthandler > $O/gpu.log 2>&1; echo "gpu tests rc=$?"
grep -E "passed|failed|FAILED" $O/gpu.log | tail -30
