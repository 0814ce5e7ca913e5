# 1-GPU: full GPU suite (new bf16 engine / CE tests)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2u; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED|Error" $O/gpu.log | tail -15
