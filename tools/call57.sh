# 1-GPU: final GPU suite (incl. the NVLS guard-rail test) + smoke on the final code
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ad; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED|Error" $O/gpu.log | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 $O/smoke.log
