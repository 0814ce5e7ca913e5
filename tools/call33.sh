cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2cc; mkdir -p $O
python tools/drain_probe.py --trace googlenet --P 1 --iters 3 --stamps > $O/drain_gn.log 2>&1; echo "rc=$?"; tail -n 3 $O/drain_gn.log | cut -c1-250
python tools/drain_probe.py --trace densenet201 --P 1 --iters 3 > $O/drain_dn.log 2>&1; tail -n 1 $O/drain_dn.log | cut -c1-250
timeout 1500 python -m pytest tests -m gpu -q -p no:faulthandler -x > $O/gpu.log 2>&1; echo "gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/gpu.log | tail -5
