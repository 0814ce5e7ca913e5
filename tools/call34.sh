cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2dd; mkdir -p $O
python tools/drain_probe.py --trace googlenet --P 1 --iters 3 --stamps > $O/drain_gn.log 2>&1; echo "rc=$?"; grep "CTA\|span" $O/drain_gn.log | cut -c1-1500
