# 4-GPU: bounds-checked build + GPU suites (1 GPU) + multirank (P=2/4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ag bash tools/bounds_check.sh
