# 4-GPU: bounds-checked build incl. the NVLS kernel (GPU suite + multirank with NVLS), then the normal build: multirank + smoke
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2ai bash tools/bounds_check.sh
make -C paper_1912_09268_b200/csrc clean > /dev/null; make -C paper_1912_09268_b200/csrc > gpurun_out/r2ai/build_normal.log 2>&1; echo "normal build rc=$?"
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/r2ai/mr_normal.log 2>&1; echo "mr (normal) rc=$?"; tail -n 1 gpurun_out/r2ai/mr_normal.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -m gpu -q -p no:faulthandler > gpurun_out/r2ai/gpu_normal.log 2>&1; echo "gpu suite (normal) rc=$?"; tail -n 1 gpurun_out/r2ai/gpu_normal.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ai/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/r2ai/smoke.log
