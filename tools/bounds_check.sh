#!/bin/bash
# Memory-safety run in place of compute-sanitizer (closed on this pool):
# rebuild libmgwfbp.so with device bounds checks at every remote-write site
# (-DMGW_BOUNDS_CHECK: TMA / register pushes into peer arenas, all-gather
# stores, LL packet slots, barrier flag indices; a violation traps), then run
# the GPU parity suites against the checked build. The box is scratch: the
# checked .so never comes back.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=${O:-gpurun_out/bounds}; mkdir -p $O
make -C paper_1912_09268_b200/csrc clean > /dev/null
make -C paper_1912_09268_b200/csrc EXTRA_NVCC=-DMGW_BOUNDS_CHECK > $O/build.log 2>&1; echo "checked build rc=$?"
strings paper_1912_09268_b200/lib/libmgwfbp.so | grep -c "MGW_BOUNDS_CHECK failed" | sed 's/^/bounds-check format strings in the .so: /'
CUDA_VISIBLE_DEVICES=0 timeout 1800 python -m pytest tests -m gpu -q -p no:faulthandler -rs > $O/gpu.log 2>&1; echo "gpu suite (checked) rc=$?"; grep -E "passed|failed" $O/gpu.log | tail -2
NG=$(nvidia-smi -L | wc -l)
if [[ $NG -ge 2 ]]; then
  timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -rs > $O/mr.log 2>&1; echo "multirank (checked) rc=$?"; tail -n 1 $O/mr.log
fi
grep -h "MGW_BOUNDS_CHECK failed" $O/*.log | head -5; echo "bounds violations: $(cat $O/*.log | grep -c 'MGW_BOUNDS_CHECK failed')"
