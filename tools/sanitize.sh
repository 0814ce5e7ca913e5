#!/bin/bash
# compute-sanitizer over the fused kernels (tools/sanitize_host.c): loopback
# P = 1/2/4/8, standalone group launches + the engine drain, tools memcheck,
# racecheck, synccheck, initcheck. Logs: $OUT/san_<tool>_P<P>.log.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=${OUT:-gpurun_out/r2}
mkdir -p "$OUT"
CUDA=${CUDA_HOME:-/usr/local/cuda}
LIB=$PWD/paper_1912_09268_b200/lib
gcc -std=c11 -O2 -Wall -Iinclude -I$CUDA/include tools/sanitize_host.c -o "$OUT/sanitize_host" \
    -L$LIB -lmgwfbp -L$CUDA/lib64 -lcudart -Wl,-rpath,$LIB -Wl,-rpath,$CUDA/lib64 || exit 1
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for P in ${PS:-1 2 4 8}; do
    timeout 900 $CUDA/bin/compute-sanitizer --tool $tool --error-exitcode 9 "$OUT/sanitize_host" $P \
      > "$OUT/san_${tool}_P$P.log" 2>&1
    echo "$tool P=$P rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|mismatches' "$OUT/san_${tool}_P$P.log" | tr '\n' ' ')"
  done
done
