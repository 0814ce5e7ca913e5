# 4-GPU: NVLS probe v2 (in-kernel iterations, out-of-place, inputs read back for the bit-exact check)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2nn; mkdir -p $O
for P in 2 4; do timeout 300 ./tools/nvls_probe $P > $O/nvls_p$P.log 2>&1; echo "nvls P=$P rc=$?"; cat $O/nvls_p$P.log | head -60; done
