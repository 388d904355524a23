set -u
O=gpurun_out/r2f
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid_c2.log 2>&1
timeout 300 python scripts/chol_reuse_profile.py 2 > $O/reuse_c2.log 2>&1
echo done
