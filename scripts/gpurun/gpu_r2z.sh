set -u
O=gpurun_out/r2z
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid.txt 2>&1
timeout 300 python scripts/chol_reuse_profile.py 2 > $O/chol_reuse.txt 2>&1
echo done
