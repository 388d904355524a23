set -u
O=gpurun_out/r5d
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid.txt 2>&1
echo done
