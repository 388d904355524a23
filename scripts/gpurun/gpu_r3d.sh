set -u
O=gpurun_out/r3d
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid.txt 2>&1
timeout 300 python scripts/lsqr_c2_run.py 2 > $O/run.txt 2>&1 || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:lsqr_resident -s 1 -c 1 -o $O/lsqr_res -f python scripts/lsqr_c2_run.py 2 > $O/ncu.log 2>&1
echo done
