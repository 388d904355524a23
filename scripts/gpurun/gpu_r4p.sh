set -u
O=gpurun_out/r4p
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "config2 or lsqr" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
