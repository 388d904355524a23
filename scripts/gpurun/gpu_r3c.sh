set -u
O=gpurun_out/r3c
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid.txt 2>&1
NNLS_NO_RESIDENT_LSQR=1 timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid_old.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --steps 10 > $O/bench.json 2> $O/bench.err
echo done
