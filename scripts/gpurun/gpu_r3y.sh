set -u
O=gpurun_out/r3y2
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 10 > $O/bench.json 2> $O/bench.err
echo done
