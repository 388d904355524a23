set -u
O=gpurun_out/r2v
mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "grid or no_cluster or NO_CLUSTER" > $O/pytest_small.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "lsqr or config2 or grid or whole or fig2 or notpd" > $O/pytest.log 2>&1
timeout 200 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid_c2.log 2>&1
timeout 200 python bench.py --no-extra --no-cpu-baseline --steps 10 > $O/bench.json 2> $O/bench.err
echo done
