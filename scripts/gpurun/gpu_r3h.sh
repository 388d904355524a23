set -u
O=gpurun_out/r3h
mkdir -p $O
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid.txt 2>&1
timeout 300 python scripts/chol_reuse_profile.py 2 > $O/chol_reuse.txt 2>&1
NNLS_RESTART_HALVES=1 timeout 300 python scripts/chol_reuse_profile.py 2 > $O/chol_reuse_h1.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 10 > $O/bench.json 2> $O/bench.err
NNLS_RESTART_HALVES=1 timeout 600 python bench.py --no-cpu-baseline --no-extra --no-e2e --steps 10 > $O/bench_h1.json 2> $O/bench_h1.err
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
