set -u
O=gpurun_out/r2u
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "lsqr or config2 or grid or whole or fig2 or notpd" > $O/pytest.log 2>&1
timeout 300 python scripts/lsqr_grid_profile.py 2 > $O/lsqr_grid_c2.log 2>&1
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 10 > $O/bench.json 2> $O/bench.err
NNLS_LSQR_NOBLK=1 timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 10 > $O/bench_noblk.json 2> $O/bench_noblk.err
echo done
