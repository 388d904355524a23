set -u
O=gpurun_out/r2m
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "reuse or restart or config2 or random or whole or factor" > $O/pytest.log 2>&1
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 10 > $O/bench.json 2> $O/bench.err
timeout 300 python scripts/chol_reuse_profile.py 2 > $O/reuse_c2.log 2>&1
echo done
