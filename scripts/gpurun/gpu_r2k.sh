set -u
O=gpurun_out/r2k
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "batch or config4" > $O/pytest.log 2>&1
timeout 300 python scripts/batched_profile.py 8192 > $O/batched_profile.log 2>&1
timeout 300 python bench.py --config 4 --no-extra --no-cpu-baseline --no-e2e --steps 5 > $O/b4.json 2> $O/b4.err
echo done
