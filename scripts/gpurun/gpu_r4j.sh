set -u
O=gpurun_out/r4j
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 10 > $O/bench.json 2> $O/bench.err
echo done
