set -u
O=gpurun_out/r4d
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in 1 3 2; do
timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c$c.json 2> $O/bench_c$c.err
done
echo done
