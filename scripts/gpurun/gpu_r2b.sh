# round 2: tests, smoke, default bench (config 2 + other configs), reference arm
set -u
O=gpurun_out/r2b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
echo done
