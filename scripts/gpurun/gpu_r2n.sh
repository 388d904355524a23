set -u
O=gpurun_out/r2n
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python scripts/fig1_sweep.py --out $O/fig1_sweep.json > $O/fig1.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo done
