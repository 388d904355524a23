set -u
O=gpurun_out/r2y
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
NNLS_NO_FUSED_DUAL=1 timeout 300 python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 10 > $O/bench_nofuse.json 2> $O/bench_nofuse.err
echo done
