set -u
O=gpurun_out/r2x
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 120 env LD_LIBRARY_PATH=/usr/local/cuda/lib64 ./bench/yardstick_cusolver > $O/yardstick.json 2> $O/yardstick.err
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
NNLS_NO_FUSED_DUAL=1 timeout 300 python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 10 > $O/bench_nofuse.json 2> $O/bench_nofuse.err
echo done
