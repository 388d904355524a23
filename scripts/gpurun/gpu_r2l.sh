set -u
O=gpurun_out/r2l
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "adaptive or notpd" > $O/pytest_next2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --config 4 --no-extra --no-cpu-baseline --no-e2e --steps 5 > $O/b4.json 2> $O/b4.err
echo done
