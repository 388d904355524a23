set -u
O=gpurun_out/r5c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "large" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
