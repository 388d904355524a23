set -u
O=gpurun_out/r5f
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "repeatable" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
