set -u
O=gpurun_out/r3v
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 10 > $O/bench.json 2> $O/bench.err
timeout 300 python scripts/chol_reuse_profile.py 2 > $O/chol_reuse.txt 2>&1
echo done
