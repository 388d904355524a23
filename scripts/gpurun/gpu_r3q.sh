set -u
O=gpurun_out/r3q
mkdir -p $O
timeout 300 python scripts/chol_dag_profile.py 2 3981 > $O/dag_c2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 10 > $O/bench.json 2> $O/bench.err
echo done
