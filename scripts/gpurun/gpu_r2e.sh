set -u
O=gpurun_out/r2e
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
CMD="python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
timeout 300 $CMD > $O/plain.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_factor_kernel -c 1 \
  -o $O/full_c2_chol_factor -f $CMD > $O/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches_c2.csv $CMD > $O/ncu_launch.log 2>&1
ncu -i $O/full_c2_chol_factor.ncu-rep --page raw --csv > $O/full_c2_chol_factor_raw.csv 2>&1
echo done
