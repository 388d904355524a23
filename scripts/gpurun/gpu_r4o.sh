set -u
O=gpurun_out/r4o
mkdir -p $O
nvidia-smi -q -d CLOCK > $O/smi_clock.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as e; e.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
CMD="python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
timeout 300 $CMD > $O/plain.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches_c2.csv $CMD > $O/ncu_launch.log 2>&1
for k in chol_factor_kernel lsqr_resident_kernel dual_kernel chol_backsolve_kernel gram_exact_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o $O/full_c2_$k -f $CMD > $O/ncu_$k.log 2>&1
done
echo done
