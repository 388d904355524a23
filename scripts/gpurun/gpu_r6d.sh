set -u
O=gpurun_out/r6d
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -x -q -k "batch or smoke or adaptive" > $O/pytest_batched.log 2>&1; echo "rc=$?" >> $O/pytest_batched.log
timeout 600 python bench.py --config 4 --no-cpu-baseline --no-extra > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python scripts/batched_profile.py > $O/batched_profile.txt 2>&1
CMD="python bench.py --config 4 --batch 16384 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
for k in batched_lsqr_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$k\$" --launch-skip 2 -c 1 \
    -o $O/full_c4_$k -f $CMD > $O/ncu_$k.log 2>&1
done
echo done
