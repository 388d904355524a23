set -u
O=gpurun_out/r6b
mkdir -p $O
CMD="python bench.py --config 4 --batch 16384 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-extra"
timeout 300 $CMD > $O/plain_c4.json 2>&1 || exit 1
for k in batched_lsqr_kernel batched_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$k\$" --launch-skip 2 -c 1 \
    -o $O/full_c4_$k -f $CMD > $O/ncu_$k.log 2>&1
done
echo done
