# ncu --set full of the two config-4 batched kernels (8192-problem batch): hot SASS and stall reasons
set -u
O=gpurun_out/r4c
mkdir -p $O
CMD="python bench.py --config 4 --batch 8192 --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
timeout 600 $CMD > $O/plain.json 2> $O/plain.err || exit 1
for k in batched_lsqr_kernel batched_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^$k" -c 1 \
    -o $O/full_c4_$k -f $CMD > $O/ncu_$k.log 2>&1
done
echo done
