#!/bin/bash
# One `ncu --set full` capture per hot kernel (config 1; chol_factor also at
# config 2), each after the same command exited 0 without ncu.
set -u
O=gpurun_out/prof
mkdir -p $O
CMD1="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
CMD2="python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 $CMD1 > $O/plain_c1.json 2>&1 || exit 1
for k in chol_factor_kernel lsqr_cluster_kernel chol_backsolve_kernel dual_kernel decide_kernel gram_kernel lsqr_plan_kernel; do
  timeout 600 ncu --set full --import-source on --clock-control none -k $k --launch-skip 2 -c 1 \
    -o $O/full_c1_$k -f $CMD1 > $O/ncu_$k.log 2>&1
done
timeout 300 $CMD2 > $O/plain_c2.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none -k chol_factor_kernel --launch-skip 2 -c 1 \
  -o $O/full_c2_chol_factor_kernel -f $CMD2 > $O/ncu_c2.log 2>&1
echo done
