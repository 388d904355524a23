set -u
O=gpurun_out/prof
mkdir -p $O
for k in chol_factor_kernel chol_backsolve_kernel lsqr_cluster_kernel gram_exact_kernel dual_kernel decide_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 \
    -o $O/full_c1_$k -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_full_$k.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_factor_kernel -c 1 \
  -o $O/full_c2_chol_factor_kernel -f python bench.py --config 2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > $O/ncu_full_c2.log 2>&1
ls -la $O
