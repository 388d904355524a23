#!/bin/bash
# Runs on the GPU box (gpurun): bench lines for configs 1-4, the ncu launch
# list of config 1 and one `ncu --set full` capture of the top kernels.
# Output under gpurun_out/prof/; summarise locally into profiles/.
set -u
mkdir -p gpurun_out/prof
O=gpurun_out/prof
timeout 600 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --config 3 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c1.json 2> $O/bench_ref_c1.err
# launch list (cold-cache, serialised) of the same command as the bench value pass
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
# full capture of the dominant kernels: one launch of each, one ncu run per
# kernel (a single regex with -c N would stop at the first N matches)
for k in chol_factor_kernel chol_backsolve_kernel lsqr_cluster_kernel gram_exact_kernel dual_kernel decide_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 \
    -o $O/full_c1_$k -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > $O/ncu_full_$k.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_factor_kernel -c 1 \
  -o $O/full_c2_chol_factor_kernel -f python bench.py --config 2 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
  > $O/ncu_full_c2.log 2>&1
for k in batched_kernel batched_lsqr_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" --launch-skip 1 -c 1 \
    -o $O/full_c4_$k -f python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > $O/ncu_full_c4_$k.log 2>&1
done
echo done
