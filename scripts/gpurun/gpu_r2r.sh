set -u
O=gpurun_out/r2r
mkdir -p $O
CMD="python bench.py --config 4 --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:batched_lsqr_kernel -c 1 -o $O/b4_lsqr -f $CMD > $O/ncu_lsqr.log 2>&1
ncu -i $O/b4_lsqr.ncu-rep --page source --csv --print-source cuda,sass > $O/b4_lsqr_source.csv 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"^batched_kernel|nnls::batched_kernel" -c 1 -o $O/b4_pivot -f $CMD > $O/ncu_pivot.log 2>&1
ncu -i $O/b4_pivot.ncu-rep --page source --csv --print-source cuda,sass > $O/b4_pivot_source.csv 2>&1
echo done
