set -u
O=gpurun_out/r2h
mkdir -p $O
CMD="python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lsqr_final_kernel -c 1 \
  -o $O/full_c2_lsqr -f $CMD > $O/ncu_lsqr.log 2>&1
ncu -i $O/full_c2_lsqr.ncu-rep --page source --csv > $O/lsqr_source.csv 2>&1
ncu -i $O/full_c2_lsqr.ncu-rep --page details --csv > $O/lsqr_details.csv 2>&1
echo done
