# the ordered Gram kernel at config 2 with unquantized values: phase times and one ncu --set full capture
set -u
O=gpurun_out/r4d
mkdir -p $O
timeout 600 python scripts/gram_raw_run.py 5 > $O/plain.log 2>&1 || { cat $O/plain.log; exit 1; }
cat $O/plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gram_kernel" --launch-skip 1 -c 1 \
  -o $O/full_c2raw_gram_kernel -f python scripts/gram_raw_run.py 2 > $O/ncu.log 2>&1
echo done
