# claim-ordered Gram kernel at config 2 raw: timing and one ncu --set full capture
set -u
O=gpurun_out/r4f
mkdir -p $O
timeout 600 python scripts/gram_raw_run.py 5 > $O/claim.log 2>&1; cat $O/claim.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gram_claim" --launch-skip 1 -c 1 \
  -o $O/full_c2raw_gram_claim -f python scripts/gram_raw_run.py 2 > $O/ncu.log 2>&1
echo done
