# claim-ordered Gram with long columns (segments): tall problems, unquantized values
set -u
O=gpurun_out/r4j
mkdir -p $O
for SH in "200000 8000 0.005" "100000 4000 0.01" "400000 12000 0.003"; do
  set -- $SH
  for MIN in 1 1000000; do
    echo "m=$1 n=$2 d=$3 min_n=$MIN" >> $O/sweep.log
    M=$1 N=$2 D=$3 NNLS_CLAIM_MIN_N=$MIN timeout 900 python scripts/gram_raw_run.py 3 2>&1 | grep -v checksum >> $O/sweep.log
  done
done
cat $O/sweep.log
