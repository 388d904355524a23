# claim-ordered vs warp-per-row Gram (unquantized values): crossover in n (m = 5 n, ~40 entries per row)
set -u
O=gpurun_out/r4g
mkdir -p $O
for N in 2048 3000 4000 6000 12000 16000; do
  D=$(python -c "print(40.0/$N)")
  for MIN in 1 1000000; do
    echo "n=$N min_n=$MIN" >> $O/sweep.log
    M=$((5*N)) N=$N D=$D NNLS_CLAIM_MIN_N=$MIN timeout 600 python scripts/gram_raw_run.py 5 >> $O/sweep.log 2>&1
  done
done
cat $O/sweep.log
