# claim-ordered Gram at the top of its range (n = 17000: 204 KB of dynamic shared memory, one CTA per SM) vs the warp kernel
set -u
O=gpurun_out/r4l
mkdir -p $O
for MIN in 1 1000000; do
  echo "n=17000 min_n=$MIN" >> $O/log.txt
  M=34000 N=17000 D=0.00235 NNLS_CLAIM_MIN_N=$MIN timeout 900 python scripts/gram_raw_run.py 2 >> $O/log.txt 2>&1
done
cat $O/log.txt
