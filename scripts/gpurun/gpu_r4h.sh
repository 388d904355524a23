# claim-ordered Gram: one barrier per pass (parity tags, 1024 threads) vs two barriers (512 threads): tests + timing
set -u
O=gpurun_out/r4h
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "gram" > $O/pytest_gram.log 2>&1; echo "rc=$?" >> $O/pytest_gram.log
tail -3 $O/pytest_gram.log
NNLS_CLAIM_TWO_BARRIERS=1 timeout 900 python -m pytest tests -m gpu -q -x -k "gram" > $O/pytest_gram2.log 2>&1; echo "rc=$?" >> $O/pytest_gram2.log
tail -3 $O/pytest_gram2.log
for TB in 0 1; do
  echo "two_barriers=$TB config 2 raw"; NNLS_CLAIM_TWO_BARRIERS=$TB timeout 600 python scripts/gram_raw_run.py 5 2>&1 | grep -v checksum
  for N in 4000 6000 12000; do
    D=$(python -c "print(40.0/$N)")
    echo "two_barriers=$TB n=$N"; M=$((5*N)) N=$N D=$D NNLS_CLAIM_TWO_BARRIERS=$TB timeout 600 python scripts/gram_raw_run.py 5 2>&1 | grep -v checksum
  done
done
echo done
