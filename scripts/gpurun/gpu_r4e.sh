# claim-ordered Gram kernel: bitwise tests, config-2 raw timing against the warp-per-row kernel
set -u
O=gpurun_out/r4e
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "gram" > $O/pytest_gram.log 2>&1; echo "rc=$?" >> $O/pytest_gram.log
tail -5 $O/pytest_gram.log
timeout 600 python scripts/gram_raw_run.py 5 > $O/claim.log 2>&1; cat $O/claim.log
NNLS_CLAIM_MIN_N=1000000 timeout 600 python scripts/gram_raw_run.py 5 > $O/warp.log 2>&1; cat $O/warp.log
CFG=3 timeout 600 python scripts/gram_raw_run.py 5 > $O/claim_c3.log 2>&1; cat $O/claim_c3.log
CFG=3 NNLS_CLAIM_MIN_N=1 timeout 600 python scripts/gram_raw_run.py 5 > $O/claim_c3f.log 2>&1; cat $O/claim_c3f.log
CFG=1 timeout 600 python scripts/gram_raw_run.py 5 > $O/claim_c1.log 2>&1; cat $O/claim_c1.log
CFG=1 NNLS_CLAIM_MIN_N=1 timeout 600 python scripts/gram_raw_run.py 5 > $O/claim_c1f.log 2>&1; cat $O/claim_c1f.log
echo done
