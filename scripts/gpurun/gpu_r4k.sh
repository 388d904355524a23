# claim-ordered Gram: the epoch restart exercised (threshold 40 epochs, a rebuilt library), then the normal build again
set -u
O=gpurun_out/r4k
mkdir -p $O
NNLS_EXTRA_NVCC_FLAGS="-DNNLS_CLAIM_EPOCH_MAX=40" python paper_cs_0408029_b200/build.py --force > $O/build_small.log 2>&1 || { tail $O/build_small.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "gram" > $O/pytest_small.log 2>&1; echo "rc=$?" >> $O/pytest_small.log
tail -3 $O/pytest_small.log
python paper_cs_0408029_b200/build.py --force > $O/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "gram" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python scripts/gram_raw_run.py 5 2>&1 | grep -v checksum
echo done
