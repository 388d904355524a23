set -u
O=gpurun_out/r2i
mkdir -p $O
for cfg in "1 0 0" "8 4 4" "8 3 5" "8 5 3" "16 4 4" "4 4 4" "8 0 0"; do
  set -- $cfg
  NNLS_BATCH_SPLIT=$1 NNLS_BATCH_PSM=$2 NNLS_BATCH_LSM=$3 timeout 300 python bench.py --config 4 --no-extra --no-cpu-baseline --no-e2e --steps 5 > $O/b4_$1_$2_$3.json 2> $O/b4_$1_$2_$3.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "batch or config4" > $O/pytest.log 2>&1
echo done
