set -u
O=gpurun_out/r2o
mkdir -p $O
timeout 900 python scripts/fig2_sweep.py --out $O/fig2_sweep.json > $O/fig2.log 2>&1
echo done
