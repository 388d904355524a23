set -u
O=gpurun_out/r2q
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "fig2 or dense or gram or shard" > $O/pytest.log 2>&1
timeout 900 python scripts/fig2_sweep.py --out $O/fig2_sweep.json > $O/fig2.log 2>&1
echo done
