set -u
O=gpurun_out/r3s
mkdir -p $O
timeout 600 python bench.py --no-cpu-baseline --no-extra --steps 10 > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --no-cpu-baseline --no-extra --no-e2e --steps 10 > $O/bench2.json 2> $O/bench2.err
timeout 300 python scripts/chol_reuse_profile.py 2 > $O/chol_reuse.txt 2>&1
echo done
