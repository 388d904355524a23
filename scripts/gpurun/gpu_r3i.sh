set -u
O=gpurun_out/r3i
mkdir -p $O
timeout 300 python scripts/batched_profile.py 65536 > $O/bprof.txt 2>&1
timeout 300 python bench.py --config 4 --no-cpu-baseline --no-extra --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
echo done
