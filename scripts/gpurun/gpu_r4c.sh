set -u
O=gpurun_out/r4c
mkdir -p $O
for c in 1 3; do
timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c$c.json 2> $O/bench_c$c.err
NNLS_NO_SORT_CSC=1 timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c${c}_nosort.json 2> $O/bench_c${c}_nosort.err
done
echo done
