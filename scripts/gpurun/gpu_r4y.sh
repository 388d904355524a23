set -u
O=gpurun_out/r4y
mkdir -p $O
for c in 1 3; do
timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c$c.json 2> $O/bench_c$c.err
NNLS_NO_CLUSTER=1 timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c${c}_nc.json 2> $O/bench_c${c}_nc.err
for f in bench_c$c bench_c${c}_nc; do python -c "
import json; d=json.load(open('$O/$f.json')); print('$f', d['value'], d['ms_per_step'], d['phase_ms_per_step']['lsqr'], d['per_solve']['lsqr_iterations'])" >> $O/summary.txt; done
done
echo done
