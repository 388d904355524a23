set -u
O=gpurun_out/r5g
mkdir -p $O
timeout 300 python scripts/chol_dag_profile.py 2 3981 > $O/dag_c2.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in 2 2 1; do
timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "
import json; d=json.load(open('$O/bench_c$c.json')); print('c$c', d['value'], d['ms_per_step'], d['phase_ms_per_step']['chol_solve'])" >> $O/summary.txt
done
NNLS_BS_RING=1 timeout 300 python bench.py --config 2 --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_ring.json 2> $O/bench_ring.err
python -c "
import json; d=json.load(open('$O/bench_ring.json')); print('ring', d['value'], d['ms_per_step'], d['phase_ms_per_step']['chol_solve'])" >> $O/summary.txt
echo done
