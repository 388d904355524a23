set -u
O=gpurun_out/r4h
mkdir -p $O
for c in 2 1 3; do
timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "
import json; d=json.load(open('$O/bench_c$c.json')); ps=d.get('per_solve',{}); print('c$c', d['value'], d['ms_per_step'], d['phase_ms_per_step']['chol_factor'], [ (t['f'], t['kept']) for t in ps.get('trace',[])])" >> $O/summary.txt
NNLS_ORDER_MODE=1 timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c${c}_m1.json 2> $O/bench_c${c}_m1.err
python -c "
import json; d=json.load(open('$O/bench_c${c}_m1.json')); ps=d.get('per_solve',{}); print('c$c m1', d['value'], d['ms_per_step'], d['phase_ms_per_step']['chol_factor'], [ (t['f'], t['kept']) for t in ps.get('trace',[])])" >> $O/summary.txt
done
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
echo done
