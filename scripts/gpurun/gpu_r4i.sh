set -u
O=gpurun_out/r4i
mkdir -p $O
timeout 120 python scripts/chol_reuse_profile.py 2 > $O/chol_reuse.txt 2>&1; echo "rc=$?" >> $O/chol_reuse.txt
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in 2 1 3; do
timeout 200 python bench.py --config $c --no-extra --no-cpu-baseline --no-e2e --steps 20 > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "
import json; d=json.load(open('$O/bench_c$c.json')); ps=d.get('per_solve',{}); print('c$c', d['value'], d['ms_per_step'], d['phase_ms_per_step']['chol_factor'], d['roofline']['frac'], [ (t['f'], t['kept']) for t in ps.get('trace',[])])" >> $O/summary.txt
done
echo done
