set -u
O=gpurun_out/r4z
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for c in 2 1; do
timeout 300 python bench.py --config $c --no-extra --no-cpu-baseline --steps 20 > $O/bench_c$c.json 2> $O/bench_c$c.err
python -c "
import json; d=json.load(open('$O/bench_c$c.json')); print('c$c', d['value'], d['ms_per_step'], d['e2e']['value'], d['phase_ms_per_step']['upload'])" >> $O/summary.txt
done
echo done
