set -u
O=gpurun_out/r5b
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 20 > $O/bench_c2.json 2> $O/bench_c2.err
python -c "
import json; d=json.load(open('$O/bench_c2.json')); print('c2', d['value'], d['ms_per_step'], d['e2e']['value'], d['phase_ms_per_step']['csc'])" >> $O/summary.txt
echo done
