# batched LSQR: the norm estimates kept by thread 0 alone -- batched tests and the config-4 bench
set -u
O=gpurun_out/r4i
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "batched or config4" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python bench.py --config 4 --no-extra --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
python -c "
import json; d=json.loads(open('$O/bench_c4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('phase_ms_per_step'))"
echo done
