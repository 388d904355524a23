set -u
O=gpurun_out/r4k
mkdir -p $O
timeout 600 python -m pytest tests -m gpu -q -k "batch" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python scripts/batched_profile.py 65536 > $O/bprof.txt 2>&1
timeout 300 python bench.py --config 4 --no-cpu-baseline --no-extra --steps 5 > $O/bench_c4.json 2> $O/bench_c4.err
python -c "
import json; d=json.load(open('$O/bench_c4.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['phase_ms_per_step'])" > $O/summary.txt
echo done
