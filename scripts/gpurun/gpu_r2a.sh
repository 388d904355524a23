set -u
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi -q | grep -iE "product name|clocks|SM  " | head -20 > $O/smi.txt
nproc > $O/nproc.txt
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 300 python bench.py --config 4 --steps 5 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --config 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
echo done
