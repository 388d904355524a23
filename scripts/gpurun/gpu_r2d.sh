set -u
O=gpurun_out/r2d
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bench/mb_chol bench/microbench_chol_tile.cu > $O/mb_build.log 2>&1
timeout 120 ./bench/mb_chol > $O/mb_chol.log 2>&1
timeout 300 python scripts/chol_dag_profile.py 2 4000 > $O/dag_c2.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "normal_solve or config2 or factor or restart or reuse or whole or config" > $O/pytest.log 2>&1
timeout 300 python bench.py --no-extra --no-cpu-baseline --steps 10 > $O/bench.json 2> $O/bench.err
echo done
