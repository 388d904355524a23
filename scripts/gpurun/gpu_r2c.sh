set -u
O=gpurun_out/r2c
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bench/mb_chol bench/microbench_chol_tile.cu > $O/mb_build.log 2>&1
timeout 120 ./bench/mb_chol > $O/mb_chol.log 2>&1
timeout 300 python scripts/chol_dag_profile.py 2 4000 > $O/dag_c2.log 2>&1
echo done
