set -u
O=gpurun_out/r4x
mkdir -p $O
timeout 300 python scripts/chol_dag_profile.py 2 3981 > $O/dag_c2.txt 2>&1
echo done
