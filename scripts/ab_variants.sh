set -u
run() { timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c1', d['value'])"; timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c2', d['value'])"; timeout 200 python scripts/chol_dag_profile.py 2>&1 | grep "potrf\|period"; }
echo BASE; run
for v in "$@"; do echo "VARIANT $v"; NNLS_EXTRA_NVCC_FLAGS="$v" python -c "from paper_cs_0408029_b200 import build; build.build(force=True)" && run; done
