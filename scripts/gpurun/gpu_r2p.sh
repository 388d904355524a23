set -u
O=gpurun_out/r2p
mkdir -p $O
CMD="python bench.py --no-extra --no-cpu-baseline --no-e2e --steps 1 --warmup 3"
for k in dual_kernel chol_backsolve_kernel gram_exact_kernel lsqr_final_kernel decide_kernel; do
  timeout 600 ncu --set full --clock-control none -k regex:$k -c 1 -o $O/full_c2_$k -f $CMD > $O/ncu_$k.log 2>&1
done
python - <<'PY' > $O/dense1000.log 2>&1
import numpy as np, torch, nnls_gen as g, paper_cs_0408029_b200 as P
prob = g.make_fig2(1000, 1.0, 0)
S = P.setup(prob); S.solve()
P.timing_enable(S.h, True)
S.load_problem(prob); x, info = S.solve()
print(info)
print({k: v for k, v in P.timing_read(S.h).items() if v[1]})
PY
echo done
