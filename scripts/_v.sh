for v in "" "-DNO_ORDER_SORT"; do
  NNLS_EXTRA_NVCC_FLAGS="$v" python -c "from paper_cs_0408029_b200 import build; build.build(force=True)"
  tag=$(echo "x$v" | tr -d ' -')
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decide" -c 10 --csv --log-file gpurun_out/dec_$tag.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
