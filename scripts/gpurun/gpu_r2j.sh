set -u
O=gpurun_out/r2j
mkdir -p $O
timeout 300 python scripts/batched_profile.py 8192 > $O/batched_profile.log 2>&1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 50 python scripts/sanitize_run.py > $O/memcheck.log 2>&1
echo "rc=$?" >> $O/memcheck.log
echo done
