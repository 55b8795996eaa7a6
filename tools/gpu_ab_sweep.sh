# sweep plan: the parity tests that cover its kernels, then the sweep bench with and without
# an environment switch (A/B of two kernel variants in one library: $1 = variable name)
[ -n "$SKIP_TESTS" ] || timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_bandpin.py tests/test_gpu_workloads.py tests/test_gpu_fullgrid.py -k "sweep" > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
for r in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export $1=1; else unset $1; fi
    python bench.py --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); n = d['config']['rotations_per_rank']
print('$v', round(d['value'] / 1e10, 4), d['roofline']['frac'], {k: round(v / n, 5) for k, v in d['stages_ms_per_step'].items()})" >> gpurun_out/ab_sweep.log
  done
done
