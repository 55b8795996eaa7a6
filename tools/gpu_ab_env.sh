# A/B of an environment switch on one workload: $1 = variable, $2 = workload; then its tests
W=$2
for r in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export $1=1; else unset $1; fi
    python bench.py --workload $W --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); n = d['config']['rotations_per_rank']
print('$v', d['value'], {k: round(v / n, 5) for k, v in d['stages_ms_per_step'].items()})" >> gpurun_out/ab_env.log
  done
done
unset $1
[ -n "$TESTS" ] && timeout 1200 python -m pytest -q -p no:cacheprovider $TESTS > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
