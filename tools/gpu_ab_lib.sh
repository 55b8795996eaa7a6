# A/B of the in-tree library against an alternative build (lib_$1) on workloads $2...; then tests
ALT=$1; shift
for W in "$@"; do
for r in 1 2; do
  for v in main $ALT; do
    if [ $v = main ]; then unset BALLCORR_LIB; else export BALLCORR_LIB=$PWD/paper_1711_05075_b200/lib_$v/libballcorr.so; fi
    python bench.py --workload $W --no-cpu-baseline --steps 3 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); n = d['config']['rotations_per_rank']
print('$W', '$v', d['value'], {k: round(v / n, 5) for k, v in d['stages_ms_per_step'].items()})" >> gpurun_out/ab_lib.log
  done
done
done
unset BALLCORR_LIB
[ -n "$TESTS" ] && timeout 1500 python -m pytest -q -p no:cacheprovider $TESTS > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
