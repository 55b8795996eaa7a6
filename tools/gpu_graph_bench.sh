for w in tiny single; do
  for st in 5 200; do
    python bench.py --workload $w --no-cpu-baseline --steps $st 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', $st, d['value'], d['ms_per_step'], d['gpu_launches'], d['config']['cuda_graph'], d['e2e']['value'])" >> gpurun_out/gb.log
  done
  python bench.py --workload $w --no-cpu-baseline --steps 200 --graph off 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w off', d['value'], d['ms_per_step'], d['gpu_launches'], d['config']['cuda_graph'])" >> gpurun_out/gb.log
done
