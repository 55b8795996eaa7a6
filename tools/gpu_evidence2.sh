# Per-config evidence refresh: bench lines of the non-headline configs and an ncu --set full
# summary of the docking plan's kernels (summarised on the box).
set -x
E=gpurun_out/ev2; mkdir -p $E
for w in docking single tiny torus; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $E/bench_$w.json 2> $E/bench_$w.err
done
timeout 900 ncu --set full --clock-control none -k regex:"spread_z_kernel|pass_z_dk|pass_y_dk|fold_dk" -s 5 -c 5 \
  -o /tmp/dock -f python tools/prof_sweep.py docking 4 > $E/ncu_dock.log 2>&1
python - <<'PY' > $E/ncu_docking.md
import sys; sys.path.insert(0, "tools")
from summarize_ncu import full_metrics
print("# ncu --set full: docking plan kernels, one 4-rotation batch (`tools/prof_sweep.py docking 4`, `tools/gpu_evidence2.sh`)\n")
for d in full_metrics("/tmp/dock.ncu-rep"):
    print(f"## `{d['kernel']}`")
    for k, v in d.items():
        if k == "kernel": continue
        print(f"- top stalls: {v}" if k == "top_stalls" else f"- {k}: {v[0]} {v[1]}")
    print()
PY
