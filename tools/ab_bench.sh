#!/usr/bin/env bash
# A/B timing of library builds on the GPU box: alternates bench.py between the in-tree
# libballcorr.so ("main") and alternative builds, printing throughput and per-stage ms/rotation.
#   make LIB=paper_1711_05075_b200/lib_alt/libballcorr.so OBJDIR=build/obj_alt \
#        paper_1711_05075_b200/lib_alt/libballcorr.so          # from a patched tree
#   gpurun -- 'bash tools/ab_bench.sh alt'                      # lib_<name> per argument
set -u
names=("$@")
for round in 1 2; do
  for v in main "${names[@]}"; do
    if [ "$v" = main ]; then unset BALLCORR_LIB; else export BALLCORR_LIB=$PWD/paper_1711_05075_b200/lib_$v/libballcorr.so; fi
    python bench.py --no-cpu-baseline 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); n = d['config']['rotations_per_rank']
print('$v', round(d['value'] / 1e10, 4), {k: round(v / n, 5) for k, v in d['stages_ms_per_step'].items()})"
  done
done
