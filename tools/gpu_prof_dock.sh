# ncu --set full of the docking plan's kernels (one 4-rotation batch) and exact mode on Single
set -x
mkdir -p gpurun_out/prof
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"spread_z_kernel|pass_z_dk|pass_y_dk|fold_dk" -s 4 -c 4 -o gpurun_out/prof/dock -f python tools/prof_sweep.py docking 4 > gpurun_out/prof/dock.log 2>&1
timeout 600 $NCU -k regex:"exact_knot" -s 1 -c 1 -o gpurun_out/prof/single -f python tools/prof_exact.py single > gpurun_out/prof/single.log 2>&1
