set -x
mkdir -p gpurun_out/prof
NCU="ncu --set full --clock-control none --import-source on"
timeout 900 $NCU -k regex:"spread_z_kernel|pass_z_dk|pass_y_dk|fold_dk" -s 5 -c 5 -o gpurun_out/prof/dock2 -f python tools/prof_sweep.py docking 4 > gpurun_out/prof/dock2.log 2>&1
