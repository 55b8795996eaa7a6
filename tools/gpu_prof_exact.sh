mkdir -p gpurun_out/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"exact_" -s 6 -c 6 -o gpurun_out/prof/single2 -f python tools/prof_exact.py single > gpurun_out/prof/single2.log 2>&1
