mkdir -p gpurun_out/prof
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"exact_bin" -s 4 -c 4 -o gpurun_out/prof/single3 -f python tools/prof_exact.py single > gpurun_out/prof/single3.log 2>&1
