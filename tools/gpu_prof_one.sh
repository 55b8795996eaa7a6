# ncu --set full with source of one kernel of a workload batch: $1 = kernel regex, $2 = workload, $3 = skip
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${3:-1} -c 1 \
  -o gpurun_out/prof/one -f python tools/prof_sweep.py $2 4 > gpurun_out/prof/one.log 2>&1
