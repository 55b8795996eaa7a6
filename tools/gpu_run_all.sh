set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload docking --no-cpu-baseline > gpurun_out/bench_docking.json 2> gpurun_out/bench_docking.err
timeout 600 python bench.py --workload single --no-cpu-baseline > gpurun_out/bench_single.json 2> gpurun_out/bench_single.err
timeout 600 python bench.py --workload tiny --no-cpu-baseline > gpurun_out/bench_tiny.json 2> gpurun_out/bench_tiny.err
timeout 600 python bench.py --workload torus --no-cpu-baseline > gpurun_out/bench_torus.json 2> gpurun_out/bench_torus.err
