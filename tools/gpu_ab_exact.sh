# exact mode: its GPU tests, then the single / tiny benches
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_exact.py tests/test_gpu_workloads.py -k "exact or single or tiny" > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
timeout 300 python bench.py --workload single --no-cpu-baseline > gpurun_out/ab_single.json 2> gpurun_out/ab_single.err
timeout 300 python bench.py --workload tiny --no-cpu-baseline > gpurun_out/ab_tiny.json 2> gpurun_out/ab_tiny.err
