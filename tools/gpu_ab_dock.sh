# docking plan: parity tests that cover its kernels, then the docking bench (stage times)
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_bandpin.py tests/test_gpu_workloads.py tests/test_gpu_complementarity.py -k "dock or complementarity" > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
timeout 600 python bench.py --workload docking --no-cpu-baseline --steps 3 > gpurun_out/ab_docking.json 2> gpurun_out/ab_docking.err
