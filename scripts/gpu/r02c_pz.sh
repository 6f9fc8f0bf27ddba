timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_sharded.py tests/test_gpu_spec_criteria.py -x -q -p no:cacheprovider > gpurun_out/r02c_pz_tests.log 2>&1; tail -2 gpurun_out/r02c_pz_tests.log
timeout 900 python bench.py > gpurun_out/r02c_bench3.log 2>&1; tail -1 gpurun_out/r02c_bench3.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:cg_ --csv --log-file gpurun_out/r02c_cg_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/r02c_ncu_cg.log 2>&1; tail -2 gpurun_out/r02c_ncu_cg.log
