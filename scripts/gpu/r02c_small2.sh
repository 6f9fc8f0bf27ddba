timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_spec_criteria.py tests/test_gpu_large_configs.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python scripts/small_n.py C1 > gpurun_out/r02c_small_C1b.log 2>&1; cat gpurun_out/r02c_small_C1b.log
timeout 600 python scripts/prof_small.py C1 > gpurun_out/r02c_prof_C1b.log 2>&1; grep -E "pivchol|precond_factor|xtx|span" gpurun_out/r02c_prof_C1b.log
