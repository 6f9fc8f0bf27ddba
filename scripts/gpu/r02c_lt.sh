TAIL=2 timeout 1200 bash scripts/ab.sh 2 "python scripts/woodbury_once.py 1000000 20" ltbase ltbulk > gpurun_out/r02c_lt_ab.log 2>&1
cat gpurun_out/r02c_lt_ab.log
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_sharded.py tests/test_gpu_spec_criteria.py tests/test_gpu_love.py -x -q -p no:cacheprovider 2>&1 | tail -2
