GPBBMM_LIB=scripts/variants/lib_run2.so timeout 600 python -m pytest tests/test_gpu_kv.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 bash scripts/ab.sh 2 "python scripts/kv_once.py 3 262144 11 matern32 20" cur run1 run2 > gpurun_out/r02c_ab_run.log 2>&1
timeout 900 bash scripts/ab.sh 2 "python scripts/kv_once.py 3 1000000 11 matern32 3" cur run1 run2 >> gpurun_out/r02c_ab_run.log 2>&1
cat gpurun_out/r02c_ab_run.log
