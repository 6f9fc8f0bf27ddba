GPBBMM_LIB=scripts/variants/lib_ql.so timeout 900 python -m pytest tests/test_gpu_kv.py tests/test_gpu_sharded.py tests/test_gpu_multidev.py tests/test_gpu_bounds.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 bash scripts/ab.sh 2 "python scripts/kv_once.py 3 262144 11 matern32 20" cur ql > gpurun_out/r02c_ab_ql.log 2>&1
timeout 900 bash scripts/ab.sh 2 "python scripts/kv_once.py 3 1000000 11 matern32 3" cur ql >> gpurun_out/r02c_ab_ql.log 2>&1
cat gpurun_out/r02c_ab_ql.log
