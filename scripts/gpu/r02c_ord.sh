GPBBMM_LIB=scripts/variants/lib_ord1.so timeout 600 python -m pytest tests/test_gpu_kv.py -x -q -p no:cacheprovider 2>&1 | tail -1
GPBBMM_LIB=scripts/variants/lib_ord2.so timeout 600 python -m pytest tests/test_gpu_kv.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 bash scripts/ab.sh 3 "python scripts/kv_once.py 3 262144 11 matern32 20" early ord1 ord2 > gpurun_out/r02c_ab_ord.log 2>&1
timeout 900 bash scripts/ab.sh 2 "python scripts/kv_once.py 3 1000000 11 matern32 3" early ord1 ord2 >> gpurun_out/r02c_ab_ord.log 2>&1
cat gpurun_out/r02c_ab_ord.log
