GPBBMM_LIB=scripts/variants/lib_nb.so timeout 600 python -m pytest tests/test_gpu_kv.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > gpurun_out/r02c_nb_tests.log 2>&1; tail -2 gpurun_out/r02c_nb_tests.log
timeout 900 bash scripts/ab.sh 3 "python scripts/kv_once.py 3 262144 11 matern32 20" cur nb > gpurun_out/r02c_ab_nb.log 2>&1
timeout 600 bash scripts/ab.sh 2 "python scripts/kv_once.py 3 1000000 11 matern32 3" cur nb >> gpurun_out/r02c_ab_nb.log 2>&1
cat gpurun_out/r02c_ab_nb.log
