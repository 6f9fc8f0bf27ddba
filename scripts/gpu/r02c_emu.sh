GPBBMM_LIB=scripts/variants/lib_emu4.so timeout 600 python -m pytest tests/test_gpu_kv.py tests/test_gpu_large_configs.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 900 bash scripts/ab.sh 3 "python scripts/kv_once.py 3 262144 11 matern32 20" early emu4 emu8 emu16 > gpurun_out/r02c_ab_emu.log 2>&1
timeout 900 bash scripts/ab.sh 2 "python scripts/kv_once.py 3 262144 11 rbf 20" early emu4 emu8 emu16 >> gpurun_out/r02c_ab_emu.log 2>&1
cat gpurun_out/r02c_ab_emu.log
