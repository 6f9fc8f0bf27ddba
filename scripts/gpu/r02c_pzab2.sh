TAIL=2 timeout 1200 bash scripts/ab.sh 2 "python scripts/woodbury_once.py 1000000 20" pzu1 pzks2 pzks3 pzks4 > gpurun_out/r02c_pz_ab2.log 2>&1
cat gpurun_out/r02c_pz_ab2.log
GPBBMM_LIB=scripts/variants/lib_pzks3.so timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider 2>&1 | tail -2
