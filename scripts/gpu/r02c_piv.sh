timeout 900 python -m pytest tests/test_gpu_large_configs.py tests/test_gpu_solve.py -x -q -p no:cacheprovider 2>&1 | tail -2
python scripts/pivchol_once.py 1000000 100 5
GPBBMM_LIB=scripts/variants/lib_pivbase.so python scripts/pivchol_once.py 1000000 100 5
