for v in pf1024 pf256 pf512 pf1024 pf256 pf512; do echo -n "$v: "; GPBBMM_LIB=scripts/variants/lib_$v.so python scripts/small_n.py C1 4096 20 2>&1 | head -3 | tr '\n' ' '; echo; done
GPBBMM_LIB=scripts/variants/lib_pf256.so timeout 600 python -m pytest tests/test_gpu_solve.py -x -q -p no:cacheprovider 2>&1 | tail -1
