timeout 600 python -m pytest tests/test_gpu_solve.py -x -q -p no:cacheprovider -k lt_mul 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02c_gputest_last.log 2>&1; tail -2 gpurun_out/r02c_gputest_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
