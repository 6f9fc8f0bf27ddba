timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02c_gputest_prod.log 2>&1; tail -2 gpurun_out/r02c_gputest_prod.log
timeout 900 python bench.py > gpurun_out/r02c_bench_prod.log 2>&1; tail -1 gpurun_out/r02c_bench_prod.log | cut -c1-300
