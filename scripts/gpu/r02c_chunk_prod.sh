timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02c_gputest_chunk.log 2>&1; tail -2 gpurun_out/r02c_gputest_chunk.log
timeout 900 python bench.py > gpurun_out/r02c_bench_chunk.log 2>&1; tail -1 gpurun_out/r02c_bench_chunk.log | cut -c1-250
