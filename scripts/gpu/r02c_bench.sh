timeout 900 python bench.py > gpurun_out/r02c_bench2.log 2>&1; tail -1 gpurun_out/r02c_bench2.log
