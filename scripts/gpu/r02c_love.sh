timeout 900 python -m pytest tests/test_gpu_love.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 1200 python scripts/love_bench.py C2 256 1024 1024:100 1024:500 2048:500 > gpurun_out/r02c_love_c2.json 2>gpurun_out/r02c_love_c2.err; cat gpurun_out/r02c_love_c2.json; tail -3 gpurun_out/r02c_love_c2.err
