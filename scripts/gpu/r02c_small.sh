timeout 600 python scripts/small_n.py C1 > gpurun_out/r02c_small_C1.log 2>&1; cat gpurun_out/r02c_small_C1.log
timeout 600 python scripts/prof_small.py C1 > gpurun_out/r02c_prof_C1.log 2>&1; tail -80 gpurun_out/r02c_prof_C1.log
