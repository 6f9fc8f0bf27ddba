timeout 900 python bench.py > gpurun_out/r02c_bench_final.log 2>&1; tail -1 gpurun_out/r02c_bench_final.log | cut -c1-150
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02c_bench_ref.log 2>&1; tail -1 gpurun_out/r02c_bench_ref.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c_launches_raw.csv python bench.py --steps 2 --warmup 1 --no-e2e > gpurun_out/r02c_ncu_launch.log 2>&1; tail -1 gpurun_out/r02c_ncu_launch.log | cut -c1-100
