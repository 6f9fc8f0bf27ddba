timeout 2000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02c_gputest_full.log 2>&1; tail -5 gpurun_out/r02c_gputest_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; tail -2 gpurun_out/r02c_smoke.log
