timeout 1200 bash scripts/ab.sh 2 "python scripts/woodbury_once.py 1000000 20" pzu1 pzu2 pzu4 > gpurun_out/r02c_pz_ab.log 2>&1
cat gpurun_out/r02c_pz_ab.log
