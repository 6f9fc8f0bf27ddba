timeout 1200 python scripts/workflow.py C5 --m 256 --skip-variance --skip-cache > gpurun_out/r02c_workflow_C5.jsonl 2>&1; head -c 300 gpurun_out/r02c_workflow_C5.jsonl
timeout 900 python scripts/workflow.py C3 --m 256 --skip-variance > gpurun_out/r02c_workflow_C3.jsonl 2>&1; grep -v mll_result gpurun_out/r02c_workflow_C3.jsonl | head -5
timeout 900 python scripts/workflow.py C2 --m 1000 > gpurun_out/r02c_workflow_C2.jsonl 2>&1; grep seconds gpurun_out/r02c_workflow_C2.jsonl | head -6
