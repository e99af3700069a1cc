timeout 600 python tools/ls_fraction_sweep.py > gpurun_out/ls_fraction_r02.jsonl 2>&1; cat gpurun_out/ls_fraction_r02.jsonl
