mkdir -p gpurun_out
timeout 900 python tools/serve_profile.py 7 10 baseline --no-cprofile > gpurun_out/serve_gaps_fcfs.txt 2>&1
grep busy_frac gpurun_out/serve_gaps_fcfs.txt | cut -c1-700
bash tools/gpu/r02_qwen_serving.sh
