mkdir -p gpurun_out
timeout 900 python tools/serve_profile.py 7 10 baseline > gpurun_out/serve_profile_fcfs.txt 2>&1
timeout 900 python tools/serve_profile.py 7 10 qllm-arrival > gpurun_out/serve_profile_arrival.txt 2>&1
head -c 600 gpurun_out/serve_profile_fcfs.txt
