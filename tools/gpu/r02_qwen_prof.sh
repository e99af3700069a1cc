mkdir -p gpurun_out
timeout 900 python tools/serve_profile.py 14 10 qllm-arrival --qwen > gpurun_out/serve_prof_qwen.txt 2>&1
grep busy_frac gpurun_out/serve_prof_qwen.txt | cut -c1-500
