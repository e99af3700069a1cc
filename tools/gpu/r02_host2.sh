mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_decoder_gpu.py tests/test_engine_gpu.py tests/test_arrival_flag_gpu.py tests/test_ep_serving_gpu.py tests/test_emit_gpu.py tests/test_integration_gpu.py -q -x > gpurun_out/t_host2.log 2>&1; echo "exit $?" >> gpurun_out/t_host2.log
timeout 900 python tools/serve_profile.py 14 10 qllm-arrival --qwen --no-cprofile > gpurun_out/serve_prof_qwen2.txt 2>&1
timeout 900 python tools/serve_profile.py 7 10 baseline --no-cprofile > gpurun_out/serve_gaps_fcfs3.txt 2>&1
tail -n 3 gpurun_out/t_host2.log; grep busy_frac gpurun_out/serve_prof_qwen2.txt gpurun_out/serve_gaps_fcfs3.txt | cut -c1-420
