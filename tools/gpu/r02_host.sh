mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_decoder_gpu.py tests/test_engine_gpu.py tests/test_arrival_flag_gpu.py tests/test_attention_gpu.py tests/test_ep_serving_gpu.py tests/test_emit_gpu.py -q -x > gpurun_out/t_host.log 2>&1; echo "exit $?" >> gpurun_out/t_host.log
timeout 900 python tools/serve_profile.py 7 10 baseline --no-cprofile > gpurun_out/serve_gaps_fcfs2.txt 2>&1
tail -n 3 gpurun_out/t_host.log; grep busy_frac gpurun_out/serve_gaps_fcfs2.txt | cut -c1-600
timeout 900 python tools/serve.py --model qwen --rates 14 --seeds 0 --duration 30 --schedulers baseline,qllm-arrival --kv-gib 40 > gpurun_out/serving_qwen_elide.jsonl 2>&1
