mkdir -p gpurun_out
timeout 3300 python tools/serve.py --model qwen --rates 7,14,20,28 --seeds 0,1 --duration 60 --schedulers baseline,qllm,qllm-arrival --kv-gib 40 > gpurun_out/serving_qwen_r02_sweep.jsonl 2> gpurun_out/serving_qwen_r02_sweep.err
tail -n 2 gpurun_out/serving_qwen_r02_sweep.err
