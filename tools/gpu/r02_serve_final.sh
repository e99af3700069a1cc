# serving with the final kernels: Qwen-shaped decoder at 14 / 20 req/s, Mixtral at 7 req/s (60 s paper traces, seed 0)
timeout 1200 python tools/serve.py --model qwen --rates 14,20 --seeds 0 --duration 60 --schedulers baseline,qllm,qllm-arrival --kv-gib 40 > gpurun_out/serve_final_qwen.jsonl 2> gpurun_out/serve_final_qwen.err
timeout 900 python tools/serve.py --model mixtral --rates 7 --seeds 1 --duration 60 --schedulers baseline,qllm,qllm-arrival --kv-gib 40 > gpurun_out/serve_final_mixtral.jsonl 2> gpurun_out/serve_final_mixtral.err
