# Qwen1.5-MoE-shaped 24-layer decoder serving (shared expert in the grouped launch, hand-written decode
# attention), 60 s paper traces, FCFS vs qllm vs qllm-arrival
mkdir -p gpurun_out
timeout 2400 python tools/serve.py --model qwen --rates 7,14,20 --seeds 0 --duration 60 --schedulers baseline,qllm,qllm-arrival --kv-gib 40 > gpurun_out/serving_qwen_r02.jsonl 2> gpurun_out/serving_qwen_r02.err
tail -n 3 gpurun_out/serving_qwen_r02.err
