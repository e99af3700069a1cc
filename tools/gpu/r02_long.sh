# round 2: router parity after the 4-CTA build, layer sweep (incl. CUDA-graph preempt cost), per-stage
# cost-model fits, then the second half of the 60 s serving sweep
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k router > gpurun_out/t_router2.log 2>&1; echo "exit $?" >> gpurun_out/t_router2.log
timeout 1200 python tools/layer_sweep.py > gpurun_out/layer_sweep_r02b.jsonl 2> gpurun_out/layer_sweep_r02b.err
timeout 900 python tools/fit_cost_model.py gpurun_out/cost_model_b200_r02.json mixtral > gpurun_out/fit_mixtral.log 2>&1
timeout 900 python tools/fit_cost_model.py gpurun_out/cost_model_b200_r02_qwen.json qwen > gpurun_out/fit_qwen.log 2>&1
timeout 2700 python tools/serve.py --rates 2,4,6,8,10 --seeds 0,1 --duration 60 --schedulers baseline,qllm,qllm-arrival --kv-gib 40 > gpurun_out/serving_r02_sweep_b.jsonl 2> gpurun_out/serving_r02_sweep_b.err
tail -2 gpurun_out/t_router2.log; tail -2 gpurun_out/layer_sweep_r02b.err; tail -2 gpurun_out/fit_*.log
