# the 60 s serving sweep again after the host-path changes (report elision, PDL helpers, KV append in place)
mkdir -p gpurun_out
timeout 3000 python tools/serve.py --rates 1,4,7,8,10 --seeds 0 --duration 60 --schedulers baseline,qllm,qllm-arrival --kv-gib 40 > gpurun_out/serving_r02_sweep_c.jsonl 2> gpurun_out/serving_r02_sweep_c.err
tail -n 2 gpurun_out/serving_r02_sweep_c.err
