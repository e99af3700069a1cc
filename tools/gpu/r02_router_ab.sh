# router A/B on one box (tools/router_ab.py under several QMOE_ROUTER_* settings), then the first half
# of the 60 s serving sweep (tools/serve.py, clocks sampled)
mkdir -p gpurun_out
for cfg in "QMOE_ROUTER_CFG=0" "QMOE_ROUTER_CFG=3" "QMOE_ROUTER_CFG=4" "QMOE_ROUTER_MT=4" "QMOE_ROUTER_CFG=1" "QMOE_ROUTER_CFG=2" "QMOE_ROUTER_STREAM=0"; do
  echo "== $cfg" >> gpurun_out/router_ab.log
  env $cfg timeout 300 python tools/router_ab.py /tmp/r.pt >> gpurun_out/router_ab.log 2>&1
done
timeout 2700 python tools/serve.py --rates 1,3,5,7 --seeds 0,1 --duration 60 --schedulers baseline,qllm,qllm-arrival --kv-gib 40 > gpurun_out/serving_r02_sweep_a.jsonl 2> gpurun_out/serving_r02_sweep_a.err
tail -3 gpurun_out/serving_r02_sweep_a.err
