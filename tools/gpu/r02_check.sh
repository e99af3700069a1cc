mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_decoder_gpu.py tests/test_ep_serving_gpu.py "tests/test_paths_gpu.py::test_preempt_flag_raised_mid_launch" -q > gpurun_out/t3.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3.log)
timeout 600 python tools/record_virtual_run.py gpurun_out/mixtral_b200_run.json.gz > gpurun_out/rec_mixtral.log 2>&1
timeout 600 python tools/record_virtual_run.py gpurun_out/qwen_b200_run.json.gz qwen > gpurun_out/rec_qwen.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 2 --warmup 3 --serve-duration 0 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router -c 4 -o gpurun_out/router_r02 -f python tools/ncu_router.py > gpurun_out/ncu_router.log 2>&1
tail -5 gpurun_out/t3.log; cat gpurun_out/rec_*.log | tail -4
