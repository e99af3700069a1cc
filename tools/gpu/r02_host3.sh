mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_decoder_gpu.py tests/test_engine_gpu.py tests/test_arrival_flag_gpu.py tests/test_ep_serving_gpu.py tests/test_emit_gpu.py tests/test_integration_gpu.py -q -x > gpurun_out/t_host3.log 2>&1; echo "exit $?" >> gpurun_out/t_host3.log
tail -n 3 gpurun_out/t_host3.log
