(timeout 1200 python -m pytest tests/test_engine_gpu.py tests/test_decoder_gpu.py tests/test_kernels_gpu.py tests/test_hf_block_gpu.py -m gpu -x -q -k "b200_virtual or combine or qwen or Qwen or decoder" > gpurun_out/c8_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/c8_test.log)
timeout 300 python tools/qwen_layer_timeline.py 8192 > gpurun_out/qwen_timeline_c8.jsonl 2>&1
timeout 300 python tools/qwen_ab.py 1024,4096,8192,16384 > gpurun_out/qwen_ab_c8.jsonl 2>&1
