(timeout 1200 python -m pytest tests/test_attention_gpu.py tests/test_engine_gpu.py -m gpu -x -q -k "prefill or b200_virtual" > gpurun_out/t_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/t_test.log)
timeout 300 python tools/qwen_layer_timeline.py 8192 > gpurun_out/qwen_timeline.jsonl 2>&1
timeout 300 python tools/qwen_layer_timeline.py 32 > gpurun_out/qwen_timeline_32.jsonl 2>&1
