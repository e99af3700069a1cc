(timeout 900 python -m pytest tests/test_attention_gpu.py tests/test_decoder_gpu.py -m gpu -x -q > gpurun_out/p_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/p_test.log)
timeout 300 python tools/prefill_attn_ab.py > gpurun_out/p_ab.jsonl 2>&1
timeout 900 python tools/record_virtual_run.py gpurun_out/mixtral_b200_run.json.gz > gpurun_out/rec_mixtral.log 2>&1
timeout 900 python tools/record_virtual_run.py gpurun_out/qwen_b200_run.json.gz qwen > gpurun_out/rec_qwen.log 2>&1
