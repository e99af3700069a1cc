mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_paths_gpu.py tests/test_hf_block_gpu.py tests/test_engine_gpu.py tests/test_decoder_gpu.py -q -x > gpurun_out/t_direct2.log 2>&1; echo "exit $?" >> gpurun_out/t_direct2.log
for v in 1 0 1 0; do echo "== QMOE_SHARED_DIRECT=$v" >> gpurun_out/qwen_direct_ab2.log; QMOE_SHARED_DIRECT=$v timeout 300 python tools/qwen_ab.py 2048,4096,8192,16384 >> gpurun_out/qwen_direct_ab2.log 2>&1; done
tail -n 3 gpurun_out/t_direct2.log; cat gpurun_out/qwen_direct_ab2.log | cut -c1-250
