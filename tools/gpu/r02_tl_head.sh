for i in 1 2; do timeout 300 python tools/qwen_layer_timeline.py 8192 > gpurun_out/hd_tl_8192_$i.jsonl 2>&1; done
timeout 300 python tools/qwen_layer_timeline.py 32 > gpurun_out/hd_tl_32.jsonl 2>&1
