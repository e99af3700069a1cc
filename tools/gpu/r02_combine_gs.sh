(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gs_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/gs_test.log)
for T in 8192 32; do timeout 300 python tools/qwen_layer_timeline.py $T > gpurun_out/gs_tl_$T.jsonl 2>&1; done
timeout 600 python bench.py --no-cpu-baseline --serve-duration 0 > gpurun_out/gs_bench.log 2>&1
