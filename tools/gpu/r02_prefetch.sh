(timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pf_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/pf_test.log)
bash tools/ab_env.sh QMOE_SWAP_PREFETCH_KB 0 553 > gpurun_out/pf_ab.log 2>&1
for v in 0 553; do QMOE_SWAP_PREFETCH_KB=$v timeout 300 python tools/qwen_layer_timeline.py 32 > gpurun_out/pf_tl_$v.jsonl 2>&1; done
