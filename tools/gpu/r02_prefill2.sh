(timeout 900 python -m pytest tests/test_attention_gpu.py -m gpu -x -q > gpurun_out/p2_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/p2_test.log)
for w in 4 8; do QMOE_PREFILL_W=$w timeout 300 python tools/prefill_attn_ab.py > gpurun_out/p2_ab_w$w.jsonl 2>&1; done
