# prefill wide kernel: attention tests, A/B of the CTA shapes, then the layer sweep with the final router
(timeout 900 python -m pytest tests/test_attention_gpu.py -m gpu -x -q > gpurun_out/p3_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/p3_test.log)
for w in 2 4 8; do QMOE_PREFILL_W=$w timeout 300 python tools/prefill_attn_ab.py > gpurun_out/p3_ab_w$w.jsonl 2>&1; done
timeout 1500 python tools/layer_sweep.py > gpurun_out/layer_sweep_r02c.jsonl 2> gpurun_out/layer_sweep_r02c.err
