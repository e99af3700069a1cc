# swap-AB pair wide last tile: parity + same-box A/B of the FFN alone, then the bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_paths_gpu.py -q -x > gpurun_out/t_paths.log 2>&1; echo "exit $?" >> gpurun_out/t_paths.log
for m in 128 0 256 64; do
  echo "== QMOE_SP_MERGE=$m" >> gpurun_out/ffn_ab_wide.log
  QMOE_SP_MERGE=$m timeout 300 python tools/ffn_ab.py 768 1024 1100 1280 1536 2048 3072 4096 8192 16384 >> gpurun_out/ffn_ab_wide.log 2>&1
done
timeout 900 python bench.py --serve-duration 0 > gpurun_out/bench_wide.log 2>&1
tail -3 gpurun_out/t_paths.log
timeout 900 python tools/fit_cost_model.py gpurun_out/cost_model_b200_r02.json mixtral > gpurun_out/fit_mixtral.log 2>&1
timeout 900 python tools/fit_cost_model.py gpurun_out/cost_model_b200_r02_qwen.json qwen > gpurun_out/fit_qwen.log 2>&1
