# full validation: pytest -m gpu, smoke, default bench; decode-iteration breakdown for both decoders
mkdir -p gpurun_out
(timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputest_final.log)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_final.log 2>&1
timeout 600 python tools/decode_profile.py > gpurun_out/decode_profile_mixtral.json 2> gpurun_out/decode_profile.err
timeout 600 python tools/decode_profile.py qwen > gpurun_out/decode_profile_qwen.json 2>> gpurun_out/decode_profile.err
tail -n 4 gpurun_out/gputest_final.log; tail -n 2 gpurun_out/smoke_final.log
