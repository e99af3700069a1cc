# ncu --set full of the swap-AB pair FFN at 8192 tokens (source-level stalls)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ffn_swap_pair -s 1 -c 1 -o gpurun_out/ffn_sp8192_r02 -f python tools/ncu_ffn.py 8192 > gpurun_out/ncu_ffn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ffn_swap_pair -s 1 -c 1 -o gpurun_out/ffn_sp1024_r02 -f python tools/ncu_ffn.py 1024 >> gpurun_out/ncu_ffn.log 2>&1
tail -3 gpurun_out/ncu_ffn.log
