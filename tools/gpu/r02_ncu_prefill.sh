timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_attn -c 4 -o gpurun_out/ncu_prefill_r02 -f python tools/ncu_prefill.py > gpurun_out/ncu_prefill.log 2>&1
