mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k router > gpurun_out/t_drouter.log 2>&1; echo "exit $?" >> gpurun_out/t_drouter.log
for v in 1 0; do echo "== QMOE_ROUTER_DECODE=$v" >> gpurun_out/router_decode_ab.log; QMOE_ROUTER_DECODE=$v ROUTER_AB_T=1,8,32,64 timeout 300 python tools/router_ab.py /tmp/rd_$v.pt >> gpurun_out/router_decode_ab.log 2>&1; done
timeout 600 python tools/record_virtual_run.py gpurun_out/mixtral_b200_run.json.gz > gpurun_out/rec_mixtral2.log 2>&1
timeout 600 python tools/record_virtual_run.py gpurun_out/qwen_b200_run.json.gz qwen > gpurun_out/rec_qwen2.log 2>&1
timeout 900 python bench.py --serve-duration 0 --no-cpu-baseline > gpurun_out/bench_drouter.log 2>&1
for sh in mixtral qwen; do SHAPE=$sh timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:router -c 4 --csv --log-file gpurun_out/router_decode_ncu_$sh.csv python tools/ncu_small.py 32 > /dev/null 2>&1; done
tail -n 2 gpurun_out/t_drouter.log; cat gpurun_out/router_decode_ab.log; tail -n 1 gpurun_out/rec_*2.log
