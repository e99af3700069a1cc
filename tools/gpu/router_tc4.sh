# after select_tile16 in the mma.sync kernels: router tests, then TC off vs on across T
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k router > gpurun_out/rt4_test.log 2>&1; echo "rc=$?" >> gpurun_out/rt4_test.log
export ROUTER_AB_T=256,1024,2048,3072,4096,6144,8192,16384
QMOE_ROUTER_TC=0 timeout 300 python tools/router_ab.py gpurun_out/r4_old.pt > gpurun_out/r4_old.jsonl 2>&1
QMOE_ROUTER_TC_MIN=256 timeout 300 python tools/router_ab.py gpurun_out/r4_tc.pt > gpurun_out/r4_tc.jsonl 2>&1
QMOE_ROUTER_TC=0 QMOE_ROUTER_CFG=5 ROUTER_AB_T=4096,6144,8192,16384 timeout 300 python tools/router_ab.py gpurun_out/r4_wreg.pt > gpurun_out/r4_wreg.jsonl 2>&1
bash tools/ab_env.sh QMOE_ROUTER_TC 0 1 > gpurun_out/r4_ab_bench.log 2>&1
for v in 0 1 0 1; do echo "TC=$v"; QMOE_ROUTER_TC=$v timeout 300 python tools/qwen_ab.py 2048,4096,8192,16384; done > gpurun_out/r4_qwen_ab.log 2>&1
