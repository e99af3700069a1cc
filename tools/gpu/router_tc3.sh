timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k router > gpurun_out/rt3_test.log 2>&1; echo "rc=$?" >> gpurun_out/rt3_test.log
export ROUTER_AB_T=1024,2048,4096,8192,16384
QMOE_ROUTER_TC=0 timeout 300 python tools/router_ab.py gpurun_out/r3_old.pt > gpurun_out/r3_old.jsonl 2>&1
for S in 0 1 2 4; do QMOE_ROUTER_TC_MIN=256 QMOE_ROUTER_TC_S=$S timeout 300 python tools/router_ab.py gpurun_out/r3_tc$S.pt > gpurun_out/r3_tc$S.jsonl 2>&1; done
python tools/router_tc_cmp.py gpurun_out/r3_old.pt gpurun_out/r3_tc0.pt > gpurun_out/r3_cmp.txt 2>&1
