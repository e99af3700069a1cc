(timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k router > gpurun_out/rs_test.log 2>&1; echo "pytest exit $?" >> gpurun_out/rs_test.log)
ROUTER_AB_T=1024,2048,3072,4096,8192,16384 timeout 300 python tools/router_ab.py /tmp/r.pt > gpurun_out/rs_ab.jsonl 2>&1
