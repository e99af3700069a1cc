# bulk router: parity tests, A/B vs the previous kernels, ncu of the new kernel; then the second half
# of the 60 s serving sweep
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k router > gpurun_out/t_router.log 2>&1; echo "exit $?" >> gpurun_out/t_router.log
for cfg in "QMOE_ROUTER_BULK=1" "QMOE_ROUTER_BULK=0" "QMOE_ROUTER_BULK_CFG=1" "QMOE_ROUTER_BULK_CFG=3" "QMOE_ROUTER_BULK=2"; do
  echo "== $cfg" >> gpurun_out/router_ab2.log
  env $cfg timeout 300 python tools/router_ab.py /tmp/r.pt >> gpurun_out/router_ab2.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:router -c 4 -o gpurun_out/router_bulk_r02 -f python tools/ncu_router.py > gpurun_out/ncu_router2.log 2>&1
tail -3 gpurun_out/t_router.log
