mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k router > gpurun_out/t_wreg.log 2>&1; echo "exit $?" >> gpurun_out/t_wreg.log
for cfg in "QMOE_ROUTER_CFG=0" "QMOE_ROUTER_CFG=-1" "QMOE_ROUTER_CFG=5"; do
  echo "== $cfg" >> gpurun_out/router_ab3.log
  env $cfg timeout 300 python tools/router_ab.py /tmp/r_$cfg.pt >> gpurun_out/router_ab3.log 2>&1
done
python - <<'PY' >> gpurun_out/router_ab3.log
import torch
a = torch.load("/tmp/r_QMOE_ROUTER_CFG=0.pt"); b = torch.load("/tmp/r_QMOE_ROUTER_CFG=-1.pt")
for k in a:
    print(k, "ids equal", torch.equal(a[k][0], b[k][0]), "weights equal", torch.equal(a[k][1], b[k][1]))
PY
timeout 600 ncu --set full --clock-control none -k regex:router -c 2 -o gpurun_out/router_wreg_r02 -f python tools/ncu_router.py > /dev/null 2>&1
tail -n 2 gpurun_out/t_wreg.log; grep -A6 "CFG=0" gpurun_out/router_ab3.log | head -8; tail -n 12 gpurun_out/router_ab3.log
