# router_tc variants (tools/router_ab.py, L2 flushed): default / deep ring / no selection, per d split
export ROUTER_AB_T=1024,4096,8192,16384
for cfg in "" "QMOE_ROUTER_TC_DEEP=1" "QMOE_ROUTER_TC_NOSEL=1" "QMOE_ROUTER_TC_DEEP=1 QMOE_ROUTER_TC_NOSEL=1"; do
 for S in 0 1 2 4; do
  echo "== cfg=[$cfg] S=$S"
  env $cfg QMOE_ROUTER_TC_MIN=256 QMOE_ROUTER_TC_S=$S timeout 300 python tools/router_ab.py /tmp/x.pt 2>&1 | grep '^{'
 done
done
