# Same-box A/B of the bench's layer numbers: default paths vs QMOE_SWAP_PAIR=0, alternated.
for i in 1 2; do
  for env in "QMOE_SWAP_PAIR=0" "QMOE_SWAP_PAIR=-1"; do
    env $env python bench.py --no-cpu-baseline --serve-duration 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$env', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['achieved'],1), d['clocks']['sm_mhz'], round(d['qwen']['prefill']['ms'],3), round(d['qwen']['decode']['ms'],3), round(d['decode_step']['ms'],3))"
  done
done
