# Same-box A/B of the bench's layer numbers under two settings of one QMOE_* variable, alternated:
#   bash tools/ab_env.sh QMOE_PDL 0 1
var=$1; a=$2; b=$3
for i in 1 2; do
  for v in $a $b; do
    env $var=$v python bench.py --no-cpu-baseline --serve-duration 0 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$var=$v', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'ffn', round(d['roofline']['achieved'],1), 'sm', d['clocks']['sm_mhz'], 'qwen_pre', round(d['qwen']['prefill']['ms'],3), 'qwen_dec', round(d['qwen']['decode']['ms'],3), 'mix_dec', round(d['decode_step']['ms'],3))"
  done
done
