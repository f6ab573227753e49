# Dev A/B of the 1-CTA vs CTA-pair FMHA on the bench step (shipped library; DF_CTA_PAIR picks the kernel)
for pr in ${PAIRS:-0 1 0 1}; do
  DF_CTA_PAIR=$pr python bench.py --no-configs --no-cpu 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pair=$pr', 'fps', round(d['value'],2), 'attn_us', round(d['attn_us_per_layer'],1), 'frac', round(d['roofline']['frac'],3), 'mhz', d['clocks']['sm_mhz'], 'fused_fps', round(d['layer_fused']['fps'],2), 'base_us', round(d['baseline_all_context']['us_per_layer'],1))"
done
