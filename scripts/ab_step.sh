# Dev A/B of library variants on the 30-layer bench step (no configs, no CPU leg):
# VARIANTS="base default base default" bash scripts/ab_step.sh   (names under build_variants/; default = shipped build)
for v in ${VARIANTS:-base default base default}; do
  if [ $v = default ]; then L=""; else L="DF_LIB_PATH=build_variants/$v/libdfb200.so"; fi
  env $L python bench.py --no-configs --no-cpu ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); lf=d['layer_fused']
print('$v', 'fps', round(d['value'],2), 'attn_us', round(d['attn_us_per_layer'],1), 'frac', round(d['roofline']['frac'],3), 'mhz', d['clocks']['sm_mhz'], 'base_us', round(d['baseline_all_context']['us_per_layer'],1), 'fused_fps', round(lf['fps'],2), 'split', {k: round(x,1) for k,x in lf['split_us_per_layer'].items()}, flush=True)"
done
