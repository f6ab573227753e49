# Dev A/B of library variants on the bench step: bash scripts/ab_bench.sh (names under build_variants/)
# VARIANTS="default fence0 ..." picks the libraries (default = the shipped build)
for v in ${VARIANTS:-default emu0 emu2 default emu0 emu2}; do
  if [ $v = default ]; then L=""; else L="DF_LIB_PATH=build_variants/$v/libdfb200.so"; fi
  env $L python bench.py --no-configs 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), round(d['roofline']['achieved']), d['clocks']['sm_mhz'], round(d['layer_fused']['fps'],2))"
done
