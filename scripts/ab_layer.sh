# Dev A/B of library variants on single FMHA launches: VARIANTS="default emu2 ..." bash scripts/ab_layer.sh
for v in ${VARIANTS:-default}; do
  if [ $v = default ]; then L=""; else L="DF_LIB_PATH=build_variants/$v/libdfb200.so"; fi
  echo "== $v pair=${DF_PAIR:-0}"
  env $L timeout 200 python scripts/time_layer.py 2>&1 | head -${LINES_MAX:-9}
done
