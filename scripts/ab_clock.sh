# Dev A/B under sustained load (power cap): VARIANTS="default prev ..." bash scripts/ab_clock.sh
for v in ${VARIANTS:-default prev default prev}; do
  if [ $v = default ]; then L=""; else L="DF_LIB_PATH=build_variants/$v/libdfb200.so"; fi
  echo "== $v"
  env $L DF_PAIR=1 timeout 100 python scripts/clock_probe.py
done
