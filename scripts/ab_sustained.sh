# Dev A/B of library variants under sustained back-to-back FMHA launches (power-capped regime, CTA pair):
# VARIANTS="base default" bash scripts/ab_sustained.sh
for v in ${VARIANTS:-base default base default}; do
  if [ $v = default ]; then L=""; else L="DF_LIB_PATH=build_variants/$v/libdfb200.so"; fi
  echo "== $v"; env $L DF_PAIR=1 python scripts/clock_probe.py 2>&1 | tail -2
done
