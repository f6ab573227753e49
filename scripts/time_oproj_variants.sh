# Dev: cold/hot out-projection timings of library variants (VARIANTS names under build_variants/; default = shipped)
for v in ${VARIANTS:-default}; do
  for bn in ${BNS:-192 256}; do
    if [ $v = default ]; then L=""; else L="DF_LIB_PATH=build_variants/$v/libdfb200.so"; fi
    echo "== $v BN=$bn"; env $L DF_PROJ_BN=$bn python scripts/time_proj.py 2>&1 | grep -E "^BN=$bn|cold out-proj BN=$bn"
  done
done
