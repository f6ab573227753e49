# Dev A/B of an environment switch under sustained load and isolated: ENVS="DF_PAIR_WG=3 DF_PAIR_WG=2" bash scripts/ab_env.sh
for e in ${ENVS}; do
  echo "== $e"
  env $e DF_PAIR=1 timeout 100 python scripts/clock_probe.py
done
for e in ${ENVS}; do
  echo "== $e isolated"
  env $e DF_PAIR=1 timeout 200 python scripts/time_layer.py 2>&1 | head -${LINES_MAX:-9}
done
