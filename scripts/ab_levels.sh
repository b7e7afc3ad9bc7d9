# A/B of per-level cycle costs (c2) in one session: default lib, experiment libs, env variants, tile off
for rep in 1 2; do
  for L in paper_2102_12071_b200/libmgb.so $EXTRA_LIBS; do
    echo "== $L"; MGB_LIB_PATH=$PWD/$L timeout 300 python scripts/level_costs.py c2 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  done
  for E in $EXTRA_ENVS; do
    echo "== $E"; env $E timeout 300 python scripts/level_costs.py c2 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  done
done
