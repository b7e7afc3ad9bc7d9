# column-pair ring prefetch distance: 5 rows (default) vs 3, 4, 6 (experiments/lib_d*.so)
for rep in 1 2; do
  for L in paper_2102_12071_b200/libmgb.so experiments/lib_d3.so experiments/lib_d4.so experiments/lib_d6.so; do
    echo "== $L"; MGB_LIB_PATH=$PWD/$L timeout 300 python scripts/level_costs.py c2 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  done
done
