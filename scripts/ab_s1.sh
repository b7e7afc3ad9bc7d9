# per-level costs: column pairs (default) vs one column per thread (MGB_STREAM1=1) on every streamed level
for rep in 1 2; do
  for E in "X=0" "MGB_STREAM1=1"; do
    echo "== $E"; env $E timeout 300 python scripts/level_costs.py c2 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
    echo "== c4 $E"; env $E timeout 300 python scripts/level_costs.py c4 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  done
done
