for E in "X=0" "MGB_COARSE_MAX=63" "MGB_COARSE_MAX=255" "MGB_COARSE_MAX=1023" "MGB_COARSE_MAX=4095"; do
  echo "== $E"; env $E timeout 300 python scripts/level_costs.py c2 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  echo "== c1 $E"; env $E timeout 300 python scripts/level_costs.py c1 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
done
