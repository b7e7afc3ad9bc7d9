# per-level costs with the single-CTA coarse kernel below MGB_COARSE_MAX points (default: off)
for E in "X=0" "MGB_COARSE_MAX=63" "MGB_COARSE_MAX=255" "MGB_COARSE_MAX=1023"; do
  for cfg in c2 c1; do
    echo "== $cfg $E"; env $E timeout 300 python scripts/level_costs.py $cfg 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
  done
done
