# per-level costs (c2) under forced row-segment lengths of the streaming passes (MGB_SEG, all streamed levels)
for E in "X=0" "MGB_SEG=16" "MGB_SEG=24" "MGB_SEG=32" "MGB_SEG=48" "MGB_SEG=64" "MGB_SEG=96" "MGB_SEG=128" "MGB_SEG=256"; do
  echo "== $E"; env $E timeout 300 python scripts/level_costs.py c2 2>&1 | awk '{printf "L%s=%s ", $2, $9}'; echo
done
