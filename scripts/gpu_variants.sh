# A/B of library variants on config 2 fwd+bwd (quick_timing): product lib first, then each variant
for v in "" $VARIANTS; do
  echo "== variant: ${v:-product}"
  if [ -n "$v" ]; then DRK_LIB_PATH=$v timeout 300 python scripts/quick_timing.py $CFGS 2>&1 | cut -c1-300; else timeout 300 python scripts/quick_timing.py $CFGS 2>&1 | cut -c1-300; fi
done
