# A/B of the fast forward's tile order (DRK_TILE_ORDER 0 row-major, 1 longest-first within copy-out bands, 2 global)
for m in 0 1 2 1 0; do
  echo "== order $m"; DRK_TILE_ORDER=$m timeout 300 python scripts/quick_timing.py 1 2 3 2>&1 | grep -o "cfg[0-9] fwd [^{]*{[^}]*}" | sed "s/.backward_raster.*//" | cut -c1-200
done
