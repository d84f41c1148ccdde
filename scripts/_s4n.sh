timeout 300 python scripts/vb_sweep.py "wide_tiles=2" "wide_tiles=3" "wide_tiles=6" "wide_tiles=2" "wide_tiles=3" "wide_tiles=6" "wide_tiles=7" 2>&1 | grep -v Warn | cut -c1-260
