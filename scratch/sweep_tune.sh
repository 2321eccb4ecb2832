for cfg in "16384 16" "16384 12" "16384 8" "32768 6" "8192 16"; do
  set -- $cfg
  echo "== tile=$1 stages=$2 $(RAPDB_TILE_BYTES=$1 RAPDB_STAGES=$2 timeout 60 python tools/profile_sweep.py C1 20 2>&1 | tail -1)"
done
echo "== chunked 8192x16 $(RAPDB_TILE_BYTES=8192 RAPDB_STAGES=16 RAPDB_ROW_TILE_MAX=0 timeout 60 python tools/profile_sweep.py C1 20 2>&1 | tail -1)"
echo "== C0 default $(timeout 100 python tools/profile_sweep.py C0 50 2>&1 | tail -1)"
echo "== C2 default $(timeout 300 python tools/profile_sweep.py C2 5 2>&1 | tail -1)"
