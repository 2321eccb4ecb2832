for cfg in "16384 16 49152" "8192 24 0" "8192 16 0" "12288 16 0" "16384 12 49152" "4096 32 0"; do
  set -- $cfg
  echo "tile=$1 stages=$2 rowmax=$3"
  RAPDB_TILE_BYTES=$1 RAPDB_STAGES=$2 RAPDB_ROW_TILE_MAX=$3 python tools/profile_sweep.py C1 30
done
