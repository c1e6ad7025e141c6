for env in "X=1" "RSR_TC_CHUNK_TILES=1120" "RSR_TC_CHUNK_TILES=2240" "RSR_TC_ABUFS=3"; do
  echo "== $env"; env $env timeout 300 tools/compact_tile_sweep.sh "500000" "def" | grep -v off
done
