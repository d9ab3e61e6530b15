# development: wz-step / CG-pass times over forced tilings: tools/wz_tile_sweep.sh <cfg> "<BL list>" "<groups,warps list>"
CFG=${1:-C3}; BLS=${2:-"8 10 12 14 16 20 24"}; GNWS=${3:-"1,12 2,6 1,8 2,12"}
for bl in $BLS; do for gnw in $GNWS; do
  echo "BL=$bl GNW=$gnw $(LFSR_TILE_BL=$bl LFSR_TILE_GNW=$gnw timeout 120 python tools/quick_time.py $CFG 6 2>&1 | tail -1 | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["it_per_s"],1), [round(x*1000,1) for x in d["kernel_ms_per_launch"]])
except Exception as e: print("fail")')"
done; done
