#!/bin/bash
# C3 NORMAL/wz kernel time for forced tilings: tools/tile_sweep.sh <cfg> "BL:g,w[:nwn] ..."
CFG=${1:-C3}
for spec in $2; do
  IFS=: read bl gw nwn <<< "$spec"
  out=$(LFSR_TILE_BL=$bl LFSR_TILE_GNW=$gw LFSR_TILE_NWN=${nwn:-} timeout 300 python tools/quick_time.py $CFG 10 2>&1 | tail -1)
  echo "$CFG $spec $(echo "$out" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["it_per_s"],1), [round(x*1000,1) for x in d["kernel_ms_per_launch"]])
except Exception as e: print("fail", e)')"
done
