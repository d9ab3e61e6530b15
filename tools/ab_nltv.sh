#!/bin/bash
# wz-step with the NLTV rows split into k_wz_nltv (LFSR_NLTV_SPLIT=1) or in the tile kernel (=0), and
# library variants: tools/ab_nltv.sh "M2 C3" "variant ..."
for c in ${1:-C3 C2 C4 C5 M2 M3}; do
  for v in split0 main $2; do
    unset LFSR_LIB; export LFSR_NLTV_SPLIT=1
    [ "$v" = split0 ] && export LFSR_NLTV_SPLIT=0
    [ "$v" != split0 ] && [ "$v" != main ] && export LFSR_LIB=paper_2206_05047_b200/liblfsr_$v.so
    echo "$c $v $(timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1 | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["it_per_s"],1), [round(x*1000,1) for x in d["kernel_ms_per_launch"]])
except Exception as e: print("fail", e)')"
  done
done
