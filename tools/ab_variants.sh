#!/bin/bash
# A/B of library variants (tools/build_variants.sh): tools/ab_variants.sh "C3 C2" "novm noquad"
for c in $1; do
  for v in main $2; do
    if [ "$v" != main ]; then export LFSR_LIB=paper_2206_05047_b200/liblfsr_$v.so; else unset LFSR_LIB; fi
    echo "$c $v $(timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1 | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["it_per_s"],1), [round(x*1000,1) for x in d["kernel_ms_per_launch"]])
except Exception as e: print("fail", e)')"
  done
done
