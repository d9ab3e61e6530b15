#!/bin/bash
# time several library variants on configs: tools/variants.sh "A B C" "C3 C4"
for v in $1; do
  for c in $2; do
    echo -n "$v $c "; LFSR_LIB=$PWD/paper_2206_05047_b200/liblfsr_$v.so timeout 300 python tools/quick_time.py $c 10 2>&1 | tail -1
  done
done
