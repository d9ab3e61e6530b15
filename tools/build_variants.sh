#!/bin/bash
# build library variants for A/B timing: tools/build_variants.sh "name:-DX=1,-DY=2 name2:..."
cd "$(dirname "$0")/.."
for spec in $1; do
  name=${spec%%:*}; defs=${spec#*:}; defs=${defs//,/ }
  [ "$defs" = "$name" ] && defs=""
  LFSR_LIB_NAME=liblfsr_$name.so LFSR_VARIANT_DEFS="$defs" python -c "from paper_2206_05047_b200 import build; build.build()" > /dev/null 2>&1 &
done
wait
ls paper_2206_05047_b200/liblfsr_*.so
