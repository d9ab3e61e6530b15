#!/bin/bash
# ncu --set full of one tile-kernel launch (mode regex) on a config: tools/ncu_one.sh <tag> <cfg> <mode 0|1> <skip>
TAG=$1; CFG=${2:-C3}; MODE=${3:-1}; SKIP=${4:-3}
mkdir -p gpurun_out
export $(python tools/tuned_env.py $CFG 2>/dev/null | tail -1)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\(int\)${MODE}, \(bool\)" -s $SKIP -c 1 \
   -o gpurun_out/prof_${TAG}_${CFG}_m${MODE} -f python tools/quick_time.py $CFG 2 > gpurun_out/ncu_${TAG}_${CFG}_m${MODE}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}_${CFG}_m${MODE}.log
