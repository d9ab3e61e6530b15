#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck, initcheck) over a small solve
# (C1 and M1, 2 ADMM iterations, edge + interior tiles, all kernels incl. setup and tuning),
# then over the §8f modes (gd / gd-ls, per-view maps, user blur kernel, paper-mode adjoint,
# colour: tools/modes_smoke.py).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in C1 M1; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/quick_time.py $cfg 1 > gpurun_out/sanitize_${tool}_${cfg}.log 2>&1
    echo "$tool $cfg rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_${cfg}.log | tail -1)"
  done
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python tools/modes_smoke.py > gpurun_out/sanitize_${tool}_modes.log 2>&1
  echo "$tool modes rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_modes.log | tail -1)"
done
