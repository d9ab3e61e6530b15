#!/bin/bash
# One GPU call: parity tests, bench, ncu launch list and a full ncu capture of the top kernel.
# usage: tools/gpu_round.sh <tag> [tests|notests] [config]
set -x
TAG=${1:-r01}
TESTS=${2:-tests}
CFG=${3:-C3}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${TAG}.txt
if [ "$TESTS" = "tests" ]; then
  timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -5 gpurun_out/pytest_gpu_${TAG}.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -2 gpurun_out/smoke_${TAG}.txt
fi
timeout 600 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err; tail -c 3000 gpurun_out/bench_${TAG}_${CFG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
   python bench.py --config $CFG --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-flush > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_tile<.*1>" -s 3 -c 1 \
   -o gpurun_out/prof_normal_${TAG}_${CFG} -f python tools/quick_time.py $CFG 2 > gpurun_out/ncu_normal_${TAG}.log 2>&1; tail -3 gpurun_out/ncu_normal_${TAG}.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_tile<.*0>" -s 1 -c 1 \
   -o gpurun_out/prof_wz_${TAG}_${CFG} -f python tools/quick_time.py $CFG 2 > gpurun_out/ncu_wz_${TAG}.log 2>&1; tail -3 gpurun_out/ncu_wz_${TAG}.log
ls -la gpurun_out
