#!/bin/bash
# One GPU call: parity tests, smoke, bench (N=1), ncu launch list and full captures of the
# tile kernels.  usage: tools/gpu_round.sh <tag> [tests|notests] [config]
TAG=${1:-r01}
TESTS=${2:-tests}
CFG=${3:-C3}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${TAG}.txt
if [ "$TESTS" = "tests" ]; then
  timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
fi
timeout 900 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err; tail -c 400 gpurun_out/bench_${TAG}_${CFG}.json
timeout 600 python bench.py --impl reference --config $CFG --steps 3 --warmup 1 > gpurun_out/bench_ref_${TAG}_${CFG}.json 2>&1; tail -c 300 gpurun_out/bench_ref_${TAG}_${CFG}.json
# profile the tiling the bench runs (the tuned one), without the tuning launches
export $(python tools/tuned_env.py $CFG 2>/dev/null | tail -1); echo "tiling: $LFSR_TILE_BL $LFSR_TILE_GNW"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
   python bench.py --config $CFG --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-flush > /dev/null 2>&1
for m in 1 0; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\(int\)${m}, \(bool\)" -s 3 -c 1 \
     -o gpurun_out/prof_${TAG}_${CFG}_m${m} -f python tools/quick_time.py $CFG 2 > gpurun_out/ncu_${TAG}_${CFG}_m${m}.log 2>&1
done
timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:k_cg_update" -s 3 -c 1 \
     -o gpurun_out/prof_${TAG}_${CFG}_upd -f python tools/quick_time.py $CFG 2 > /dev/null 2>&1
ls gpurun_out | grep ${TAG}
