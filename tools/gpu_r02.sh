#!/bin/bash
# Round-2 GPU call: parity tests (with the PARITY log lines), smoke, bench (N=1) on C3.
# usage: tools/gpu_r02.sh <tag> [tests|notests|quick] [config]
TAG=${1:-r02}
TESTS=${2:-tests}
CFG=${3:-C3}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_${TAG}.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.txt 2>&1 || { tail -20 gpurun_out/build_${TAG}.txt; exit 1; }
if [ "$TESTS" = "tests" ]; then
  timeout 2400 python -m pytest tests/ -q -m gpu -rP > gpurun_out/pytest_gpu_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.txt
  grep -h "^PARITY" gpurun_out/pytest_gpu_${TAG}.txt > gpurun_out/parity_${TAG}.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.txt 2>&1; tail -1 gpurun_out/smoke_${TAG}.txt
fi
if [ "$TESTS" = "quick" ]; then
  timeout 1200 python -m pytest tests/ -q -m gpu -x -k "operator_parity or adjoint or C1 or misr or device or two_contexts or error" > gpurun_out/pytest_quick_${TAG}.txt 2>&1; tail -3 gpurun_out/pytest_quick_${TAG}.txt
fi
timeout 900 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err; tail -c 600 gpurun_out/bench_${TAG}_${CFG}.json
for c in C4 C5 C2; do timeout 300 python tools/quick_time.py $c 10 > gpurun_out/qt_${TAG}_$c.txt 2>&1; tail -1 gpurun_out/qt_${TAG}_$c.txt | cut -c1-300; done
ls gpurun_out | grep ${TAG}
