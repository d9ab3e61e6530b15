#!/bin/bash
# Round-2 GPU call: [parity tests + smoke], ncu captures of the C3 kernels (recorded into
# profiles/ncu_traffic.json with the source hash), the launch list, then bench (N=1) on C3.
# usage: tools/gpu_r02.sh <tag> [tests|notests|quick] [config] [ncu|noncu]
TAG=${1:-r02}
TESTS=${2:-tests}
CFG=${3:-C3}
NCU=${4:-ncu}
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
if [ "$NCU" = "ncu" ]; then
  ( export $(python tools/tuned_env.py $CFG 2>/dev/null | tail -1)
    for m in 1 0; do
      timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\(int\)${m}, \(bool\)" -s 3 -c 1 \
         -o gpurun_out/prof_${TAG}_${CFG}_m${m} -f python tools/quick_time.py $CFG 2 > gpurun_out/ncu_${TAG}_${CFG}_m${m}.log 2>&1
    done
    timeout 900 ncu --set full --clock-control none --kernel-name-base demangled -k "regex:k_cg_update" -s 3 -c 1 \
         -o gpurun_out/prof_${TAG}_${CFG}_upd -f python tools/quick_time.py $CFG 2 > /dev/null 2>&1
    python tools/ncu_record.py $CFG normal=gpurun_out/prof_${TAG}_${CFG}_m1.ncu-rep wz=gpurun_out/prof_${TAG}_${CFG}_m0.ncu-rep \
         upd=gpurun_out/prof_${TAG}_${CFG}_upd.ncu-rep > gpurun_out/ncu_record_${TAG}.txt 2>&1
    cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_${TAG}.json
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
       python bench.py --config $CFG --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-flush --extra "" > /dev/null 2>&1 )
fi
timeout 1200 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err; tail -c 600 gpurun_out/bench_${TAG}_${CFG}.json
ls gpurun_out | grep ${TAG}
