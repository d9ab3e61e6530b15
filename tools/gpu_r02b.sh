#!/bin/bash
# Round-2 GPU call with the assembled CG operator: [GPU tests + smoke], ncu
# captures of the C3 kernels of the path the library chose (k_asm_normal, k_asm_irr_scatter, the
# wz-step tile kernel, k_cg_update; recorded into profiles/ncu_traffic.json with the source hash),
# the cold-cache launch list, then bench (N=1).   usage: tools/gpu_r02b.sh <tag> [tests|notests] [config] [ncu|noncu]
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
if [ "$NCU" = "ncu" ]; then
  ( export $(python tools/tuned_env.py $CFG 2>/dev/null | tail -1)
    export LFSR_ASM=1   # ncu serialises and replays kernels: the timed path choice would not see the bench's choice
    Q="python tools/quick_time.py $CFG 2"
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_asm_normal" -s 6 -c 1 \
       -o gpurun_out/prof_${TAG}_${CFG}_asm -f $Q > gpurun_out/ncu_${TAG}_${CFG}_asm.log 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_asm_irr_scatter" -s 6 -c 1 \
       -o gpurun_out/prof_${TAG}_${CFG}_irr -f $Q > /dev/null 2>&1
    timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:\(int\)0, \(bool\)" -s 1 -c 1 \
       -o gpurun_out/prof_${TAG}_${CFG}_m0 -f $Q > gpurun_out/ncu_${TAG}_${CFG}_m0.log 2>&1
    timeout 900 ncu --set full --clock-control none -k "regex:k_cg_update" -s 3 -c 1 \
       -o gpurun_out/prof_${TAG}_${CFG}_upd -f $Q > /dev/null 2>&1
    python tools/ncu_record.py $CFG asm=gpurun_out/prof_${TAG}_${CFG}_asm.ncu-rep irr=gpurun_out/prof_${TAG}_${CFG}_irr.ncu-rep \
         wz=gpurun_out/prof_${TAG}_${CFG}_m0.ncu-rep upd=gpurun_out/prof_${TAG}_${CFG}_upd.ncu-rep > gpurun_out/ncu_record_${TAG}.txt 2>&1
    cp profiles/ncu_traffic.json gpurun_out/ncu_traffic_${TAG}.json
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${TAG}_${CFG}.csv \
       python bench.py --config $CFG --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-flush --extra "" > /dev/null 2>&1 )
fi
timeout 1500 python bench.py --config $CFG --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_${CFG}.json 2> gpurun_out/bench_${TAG}_${CFG}.err; tail -c 600 gpurun_out/bench_${TAG}_${CFG}.json
ls gpurun_out | grep ${TAG}
