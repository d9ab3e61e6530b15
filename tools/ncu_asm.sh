# development: ncu --set full of one CG step's assembled-operator kernels on a config
CFG=${1:-C3}; TAG=${2:-a}
mkdir -p gpurun_out
LFSR_ASM=1 timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_asm_normal|k_asm_irr}" -s ${SKIP:-4} -c ${COUNT:-4} \
   -o gpurun_out/prof_asm_${TAG}_${CFG} -f python tools/quick_time.py $CFG 2 > gpurun_out/ncu_asm_${TAG}_${CFG}.log 2>&1
tail -3 gpurun_out/ncu_asm_${TAG}_${CFG}.log
