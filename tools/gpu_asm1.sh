# development: assembled-operator tests, A/B timing and a launch list (tools/quick_time.py)
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_asm.py -x -q -s 2>&1 | tail -30
for c in ${CFGS:-C3 C4}; do LFSR_ASM=1 timeout 300 python tools/quick_time.py $c 10; done
LFSR_ASM=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/asm_launches.csv python tools/quick_time.py C3 3 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/asm_launches.csv")))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        agg[r[ki][:60]].append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print("%-60s n=%3d mean %.1f us" % (k, len(v), sum(v) / len(v) / 1000))
PY
