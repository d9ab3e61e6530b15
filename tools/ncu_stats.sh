#!/bin/bash
# Per-kernel instruction / issue / stall counters of the tile kernels (one ncu pass, a few
# metrics): tools/ncu_stats.sh <tag> <cfg> [lib]
TAG=$1; CFG=${2:-C3}
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_active.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
timeout 600 ncu --metrics $M --clock-control none --kernel-name-base demangled -k "regex:k_tile" -s 6 -c 6 --csv \
   python tools/quick_time.py $CFG 2 > gpurun_out/stats_${TAG}_${CFG}.csv 2> gpurun_out/stats_${TAG}_${CFG}.err
python - gpurun_out/stats_${TAG}_${CFG}.csv <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
rows = rows[[i for i, r in enumerate(rows) if "Kernel Name" in r][0]:]
h = rows[0]; ik = h.index("Kernel Name"); im = h.index("Metric Name"); iv = h.index("Metric Value")
d = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    d[r[ik]][r[im]].append(float(r[iv].replace(",", "")))
for k, m in d.items():
    print(k)
    for name, vals in sorted(m.items()):
        print("   %-80s %14.3f" % (name, sum(vals) / len(vals)))
PY
