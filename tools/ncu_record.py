"""Record the ncu counters bench.py reports next to its live timings.

    python tools/ncu_record.py <cfg> [normal=<rep>] [wz=<rep>] [upd=<rep>] [asm=<rep>] [irr=<rep>]

Reads each `ncu --set full` report (one launch each) with `ncu -i ... --page raw --csv`
and writes per-launch DRAM bytes, warp instructions and shared-memory wavefronts of the
kernel into profiles/ncu_traffic.json[<cfg>], stamped with bench.source_hash() of the
sources present when the capture ran (run this on the GPU box right after the capture).
bench.py uses a record only when its stamp matches the current sources.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

METRICS = {"dram": ("dram__bytes_read.sum", "dram__bytes_write.sum"),
           "instr": ("smsp__inst_executed.sum",),
           "wf": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",),
           "wf_ideal": ("memory_l1_wavefronts_shared_ideal",),
           "dur": ("gpu__time_duration.sum",)}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(head, units, vals):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-6, "nsecond": 1e-9,
                 "msecond": 1e-3, "us": 1e-6, "ns": 1e-9, "ms": 1e-3}.get(u, 1.0)
        d[h] = x * scale
    return d


def main():
    cfg = sys.argv[1]
    reps = dict(a.split("=", 1) for a in sys.argv[2:])
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    allrec = json.load(open(path)) if os.path.exists(path) else {}
    rec = {"build_hash": bench.source_hash(), "source": "tools/ncu_record.py " + " ".join(sys.argv[1:])}
    names = {"normal": "k_tile_normal", "wz": "k_tile_wz", "upd": "k_cg_update", "asm": "k_asm_normal",
             "irr": "k_asm_irr_scatter"}
    for kind, rep in reps.items():
        d = raw(rep)
        pre = names[kind]
        rec[pre + "_dram_bytes"] = int(sum(d.get(m, 0.0) for m in METRICS["dram"]))
        rec[pre + "_warp_instr"] = int(d.get(METRICS["instr"][0], 0.0))
        rec[pre + "_smem_wavefronts"] = int(d.get(METRICS["wf"][0], 0.0))
        if METRICS["wf_ideal"][0] in d:
            rec[pre + "_smem_wavefronts_ideal"] = int(d[METRICS["wf_ideal"][0]])
        rec[pre + "_ncu_duration_us"] = d.get(METRICS["dur"][0], 0.0) * 1e6
    allrec[cfg] = rec
    json.dump(allrec, open(path, "w"), indent=1)
    print(json.dumps(rec))


if __name__ == "__main__":
    main()
