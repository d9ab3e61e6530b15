"""Per-CTA phase times of one NORMAL launch (development; needs the LFSR_CTA_TIMING variant build:
tools/build_variants.sh "ctat:-DLFSR_CTA_TIMING -rdc=false").  python tools/cta_timing.py C3"""
import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lfsr_synth as S
import paper_2206_05047_b200 as L

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
lf = S.make_lightfield(cfg)
p = L.params_for(S.CONFIGS[cfg], S.defaults_for(cfg))
s = L.Solver(p)
s.set_observations(lf.y, lf.view_offsets, lf.omega)
s.admm_run(2)
torch.cuda.synchronize()
tc = s.tile_config
n = 4096
buf = (ctypes.c_ulonglong * (4 * n))()
s.lib.lfsr_debug_cta_times(buf, n)
t = np.array(buf, dtype=np.float64).reshape(n, 4)
nb = tc["view_groups"] * ((p.lr_height + tc["tile_rows"] - 1) // tc["tile_rows"]) * ((p.lr_width + 29) // 30)
t = t[:nb]   # the last NORMAL launch wrote every one of its CTAs (earlier launches of other grids may linger past nb)
t0 = t[:, 0].min()
dur = (t[:, 3] - t[:, 0]) / 1e3
views = (t[:, 1] - t[:, 0]) / 1e3
nl = (t[:, 2] - t[:, 1]) / 1e3
fl = (t[:, 3] - t[:, 2]) / 1e3
start = (t[:, 0] - t0) / 1e3
ntx = (p.lr_width + 29) // 30
print(json.dumps({"cfg": cfg, "ctas": nb, "tile_config": tc, "kernel_span_us": float((t[:, 3].max() - t0) / 1e3),
                  "cta_us": [float(np.min(dur)), float(np.mean(dur)), float(np.max(dur))],
                  "views_us": [float(np.min(views)), float(np.mean(views)), float(np.max(views))],
                  "nltv_us": [float(np.min(nl)), float(np.mean(nl)), float(np.max(nl))],
                  "flush_us": [float(np.min(fl)), float(np.mean(fl)), float(np.max(fl))],
                  "start_spread_us": float(start.max())}))
print("per tile row (mean us):", " ".join("%.0f" % dur[r * ntx:(r + 1) * ntx].mean() for r in range(nb // ntx)))
print("per tile col (mean us):", " ".join("%.0f" % dur[c::ntx].mean() for c in range(ntx)))
print("sorted CTA durations (us):", " ".join("%.0f" % v for v in np.sort(dur)[::8]))
order = np.argsort(-dur)[:12]
for i in order:
    print("cta %3d tile (%d,%d) start %.1f dur %.1f views %.1f nltv %.1f flush %.1f" % (
        i, (i % (nb)) // ntx, i % ntx, start[i], dur[i], views[i], nl[i], fl[i]))
