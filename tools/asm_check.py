"""development: the assembled operator vs the tile kernel on a config (operator and 2 ADMM iterations)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import lfsr_synth as S
import paper_2206_05047_b200 as L

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2
lf = S.make_lightfield(name)
cfg = S.CONFIGS[name]
p = L.params_for(cfg, S.defaults_for(cfg))
xin = np.random.default_rng(1).uniform(-1, 1, (p.H, p.W)).astype(np.float32)
res = {}
for flag in ("1", "0"):
    os.environ["LFSR_ASM"] = flag
    s = L.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega)
    print(flag, s.normal_path, flush=True)
    q = s.op("NORMAL", xin)
    xs = []
    for i in range(n):
        st = s.admm_run(1)
        xs.append(s.get_hr())
    res[flag] = (q, xs, st)
    s.close()
rel = lambda a, b: float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))
qa, qt = res["1"][0], res["0"][0]
print("NORMAL asm vs tile %.3e" % rel(qa, qt))
d = np.abs(qa - qt)
iy, ix = np.unravel_index(np.argmax(d), d.shape)
print("max abs diff %.3e at (%d, %d), |q| there %.3e, max|q| %.3e" % (d.max(), iy, ix, abs(qt[iy, ix]), np.abs(qt).max()))
rows = np.where(d.max(axis=1) > 1e-3 * np.abs(qt).max())[0]
cols = np.where(d.max(axis=0) > 1e-3 * np.abs(qt).max())[0]
print("bad rows", rows[:20], len(rows), "bad cols", cols[:20], len(cols))
for i in range(n):
    print("iter", i + 1, "x asm vs tile %.3e" % rel(res["1"][1][i], res["0"][1][i]))
