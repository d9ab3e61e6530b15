"""Per-iterate GPU-vs-oracle diagnostics for a config (development aid)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import lfsr_synth as S
import oracle as O
import paper_2206_05047_b200 as L
from test_gpu_parity import run_pair, rel_l2

cfg = sys.argv[1] if len(sys.argv) > 1 else "C1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
lf = S.make_lightfield(cfg)
p, ora, xs, stats, st = run_pair(L, lf, n)
print("x rel err per iterate:", " ".join("%.1e" % rel_l2(xs[i], ora.x_iters[i]) for i in range(n + 1)))
print("J rel err:", " ".join("%.1e" % (abs(g["J"] - o["J"]) / abs(o["J"])) for g, o in zip(stats, ora.stats)))
print("res rel err:", " ".join("%.1e" % (abs(g["primal_res"] - o["primal_res"]) / o["primal_res"]) for g, o in zip(stats, ora.stats)))
print("wA rel:", rel_l2(st["wA"], ora.wA), "wS rel:", rel_l2(st["wS"], ora.wS))
for d in range(ora.wS.shape[0]):
    e = np.abs(st["wS"][d] - ora.wS[d])
    if e.max() > 1e-3:
        yx = np.unravel_index(np.argmax(e), e.shape)
        print(" plane", d, "max err", e.max(), "at", yx, "gpu", st["wS"][d][yx], "ora", ora.wS[d][yx])
