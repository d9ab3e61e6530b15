"""development: small solves through the assembled CG operator at zeta = 2, 3, 4 (ragged shapes,
several tiles, irregular rows), for compute-sanitizer (tools/sanitize.sh)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LFSR_ASM", "1")
import numpy as np
import lfsr_synth as S
import paper_2206_05047_b200 as L

for seed, nv, h, w, z in ((2, 9, 40, 70, 2), (3, 9, 23, 47, 3), (4, 9, 17, 33, 4)):
    y, vo, om, _ = S.random_instance(seed, nv, h, w, z, grid=3)
    p = L.Params(n_views=nv, lr_height=h, lr_width=w, scale=z, ref_view=nv // 2)
    s = L.Solver(p)
    s.set_observations(y, vo, om)
    info = s.normal_path
    s.admm_run(2)
    q = s.op("NORMAL", np.random.default_rng(seed).uniform(-1, 1, (p.H, p.W)).astype(np.float32))
    print("zeta %d %s irregular %d/%d finite %s" % (z, info["name"], info["irregular_rows"], info["total_rows"],
                                                   bool(np.isfinite(q).all() and np.isfinite(s.get_hr()).all())))
    s.close()
