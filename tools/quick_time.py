"""Quick device timing of the ADMM iteration on a config (development aid)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lfsr_synth as S
import paper_2206_05047_b200 as L

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C3"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
per_view = len(sys.argv) > 3 and sys.argv[3] == "pv"   # per-view disparity maps (A34)
user_psf = len(sys.argv) > 3 and sys.argv[3].startswith("psf")  # 45-degree motion kernel as B (A36); psf<len>
paper = len(sys.argv) > 3 and sys.argv[3] == "paper"    # the paper's backward-warp adjoint (A37)
t0 = time.time()
lf = S.make_lightfield(cfgname)
print("gen %.1fs" % (time.time() - t0), flush=True)
cfg = S.CONFIGS[cfgname]
p = L.params_for(cfg, S.defaults_for(cfg))
if paper:
    p.paper_adjoint = 1
if user_psf:
    n = int(sys.argv[3][3:]) if len(sys.argv[3]) > 3 else (5 if cfg.scale == 2 else 7)
    p.psf = S.motion_psf(n, 45.0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s = L.Solver(p, stream=stream.cuda_stream)
om = S.per_view_disparity(lf.omega, lf.n_views, amp=0.2, seed=3) if per_view else lf.omega
s.set_observations(*[torch.from_numpy(a).cuda() for a in (lf.y, lf.view_offsets, om)])
s.admm_run(2)
try:
    print("normal path:", s.normal_path, flush=True)
except Exception as ex:   # older library
    print("normal path: n/a", ex)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
# plain graph replay first (no per-kernel events: they would split programmatic launch edges)
e0.record(stream); s.admm_enqueue(iters); e1.record(stream); e1.synchronize()
plain = e0.elapsed_time(e1) / iters
s.profile(True)
tot = 0.0
for i in range(iters):
    e0.record(stream); s.admm_enqueue(1); e1.record(stream); e1.synchronize()
    tot += e0.elapsed_time(e1)
    s.profile_read()
ms, n = s.profile_read()
st = s.admm_stats(3, iters)
print(json.dumps({"cfg": cfgname, "per_view": per_view, "psf": user_psf, "paper_adjoint": paper, "ms_per_iter": plain, "it_per_s": 1000 / plain, "it_per_s_profiled": 1000 * iters / tot,
                  "kernel_ms_per_launch": [m / max(c, 1) for m, c in zip(ms, n)], "launches": n,
                  "J_first": st[0]["J"], "J_last": st[-1]["J"], "psnr": L.psnr(s.get_hr(), lf.x_gt),
                  "psnr_x0": None}))
