"""Where the end-to-end solve time goes (development aid): set_observations (H2D + setup +
graph build), N ADMM iterations, get_hr — host wall clock around each call, warm."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lfsr_synth as S
import paper_2206_05047_b200 as L

cfg = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C3"]
lf = S.make_lightfield(cfg)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s = L.Solver(L.params_for(cfg, S.defaults_for(cfg)), stream=stream.cuda_stream)
host = [torch.from_numpy(a).pin_memory() for a in (lf.y, lf.view_offsets, lf.omega)]
xout = torch.empty((cfg.H, cfg.W), dtype=torch.float32).pin_memory()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.set_observations(*host)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s.admm_run(cfg.n_iters, want_stats=False)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    s.get_hr(xout)
    t3 = time.perf_counter()
    print("set_observations %.3f ms  admm_run(%d) %.3f ms  get_hr %.3f ms" % (1e3 * (t1 - t0), cfg.n_iters,
                                                                           1e3 * (t2 - t1), 1e3 * (t3 - t2)))
