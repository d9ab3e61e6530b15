#!/usr/bin/env python
"""Benchmark of the ADMM light-field super-resolution hot path (arXiv 2206.05047).

A "step" is one ADMM iteration (Alg.1: weights, data shrink/dual, NLTV
shrink/dual, v, and K = 5 CG steps of Alg.2) over the whole synthetic light field of
the bench workload (default C3: 9x9 views, 256x256 LR -> x2, 512x512 HR, sigma=0.05 +
20 % impulse; BASELINE.json configs[2], the "9x9 LF x2" of the metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl ours|reference]

Timing: W untimed warm-up steps, then exactly K steps, each bracketed by CUDA events on
the solver's stream, with an L2 flush (a 512 MiB write) between steps outside the events;
the sum of the K step times is the step time; barrier + synchronize on both sides; max
over ranks.  value = (ADMM iterations done by all ranks) / that time.  Multi-GPU (N > 1,
default `--multi strips`): one light field of the same workload split into HR row strips,
halo exchange and scalar all-reduces over NCCL (SURVEY §8e, strong scaling); the
replica mode (every rank its own light field, no data-path collective) is reported as
an extra key, and a C5 strip run as another.

Extra keys at N = 1: `extra_configs` (C4 = the metric's x3 workload, C5 = the largest
config) each with its own roofline; `cpu_baseline` times the oracle at all host cores
and at one thread.

--impl reference times the fp64 CPU oracle (oracle/, the only baseline this tier has)
on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "ADMM iters/s and HR Mpix/s, 9x9 LF x2/x3 SR; HBM GB/s vs B200 peak"
UNIT = "ADMM iters/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--e2e-batch", type=int, default=10, help="light fields per lfsr_solve_batch call in the e2e leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--multi", default="strips", choices=["replicas", "strips"],
                    help="N > 1: independent light fields per rank (weak scaling) or one light field split "
                         "into HR row strips with NCCL halo exchange (strong scaling, DESIGN.md §10)")
    ap.add_argument("--extra", default="C4,C5", help="extra configs measured after the main one ('' = none)")
    ap.add_argument("--extra-steps", type=int, default=6)
    return ap.parse_args()


# ----------------------------------------------------------------------------- algorithmic model
def algorithmic(cfg, d):
    """Per-launch algorithmic bytes and flops of the kernels."""
    sk, p, q = cfg.n_views, cfg.H * cfg.W, cfg.lr_h * cfg.lr_w
    sd = (2 * d.radius + 1) ** 2 - 1
    z = cfg.scale
    R = math.ceil(3 * 0.25 * math.sqrt(z * z - 1))
    fA = 10 + 2 * (2 * R + 1) * (1.0 / z + 1.0 / z ** 2)     # flops per HR px per view, one direction
    K = d.cg_max_iters
    normal_flops = 2 * sk * fA * p + 7 * sd * p              # A + A^T over all views + S^T S stencil
    normal_bytes = 4 * p * 6                                 # r, p_prev (read), p (write), omega, m, q (RED)
    wz_flops = 2 * sk * fA * p + 10 * sd * p + 8 * sk * q
    wz_bytes = 4 * (3 * sk * q + 2 * sd * p + 5 * p)
    upd_bytes = 4 * p * 6                                    # x, r, p updates (24p)
    iter_bytes = wz_bytes + K * (normal_bytes + upd_bytes)   # B = 4(3 s_k q + 2 s_d p + 5p) + K 48p
    iter_flops = wz_flops + K * normal_flops
    return dict(normal_flops=normal_flops, normal_bytes=normal_bytes, wz_flops=wz_flops, wz_bytes=wz_bytes,
                upd_bytes=upd_bytes, iter_bytes=iter_bytes, iter_flops=iter_flops)


def peaks():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json) and the FP32 CUDA-core peak derived from
    the unit counts and clock (148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz)."""
    hbm, sm_mhz, src = 6650.0, 1965.0, "fallback (B200_PROFILING.md)"
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        try:
            j = json.load(open(path))
            hbm = float(j.get("hbm_gbs", hbm))
            sm_mhz = float(j.get("sm_max_mhz", sm_mhz))
            src = "measured (MEASURED_PEAKS.json)"
        except Exception:
            pass
    fp32 = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    return hbm, fp32, src, sm_mhz * 1e6


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([v.strip() for v in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) >= 7:
                for n, v in zip(names, s[3:7]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle
def oracle_params(cfg, d):
    import oracle as O
    return O.Params(n_views=cfg.n_views, lr_h=cfg.lr_h, lr_w=cfg.lr_w, scale=cfg.scale, ref_view=cfg.ref_view,
                    radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2, lambda_reg=d.lambda_reg,
                    sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1, sigma_o2=d.sigma_o2, theta=d.theta,
                    cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol,
                    offset_weights=getattr(d, "offset_weights", None))


def time_oracle(lf, cfg, d, iters=1, threads=None):
    """Seconds per ADMM iteration of the fp64 oracle as it stands (all host cores, or `threads`)."""
    import ctypes
    import oracle as O
    O.build()
    O.lib()
    P = oracle_params(cfg, d)
    gomp = None
    if threads is not None:
        try:   # the oracle's OpenMP runtime (libgomp, already loaded with liboracle.so)
            gomp = ctypes.CDLL("libgomp.so.1")
            gomp.omp_set_num_threads(int(threads))
        except OSError:
            gomp = None
    try:
        t0 = time.perf_counter()
        O.admm(P, lf.y, lf.view_offsets, lf.omega, iters)
        return (time.perf_counter() - t0) / iters
    finally:
        if gomp is not None:
            gomp.omp_set_num_threads(int(os.cpu_count() or 1))


def source_hash():
    """sha256 over the CUDA sources of liblfsr (csrc/*): ncu counters recorded in
    profiles/ncu_traffic.json are used only when they were captured from this build."""
    import hashlib
    h = hashlib.sha256()
    d = os.path.join(ROOT, "paper_2206_05047_b200", "csrc")
    for n in sorted(os.listdir(d)):
        if n.endswith((".cu", ".cuh", ".h")):
            h.update(n.encode())
            h.update(open(os.path.join(d, n), "rb").read())
    return h.hexdigest()[:16]


def ncu_record(cfg_name):
    """The ncu counters of this config's kernels, if captured from the current sources."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return {}, "no profiles/ncu_traffic.json"
    try:
        rec = json.load(open(path)).get(cfg_name, {})
    except Exception as e:  # pragma: no cover
        return {}, "unreadable: %s" % e
    if not rec:
        return {}, "no record for %s" % cfg_name
    if rec.get("build_hash") != source_hash():
        return {}, "stale: captured from build %s, current sources %s" % (rec.get("build_hash"), source_hash())
    return rec, "ncu --set full of build %s (%s)" % (rec.get("build_hash"), rec.get("source", ""))


def cores():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, cfg, d, rank):
    if rank != 0:
        return
    import lfsr_synth as S
    lf = S.make_lightfield(cfg)
    sample = "%s: one full ADMM iteration (K=%d CG steps) per step, fp64 oracle, OMP threads=%d" % (
        cfg.name, d.cg_max_iters, cores())
    for _ in range(min(args.warmup, 1)):   # a CPU program needs no long warm-up
        time_oracle(lf, cfg, d, 1)
    ts = [time_oracle(lf, cfg, d, 1) for _ in range(args.steps)]
    t = sum(ts)
    value = args.steps / t
    hr_mpix = cfg.H * cfg.W / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": 1000 * t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "hr_mpix_it_per_s": value * hr_mpix,
            "config": {"workload": cfg.name, "desc": cfg.note, "views": cfg.n_views, "scale": cfg.scale,
                       "hr": [cfg.H, cfg.W], "cg_steps": d.cg_max_iters, "l2_flush": "n/a (CPU)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores(), "kind": "oracle", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def roofline_for(cfg, d, kms, kn, t_ms, steps, share, clk_hz, npath=None, split=None):
    """Roofline of the dominant kernel from the per-kernel CUDA-event times of the profiled region,
    plus the other kernels' fractions.  Tile-kernel CG operator: k_tile<NORMAL> (FP32 / LSU / issue).
    Assembled CG operator: the kernel with the largest share of the step among the
    wz-step tile kernel (FP32), the stencil kernel k_asm_normal (HBM) and the irregular-row kernels."""
    if npath and npath.get("name") == "assembled" and split and split[1] > 0:
        return roofline_assembled(cfg, d, kms, kn, t_ms, steps, share, clk_hz, npath, split)
    alg = algorithmic(cfg, d)
    hbm_peak, fp32_peak, peak_src, _ = peaks()
    k_normal_ms = kms[1] / max(kn[1], 1)
    k_wz_ms = kms[0] / max(kn[0], 1)
    k_upd_ms = kms[2] / max(kn[2], 1)
    achieved = alg["normal_flops"] / (k_normal_ms / 1000.0) / 1e12
    rec, rec_src = ncu_record(cfg.name)
    roofline = {"bound": "alu", "kernel": "k_tile<NORMAL> (CG normal operator q = M p, a8)",
                "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
                "traffic": rec.get("k_tile_normal_dram_bytes"),
                "peak_source": "FP32 CUDA cores, 148 SM x 128 lanes x 2 x sm_max_mhz (%s)" % peak_src,
                "algorithmic_flops_per_launch": alg["normal_flops"], "avg_launch_ms": k_normal_ms,
                "share_of_step": kms[1] / max(sum(kms), 1e-9),
                "timing": "per-kernel CUDA events on the library stream over a second timed region of the "
                          "same %d steps" % steps,
                "ncu_counters": rec_src,
                "wz_step": {"avg_launch_ms": k_wz_ms, "alg_bytes": alg["wz_bytes"],
                            "hbm_gbs": alg["wz_bytes"] / (k_wz_ms / 1000.0) / 1e9,
                            "hbm_frac": alg["wz_bytes"] / (k_wz_ms / 1000.0) / 1e9 / hbm_peak,
                            "traffic": rec.get("k_tile_wz_dram_bytes")},
                "cg_update": {"avg_launch_ms": k_upd_ms, "alg_bytes": 4 * cfg.H * cfg.W * 7,
                              "hbm_gbs": 4 * cfg.H * cfg.W * 7 / (k_upd_ms / 1000.0) / 1e9,
                              "hbm_frac": 4 * cfg.H * cfg.W * 7 / (k_upd_ms / 1000.0) / 1e9 / hbm_peak,
                              "traffic": rec.get("k_cg_update_dram_bytes")},
                "iteration_alg_bytes": alg["iter_bytes"],
                # per GPU: a strip rank moves 1/share of the iteration's bytes
                "iteration_hbm_gbs": alg["iter_bytes"] * steps / (t_ms / 1000.0) / 1e9 / share,
                "iteration_hbm_frac": alg["iter_bytes"] * steps / (t_ms / 1000.0) / 1e9 / share / hbm_peak,
                "hbm_peak_gbs": hbm_peak}
    winst = rec.get("k_tile_normal_warp_instr")
    if winst:   # instruction issue (1 warp instruction / scheduler / clock)
        issue_peak = 148 * 4 * clk_hz / 1e12
        roofline["issue"] = {"achieved": winst / (k_normal_ms / 1000.0) / 1e12, "peak": issue_peak,
                             "unit": "T warp-instr/s", "frac": winst / (k_normal_ms / 1000.0) / 1e12 / issue_peak,
                             "warp_instr_per_launch": winst,
                             "source": "ncu smsp__inst_executed.sum per launch / live launch time; "
                                       "peak = 148 SM x 4 schedulers x sm_max_mhz"}
    wf = rec.get("k_tile_normal_smem_wavefronts")
    if wf:      # shared-memory data pipe (LSU): 1 wavefront / SM / clock (SURVEY §8d's binding roofline)
        lsu_peak = 148 * clk_hz / 1e12
        roofline["lsu"] = {"achieved": wf / (k_normal_ms / 1000.0) / 1e12, "peak": lsu_peak,
                           "unit": "T smem-wavefronts/s", "frac": wf / (k_normal_ms / 1000.0) / 1e12 / lsu_peak,
                           "wavefronts_per_launch": wf,
                           "ideal_wavefronts_per_launch": rec.get("k_tile_normal_smem_wavefronts_ideal"),
                           "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum per launch / live launch "
                                     "time; peak = 148 SM x 1 wavefront/clk x sm_max_mhz"}
    return roofline


def roofline_assembled(cfg, d, kms, kn, t_ms, steps, share, clk_hz, npath, split):
    alg = algorithmic(cfg, d)
    hbm_peak, fp32_peak, peak_src, _ = peaks()
    rec, rec_src = ncu_record(cfg.name)
    p = cfg.H * cfg.W
    z = cfg.scale
    R = math.ceil(3 * 0.25 * math.sqrt(z * z - 1))
    nsw = 2 * (2 * R + 1) + 1
    nf = (nsw * nsw + 1) // 2                             # stored stencil planes (symmetric half + centre)
    sms, n = split
    k_st_ms, k_irr_ms = sms[0] / max(n, 1), sms[1] / max(n, 1)
    k_wz_ms, k_upd_ms = kms[0] / max(kn[0], 1), kms[2] / max(kn[2], 1)
    st_bytes = 4 * p * (nf + 5)                           # half planes + r, p_{k-1}, m (read), p_k, q (write);
                                                          # the transposed half's neighbour reads are L1/L2 re-reads
    tot = max(sum(kms), 1e-9)
    stencil = {"bound": "hbm", "kernel": "k_asm_normal (assembled CG operator: %d half-stencil planes + NLTV, a8)" % nf,
               "achieved": st_bytes / (k_st_ms / 1000.0) / 1e9, "peak": hbm_peak, "unit": "GB/s",
               "frac": st_bytes / (k_st_ms / 1000.0) / 1e9 / hbm_peak, "traffic": rec.get("k_asm_normal_dram_bytes"),
               "algorithmic_bytes_per_launch": st_bytes, "avg_launch_ms": k_st_ms, "share_of_step": sms[0] / tot,
               "peak_source": "HBM copy bandwidth, %s" % peak_src}
    wz_ach = alg["wz_flops"] / (k_wz_ms / 1000.0) / 1e12
    wz = {"bound": "alu", "kernel": "k_tile<WZ> (wz-step: weights, A_k / A_k^T over all views, shrink, duals, a2-a7)",
          "achieved": wz_ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": wz_ach / fp32_peak,
          "traffic": rec.get("k_tile_wz_dram_bytes"), "algorithmic_flops_per_launch": alg["wz_flops"],
          "avg_launch_ms": k_wz_ms, "share_of_step": kms[0] / tot,
          "hbm_gbs": alg["wz_bytes"] / (k_wz_ms / 1000.0) / 1e9,
          "hbm_frac": alg["wz_bytes"] / (k_wz_ms / 1000.0) / 1e9 / hbm_peak,
          "peak_source": "FP32 CUDA cores, 148 SM x 128 lanes x 2 x sm_max_mhz (%s)" % peak_src}
    winst, wf = rec.get("k_tile_wz_warp_instr"), rec.get("k_tile_wz_smem_wavefronts")
    if winst:   # instruction issue (1 warp instruction / scheduler / clock)
        issue_peak = 148 * 4 * clk_hz / 1e12
        wz["issue"] = {"achieved": winst / (k_wz_ms / 1000.0) / 1e12, "peak": issue_peak, "unit": "T warp-instr/s",
                       "frac": winst / (k_wz_ms / 1000.0) / 1e12 / issue_peak, "warp_instr_per_launch": winst,
                       "source": "ncu smsp__inst_executed.sum per launch / live launch time; peak = 148 SM x 4 "
                                 "schedulers x sm_max_mhz"}
    if wf:      # shared-memory data pipe: 1 wavefront / SM / clock
        lsu_peak = 148 * clk_hz / 1e12
        wz["lsu"] = {"achieved": wf / (k_wz_ms / 1000.0) / 1e12, "peak": lsu_peak, "unit": "T smem-wavefronts/s",
                     "frac": wf / (k_wz_ms / 1000.0) / 1e12 / lsu_peak, "wavefronts_per_launch": wf,
                     "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum per launch / live launch time"}
    irr = {"kernels": "k_asm_irr_u + k_asm_irr_t + k_asm_irr_scatter (rows across depth edges, applied as rows)",
           "avg_pass_ms": k_irr_ms, "share_of_step": sms[1] / tot, "irregular_rows": npath.get("irregular_rows"),
           "total_rows": npath.get("total_rows")}
    dom = stencil if sms[0] >= kms[0] else wz
    roofline = dict(dom)
    roofline.update({
        "timing": "per-kernel CUDA events on the library stream over a second timed region of the same %d steps" % steps,
        "ncu_counters": rec_src,
        "stencil_kernel" if dom is wz else "wz_step": stencil if dom is wz else wz,
        "irregular_rows": irr,
        "normal_operator_pass_ms": kms[1] / max(kn[1], 1),
        "cg_update": {"avg_launch_ms": k_upd_ms, "alg_bytes": 4 * p * 7,
                      "hbm_gbs": 4 * p * 7 / (k_upd_ms / 1000.0) / 1e9,
                      "hbm_frac": 4 * p * 7 / (k_upd_ms / 1000.0) / 1e9 / hbm_peak,
                      "traffic": rec.get("k_cg_update_dram_bytes")},
        "iteration_alg_bytes": alg["iter_bytes"],
        "iteration_hbm_gbs": alg["iter_bytes"] * steps / (t_ms / 1000.0) / 1e9 / share,
        "iteration_hbm_frac": alg["iter_bytes"] * steps / (t_ms / 1000.0) / 1e9 / share / hbm_peak,
        "hbm_peak_gbs": hbm_peak})
    return roofline


def time_steps(sol, stream, steps, do_flush, barrier):
    """`steps` plain graph replays, one CUDA event pair per step (flush outside the events),
    then the same steps with the library's per-kernel events (the roofline region)."""
    import torch
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier()
    for i in range(steps):
        do_flush()
        ev[i][0].record(stream)
        sol.admm_enqueue(1)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    barrier()
    t_ms = sum(a.elapsed_time(b) for a, b in ev)
    sol.profile_read()
    sol.profile(True)
    evp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier()
    for i in range(steps):
        do_flush()
        evp[i][0].record(stream)
        sol.admm_enqueue(1)
        evp[i][1].record(stream)
        evp[i][1].synchronize()
        sol.profile_read()
    barrier()
    t_prof_ms = sum(a.elapsed_time(b) for a, b in evp)
    kms, kn = sol.profile_read()
    split = sol.profile_read_split()   # assembled CG operator: (stencil kernel, irregular rows) ms
    sol.profile(False)
    return t_ms, t_prof_ms, kms, kn, split


def extra_config(name, steps, warmup, do_flush, barrier, local, clk_hz, multi_world=1, rank=0):
    """One more config in the same process (fresh solver): value, per-kernel times and roofline."""
    import torch
    import lfsr_synth as S
    import paper_2206_05047_b200 as L
    import torch.distributed as dist
    cfg = S.CONFIGS[name]
    d = S.defaults_for(cfg)
    lf = S.make_lightfield(cfg)
    stream = torch.cuda.Stream()
    p = L.params_for(cfg, d, device=local)
    if multi_world > 1:
        uid = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        p.n_ranks, p.rank, p.nccl_unique_id = multi_world, rank, uid[0]
    with torch.cuda.stream(stream):
        sol = L.Solver(p, stream=stream.cuda_stream)
        sol.set_observations(*[torch.from_numpy(a).cuda() for a in (lf.y, lf.view_offsets, lf.omega)])
        for _ in range(warmup):
            do_flush()
            sol.admm_enqueue(1)
        sol.admm_stats(1, warmup)
        t_ms, t_prof_ms, kms, kn, split = time_steps(sol, stream, steps, do_flush, barrier)
        st = sol.admm_stats(warmup + 1, steps)
        if multi_world > 1:
            tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ms = float(tt.item())
        rec = {"workload": cfg.name, "desc": cfg.note, "value": steps / (t_ms / 1000.0), "unit": UNIT,
               "ms_per_step": t_ms / steps, "steps": steps, "warmup": warmup,
               "hr_mpix_it_per_s": steps / (t_ms / 1000.0) * cfg.H * cfg.W / 1e6,
               "final_J": st[-1]["J"], "cg_iters": st[-1]["cg_iters"]}
        if kn[1] > 0:
            rec["kernel_ms_per_launch"] = {"wz": kms[0] / kn[0], "normal": kms[1] / kn[1], "cg_update": kms[2] / kn[2]}
            rec["normal_path"] = sol.normal_path
            rec["roofline"] = roofline_for(cfg, d, kms, kn, t_ms, steps, 1, clk_hz, rec["normal_path"], split)
        sol.close()
    del lf
    return rec


def cpu_baselines(lf, cfg, d):
    """The oracle as it stands on the host: all cores, then one thread."""
    out = []
    for thr in (None, 1):
        try:
            sec = time_oracle(lf, cfg, d, 1, threads=thr)
            n = cores() if thr is None else thr
            out.append({"value": 1.0 / sec, "unit": UNIT, "cores": n, "kind": "oracle", "cpu_model": cpu_model(),
                        "sample": "%s: one full ADMM iteration (wz-step + K=%d CG steps) of the fp64 oracle, "
                                  "%d OpenMP thread(s)" % (cfg.name, d.cg_max_iters, n)})
        except Exception as e:  # pragma: no cover
            out.append({"value": None, "unit": UNIT, "cores": thr or cores(), "kind": "oracle",
                        "sample": "failed: %s" % e})
    return out


def main():
    args = parse()
    import lfsr_synth as S
    cfg = S.CONFIGS[args.config]
    d = S.defaults_for(cfg)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, cfg, d, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2206_05047_b200 as L

    # development only: LFSR_BENCH_SHARE_GPU=1 runs all ranks on the visible GPUs round-robin with a
    # gloo group (exercises the multi-rank replica path on a 1-GPU box); the product launch is nccl
    share = os.environ.get("LFSR_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # (sharing one GPU, strips need an NCCL that allows it: LFSR_NCCL_LIB = the test double)
    strips = world > 1 and args.multi == "strips" and (not share or bool(os.environ.get("LFSR_NCCL_LIB")))
    # strips: every rank holds the same light field and owns a strip of it;
    # replicas: each rank super-resolves its own light field (independent problem, own seed)
    lf = S.make_lightfield(cfg, seed=None if (rank == 0 or strips) else 10007 * rank + 1000)
    stream = torch.cuda.Stream()          # a real (non-legacy) stream shared by torch and liblfsr
    torch.cuda.set_stream(stream)
    p = L.params_for(cfg, d, device=local)
    if strips:
        uid = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        p.n_ranks, p.rank, p.nccl_unique_id = world, rank, uid[0]
    sol = L.Solver(p, stream=stream.cuda_stream)
    dev_in = [torch.from_numpy(a).cuda() for a in (lf.y, lf.view_offsets, lf.omega)]
    sol.set_observations(*dev_in)
    npath = sol.normal_path   # which CG-operator implementation runs (tile kernel / MISR / assembled)
    flush = None if args.no_flush else torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def do_flush():
        if flush is not None:
            flush.fill_(1.0)

    for _ in range(args.warmup):
        do_flush()
        sol.admm_enqueue(1)
    sol.admm_stats(1, args.warmup) if args.warmup else None
    first = args.warmup + 1
    clocks = ClockSampler(local)
    clocks.start()
    # timed region 1 (the `value`): plain graph replays; region 2 (the roofline): the same steps with
    # an event after every kernel (~8 % slower at C3, so it only supplies per-kernel times)
    t_ms, t_prof_ms, kms, kn, split = time_steps(sol, stream, args.steps, do_flush, barrier)
    # kernels per timed step of the graph the value was measured on (read before the e2e leg, whose
    # batch may re-pick the CG-operator path for its own N)
    launches = sol.launches_per_iter * args.steps * (1 if strips else world)
    clk = clocks.stop()
    stats = sol.admm_stats(first, args.steps)   # raises on divergence
    sol.admm_stats(first + args.steps, args.steps)
    t_max = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    total_iters = args.steps * (1 if strips else world)
    value = total_iters / (t_max / 1000.0)
    hr_mpix = cfg.H * cfg.W / 1e6

    # ---- end to end through the public API with host buffers (full solves of N iterations)
    e2e = None
    if args.e2e_steps > 0:
        # distinct light fields (own scene / noise seeds) cycled through the e2e leg
        n_distinct = 1 if strips else 3
        fields_np = [lf] + [S.make_lightfield(cfg, seed=7919 * (i + 1) + 1000) for i in range(n_distinct - 1)]
        hosts = [tuple(torch.from_numpy(a).pin_memory() for a in (f.y, f.view_offsets, f.omega)) for f in fields_np]
        host = hosts[0]
        xout = torch.empty((cfg.H, cfg.W), dtype=torch.float32).pin_memory()
        n_it = cfg.n_iters
        sol.profile(False)
        # warm (allocations are reused for the same geometry)
        sol.set_observations(*host)
        sol.admm_run(n_it, want_stats=False)
        sol.get_hr(xout)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for i in range(args.e2e_steps):
            do_flush()
            e0.record(stream)
            sol.set_observations(*hosts[i % n_distinct])   # H2D of y, offsets, omega + setup (a1)
            sol.admm_run(n_it, want_stats=False)           # N iterations, divergence-checked
            sol.get_hr(xout)                               # D2H of x (blocks)
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([tot], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            tot = float(tt.item())
        h2d = sum(int(h.numel()) * 4 for h in host)
        seq = {"value": args.e2e_steps * n_it * (1 if strips else world) / (tot / 1000.0),
               "ms_per_solve": tot / args.e2e_steps,
               "step": "one field at a time: set_observations (H2D + setup) + %d ADMM iterations + get_hr (D2H), "
                       "%d distinct light fields cycled" % (n_it, n_distinct)}
        e2e = {"value": seq["value"], "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(xout.numel()) * 4 + 8 * 11 * n_it,
               "step": seq["step"], "ms_per_solve": seq["ms_per_solve"],
               "solve_hr_mpix_per_s": (1 if strips else world) * hr_mpix / (tot / args.e2e_steps / 1000.0),
               "psnr_db": L.psnr(xout.numpy(), fields_np[(args.e2e_steps - 1) % n_distinct].x_gt)}
        if not strips:
            # the serving path (lfsr_solve_batch): field i+1's H2D + setup maxima on a second stream
            # while field i solves; every field's inputs still cross PCIe and every x comes back
            nb = max(1, min(args.e2e_batch, args.e2e_steps))
            outs = [torch.empty((cfg.H, cfg.W), dtype=torch.float32).pin_memory() for _ in range(nb)]
            fields = [hosts[i % n_distinct] for i in range(nb)]
            sol.solve_batch(fields, n_it, outs)   # warm
            barrier()
            tb, nf = 0.0, 0
            while nf < args.e2e_steps:
                do_flush()
                e0.record(stream)
                sol.solve_batch(fields, n_it, outs)
                e1.record(stream)
                e1.synchronize()
                tb += e0.elapsed_time(e1)
                nf += nb
            if world > 1:
                tt = torch.tensor([tb], dtype=torch.float64, device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                tb = float(tt.item())
            e2e = {"value": nf * n_it * world / (tb / 1000.0), "unit": UNIT,
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": int(xout.numel()) * 4 + 8 * 11,
                   "step": "one light field through lfsr_solve_batch (batches of %d, %d distinct light fields "
                           "cycled, L2 flushed between batches): H2D of y/offsets/omega + setup + %d ADMM "
                           "iterations + D2H of x, the next field's H2D overlapping this field's iterations"
                           % (nb, n_distinct, n_it),
                   "ms_per_solve": tb / nf,
                   "solve_hr_mpix_per_s": world * hr_mpix / (tb / nf / 1000.0),
                   "psnr_db": L.psnr(outs[0].numpy(), fields_np[0].x_gt),
                   "sequential": seq}
        del hosts

    # ---- roofline of the dominant kernel
    _, _, _, clk_hz = peaks()
    if kn[1] > 0:
        roofline = roofline_for(cfg, d, kms, kn, t_max, args.steps, world if strips else 1, clk_hz, npath, split)
        roofline["timing"] += " (%.4f ms/step with the events; `value` is the region without them)" % (
            t_prof_ms / args.steps)
        k_normal_ms, k_wz_ms, k_upd_ms = (kms[1] / kn[1], kms[0] / max(kn[0], 1), kms[2] / max(kn[2], 1))
    else:   # strips (NCCL): no per-kernel events in the graph; the kernels' roofline is the replica run's
        roofline, k_normal_ms, k_wz_ms, k_upd_ms = None, None, None, None
    sol.close()
    del dev_in

    # ---- extra configs (N = 1: the metric's x3 workload and the largest config) and, N > 1, the
    # other multi-GPU mode and C5 strips
    extras = {}
    names = [n for n in args.extra.split(",") if n and n != cfg.name]
    if world > 1:
        names = ["C5"] if "C5" in names else []
    for n in names:
        try:
            extras[n] = extra_config(n, args.extra_steps, 3, do_flush, barrier, local, clk_hz,
                                     multi_world=world if strips else 1, rank=rank)
            if strips:
                extras[n]["parallelism"] = "strips%d" % world
        except Exception as e:  # pragma: no cover
            extras[n] = {"workload": n, "error": str(e)[:300]}
    replicas = None
    if strips:
        try:
            rr = extra_config(cfg.name, args.steps, args.warmup, do_flush, barrier, local, clk_hz)
            tt = torch.tensor([rr["ms_per_step"]], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            replicas = {"value": world * 1000.0 / float(tt.item()), "unit": UNIT, "scaling": "weak",
                        "ms_per_step": float(tt.item()),
                        "mode": "dp%d: every rank its own light field, no data-path collective" % world}
            if roofline is None and rr.get("roofline"):
                roofline = dict(rr["roofline"])
                roofline["timing"] = ("per-kernel CUDA events of the replica run on this rank (the strip "
                                      "graphs carry no per-kernel events); " + roofline["timing"])
                k = rr["kernel_ms_per_launch"]
                k_normal_ms, k_wz_ms, k_upd_ms = k["normal"], k["wz"], k["cg_update"]
        except Exception as e:  # pragma: no cover
            replicas = {"error": str(e)[:300]}

    # ---- CPU baseline: the oracle as it stands, on a bounded sample, rank 0 at N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpus = cpu_baselines(lf, cfg, d)
        cpu = dict(cpus[0])
        cpu["single_thread"] = cpus[1]

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "strong" if strips else "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "hr_mpix_it_per_s": value * hr_mpix,
                "cu_per_s": value * 2 * (d.cg_max_iters + 1),   # computation units (A33)
                "paper_context": {
                    "gpu_vs_oracle": (value / cpu["value"]) if cpu and cpu.get("value") else None,
                    "gpu_vs_oracle_1thread": (value / cpu["single_thread"]["value"])
                    if cpu and cpu.get("single_thread", {}).get("value") else None,
                    "paper_gpu_vs_cpu": "43-77x: unnamed OpenCL GPUs vs an i7-5820K, one ADMM iteration, 9x9 "
                                        "views (P:L1194-1203); context only (other hardware, precision, workload)",
                    "paper_vs_fl_misr": "2.46x (x2) / 1.57x (x3): 1x GTX 1080Ti vs 4x GTX 1080Ti FL-MISR, DIV8K "
                                        "MISR (P:L1110-1120); context only"},
                "config": {"workload": cfg.name, "desc": cfg.note, "views": cfg.n_views, "scale": cfg.scale,
                           "hr": [cfg.H, cfg.W], "cg_steps": d.cg_max_iters, "nltv_window": "5x5",
                           "l2_flush": "512 MiB write between timed steps (outside the events)" if flush is not None else "none",
                           "parallelism": ("strips%d (one light field, HR row strips, NCCL halos)" % world) if strips
                           else "dp%d (independent light fields per rank)" % world},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches,
                "normal_path": npath,
                "clocks": clk,
                "kernel_ms_per_launch": {"wz": k_wz_ms, "normal": k_normal_ms, "cg_update": k_upd_ms},
                "final_J": stats[-1]["J"], "cg_iters": stats[-1]["cg_iters"],
                "build_hash": source_hash()}
        if extras:
            line["extra_configs"] = extras
        if replicas is not None:
            line["replicas"] = replicas
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
