"""The multi-GPU row-strip decomposition on one device: "virtual
ranks" run every strip's kernels and the exact exchange schedule of the NCCL
mode (halo fill, ring fold, scalar all-reduce) with device copies.  Results must
match the single-strip solve (1e-5) and the fp64 oracle (1e-4 per iterate)."""
import numpy as np
import pytest

import lfsr_synth as S
from test_gpu_parity import check_iterates, oparams, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _tile_kernel_reference(monkeypatch):
    """The single-strip reference runs the same operator implementation as the strips (the fused
    tile kernel), so the comparison isolates the decomposition (the assembled operator, which only
    a single strip uses, is compared with the tile kernel in test_gpu_asm.py)."""
    monkeypatch.setenv("LFSR_ASM", "0")


def solve(L, lf, n, omega=None, **over):
    d = S.SolverDefaults()
    p = L.Params(n_views=lf.n_views, lr_height=lf.y.shape[1], lr_width=lf.y.shape[2], scale=lf.scale,
                 ref_view=lf.ref_view, nltv_radius=d.radius, lambda1=d.lambda1, lambda2=d.lambda2,
                 lambda_reg=d.lambda_reg, sigma_s=d.sigma_s, sigma_e=d.sigma_e, sigma_o1=d.sigma_o1,
                 sigma_o2=d.sigma_o2, theta=d.theta, cg_max_iters=d.cg_max_iters, cg_tol=d.cg_tol, **over)
    s = L.Solver(p)
    s.set_observations(lf.y, lf.view_offsets, lf.omega if omega is None else omega)
    xs = [s.get_hr()]
    stats = []
    for _ in range(n):
        stats += s.admm_run(1)
        xs.append(s.get_hr())
    st = s.get_state()
    s.close()
    return p, np.array(xs), stats, st


@pytest.mark.parametrize("cfg,nranks,n", [("C1", 2, 6), ("C2", 4, 3), ("C3", 3, 2), ("C4", 4, 2)])
def test_virtual_ranks_match_single_strip(lfsr_mod, cfg, nranks, n):
    lf = S.make_lightfield(cfg)
    p1, xs1, st1, s1 = solve(lfsr_mod, lf, n)
    pn, xsn, stn, sn = solve(lfsr_mod, lf, n, n_ranks=nranks, rank=-1)
    for i in range(n + 1):
        assert rel_l2(xsn[i], xs1[i]) <= 1e-5, (i, rel_l2(xsn[i], xs1[i]))
    for a, b in zip(st1, stn):
        assert a["cg_iters"] == b["cg_iters"]
        assert abs(a["J"] - b["J"]) <= 1e-6 * abs(a["J"])
        assert abs(a["primal_res"] - b["primal_res"]) <= 1e-5 * a["primal_res"]
    assert rel_l2(sn["wA"], s1["wA"]) <= 1e-5
    assert rel_l2(sn["wS"], s1["wS"]) <= 1e-4


def test_virtual_ranks_match_oracle(lfsr_mod):
    import oracle as O
    lf = S.make_lightfield("C1")
    p, xs, stats, st = solve(lfsr_mod, lf, 8, n_ranks=2, rank=-1)
    ora = O.admm(oparams(p), lf.y, lf.view_offsets, lf.omega, 8)
    check_iterates(p, ora, xs, stats, st, lf.x_gt)


def test_virtual_ranks_per_view_maps_and_user_psf(lfsr_mod):
    """The strip decomposition with the NEXT-2 per-view maps and the NEXT-4 user blur kernel:
    every rank holds every omega_k; the kernel radius stays within the halo's R."""
    lf = S.make_lightfield("C2")
    oms = S.per_view_disparity(lf.omega, lf.n_views, amp=0.2, seed=4)
    for kw in (dict(omega=oms), dict(psf=S.motion_psf(5, 45.0))):
        _, xs1, st1, _ = solve(lfsr_mod, lf, 2, **kw)
        _, xsn, stn, _ = solve(lfsr_mod, lf, 2, n_ranks=3, rank=-1, **kw)
        for i in range(3):
            assert rel_l2(xsn[i], xs1[i]) <= 1e-5, (kw.keys(), i, rel_l2(xsn[i], xs1[i]))
        for a, b in zip(st1, stn):
            assert a["cg_iters"] == b["cg_iters"] and abs(a["J"] - b["J"]) <= 1e-6 * abs(a["J"])
