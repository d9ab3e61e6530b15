"""lfsr_solve_batch (the pipelined serving path: field i+1 staged on a second stream while
field i solves) against one-field-at-a-time solves through set_observations / admm_run /
get_hr, and against the fp64 oracle."""
import numpy as np
import pytest
import torch

import oracle as O
import lfsr_synth as S
from test_gpu_parity import ITER_TOL, oparams, rel_l2

pytestmark = pytest.mark.gpu


def params(L, cfg):
    return L.params_for(S.CONFIGS[cfg], S.SolverDefaults())


@pytest.mark.parametrize("cfg,n_fields,n_iters,asm", [("C1", 4, 5, "0"), ("C3", 2, 2, "0"), ("C1", 4, 5, "1"),
                                                      ("C3", 3, 2, "1")])
def test_batch_matches_single_solves(lfsr_mod, cfg, n_fields, n_iters, asm, monkeypatch):
    """Both CG-operator paths forced (LFSR_ASM): the tile kernel, and the assembled operator, which
    the batch re-assembles per field (its stencil depends on the field's disparity)."""
    monkeypatch.setenv("LFSR_ASM", asm)
    lfs = [S.make_lightfield(cfg, seed=500 + i) for i in range(n_fields)]
    p = params(lfsr_mod, cfg)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    fields = [(pin(lf.y), pin(lf.view_offsets), pin(lf.omega)) for lf in lfs]
    outs = [torch.empty((p.H, p.W), dtype=torch.float32).pin_memory() for _ in lfs]
    with lfsr_mod.Solver(p) as s:
        s.solve_batch(fields, n_iters, outs)
        last = s.get_hr()
        assert s.normal_path["name"] == ("assembled" if asm == "1" else "tile")
    singles = []
    with lfsr_mod.Solver(p) as s:
        for lf in lfs:
            s.set_observations(lf.y, lf.view_offsets, lf.omega)
            s.admm_run(n_iters)
            singles.append(s.get_hr())
    for i in range(n_fields):
        assert rel_l2(outs[i].numpy(), singles[i]) <= 1e-6, (i, rel_l2(outs[i].numpy(), singles[i]))
        if i:
            assert rel_l2(outs[i].numpy(), outs[i - 1].numpy()) > 1e-3   # really different fields
    assert rel_l2(last, singles[-1]) <= 1e-6
    if cfg == "C1":
        ora = O.admm(oparams(p), lfs[2].y, lfs[2].view_offsets, lfs[2].omega, n_iters)
        assert rel_l2(outs[2].numpy(), ora.x_iters[-1]) <= ITER_TOL


def test_batch_rejects_device_arrays(lfsr_mod):
    lf = S.make_lightfield("C1")
    p = params(lfsr_mod, "C1")
    with lfsr_mod.Solver(p) as s:
        with pytest.raises(ValueError):
            s.solve_batch([(torch.from_numpy(lf.y).cuda(), lf.view_offsets, lf.omega)], 2)


@pytest.mark.parametrize("over", [dict(psf="motion"), dict(paper_adjoint=1)], ids=["psf", "paper"])
def test_batch_with_modes(lfsr_mod, over):
    """The serving path with a user blur kernel and with the paper-mode adjoint."""
    kw = dict(over)
    if kw.get("psf") == "motion":
        kw["psf"] = S.motion_psf(5, 45.0)
    lfs = [S.make_lightfield("C1", seed=700 + i) for i in range(3)]
    p = params(lfsr_mod, "C1")
    for k, v in kw.items():
        setattr(p, k, v)
    with lfsr_mod.Solver(p) as s:
        outs = s.solve_batch([(lf.y, lf.view_offsets, lf.omega) for lf in lfs], 3)
    with lfsr_mod.Solver(p) as s:
        for lf, o in zip(lfs, outs):
            s.set_observations(lf.y, lf.view_offsets, lf.omega)
            s.admm_run(3)
            assert rel_l2(o, s.get_hr()) <= 1e-6
