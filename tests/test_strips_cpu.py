"""Host logic of the multi-GPU row-strip decomposition, CPU only.

* the plan of lfsr_strip_plan (the same C++ code the GPU path uses) covers the
  image exactly once and its halos come from the immediate neighbours only;
* a world_size-2 gloo run executes the library's exchange schedule — fill the
  halo rows from the neighbour, apply the operator to the own tiles, fold the
  halo ring back — with the fp64 oracle standing in for the kernels, and
  reproduces the whole-image normal operator; rows outside own +- halo are NaN
  on each rank, so a halo that is one row too thin fails the test.
"""
import math
import os
import socket

import numpy as np
import pytest

import lfsr_synth as S


def _lib():
    from paper_2206_05047_b200 import build, lfsr
    build.build()
    return lfsr


@pytest.mark.parametrize("z,h,nr,shift", [(2, 256, 8, 6), (3, 171, 4, 6), (4, 512, 8, 4), (2, 32, 2, 2), (2, 40, 3, 1)])
def test_plan_covers_image(z, h, nr, shift):
    L = _lib()
    p = L.Params(n_views=81, lr_height=h, lr_width=64, scale=z, ref_view=40, n_ranks=nr, rank=-1)
    plan = L.strip_plan(p, shift)
    assert [s["rank"] for s in plan] == list(range(nr))
    assert plan[0]["hr_row0"] == 0 and plan[-1]["hr_row1"] == h * z
    assert plan[0]["lr_row0"] == 0 and plan[-1]["lr_row1"] == h
    for a, b in zip(plan, plan[1:]):
        assert a["hr_row1"] == b["hr_row0"] and a["tile_row1"] == b["tile_row0"]
        assert b["halo_top"] > 0 and a["halo_bottom"] > 0
        # halos come from the immediate neighbour only
        assert a["hr_row1"] - a["hr_row0"] >= b["halo_top"]
        assert b["hr_row1"] - b["hr_row0"] >= a["halo_bottom"]
    for s in plan:
        assert s["hr_row0"] == s["lr_row0"] * z and s["hr_row1"] == s["lr_row1"] * z
        assert s["hr_row1"] > s["hr_row0"]
    sizes = [s["tile_row1"] - s["tile_row0"] for s in plan]
    assert max(sizes) - min(sizes) <= 1
    assert plan[0]["halo_top"] == 0 and plan[-1]["halo_bottom"] == 0


def test_plan_rejects_thin_strips():
    L = _lib()
    p = L.Params(n_views=9, lr_height=32, lr_width=32, scale=2, ref_view=4, n_ranks=3, rank=-1)
    with pytest.raises(L.LFSRError):
        L.strip_plan(p, 2)
    p = L.Params(n_views=9, lr_height=64, lr_width=32, scale=2, ref_view=4, n_ranks=4, rank=-1)
    with pytest.raises(L.LFSRError):   # 32-row strips, halo 2 + 40 + 1 rows
        L.strip_plan(p, 40)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    import oracle as O
    L = _lib()
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    try:
        nv, h, w, z = 9, 48, 20, 2
        y, vo, om, _ = S.random_instance(3, nv, h, w, z, grid=3)
        g = np.random.default_rng(11)
        pvec = g.standard_normal((h * z, w * z))
        m = np.abs(g.standard_normal((h * z, w * z))) * 0.1
        P = O.Params(n_views=nv, lr_h=h, lr_w=w, scale=z, ref_view=4, radius=2, lambda1=1.0, lambda2=2.0, theta=1.5)
        shift = int(math.ceil(float(np.abs(vo[:, 1]).max()) * float(np.abs(om).max())))
        lp = L.Params(n_views=nv, lr_height=h, lr_width=w, scale=z, ref_view=4, n_ranks=world, rank=rank,
                      nccl_unique_id=b"\0" * 128)
        plan = L.strip_plan(lp, shift)
        me = plan[rank]
        top = max(s["halo_top"] for s in plan)
        bot = max(s["halo_bottom"] for s in plan)
        Y0, Y1 = me["hr_row0"], me["hr_row1"]
        H = h * z

        # --- fill: own rows exact, halos from the neighbours, everything else NaN
        loc = np.full_like(pvec, np.nan)
        loc[Y0:Y1] = pvec[Y0:Y1]
        reqs = []
        if rank > 0:   # send my first `bot` rows (the previous strip's lower halo), receive my upper halo
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(loc[Y0:Y0 + bot])), rank - 1))
            buf_up = torch.empty((top, pvec.shape[1]), dtype=torch.float64)
            reqs.append(dist.irecv(buf_up, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(loc[Y1 - top:Y1])), rank + 1))
            buf_dn = torch.empty((bot, pvec.shape[1]), dtype=torch.float64)
            reqs.append(dist.irecv(buf_dn, rank + 1))
        for r_ in reqs:
            r_.wait()
        if rank > 0:
            loc[Y0 - top:Y0] = buf_up.numpy()
        if rank + 1 < world:
            loc[Y1:Y1 + bot] = buf_dn.numpy()

        # --- the own tiles' share of M p: data term from the own LR rows, NLTV on own pixels
        a = O.apply_A(P, vo, om, np.nan_to_num(loc, nan=1e300))   # a poisoned value leaks into any LR row
        l0, l1 = me["lr_row0"], me["lr_row1"]                       # that reads outside own +- halo
        assert np.all(np.abs(a[:, l0:l1]) < 1e100), "halo too thin for the forward operator"
        rho = np.zeros_like(a)
        rho[:, l0:l1] = a[:, l0:l1]
        cA = P.lambda2 + 0.5 * P.theta * P.lambda1 ** 2
        contrib = cA * O.apply_AT(P, vo, om, rho)
        sp = O.apply_S(np.nan_to_num(loc, nan=1e300), m, 2, P.sigma_s)
        sown = np.zeros_like(sp)
        sown[:, Y0:Y1] = sp[:, Y0:Y1]
        assert np.all(np.abs(sown) < 1e100), "halo too thin for the NLTV stencil"
        contrib += 0.5 * P.theta * O.apply_ST(sown, m, 2, P.sigma_s)
        lo, hi = max(Y0 - top, 0), min(Y1 + bot, H)
        assert np.all(contrib[:lo] == 0) and np.all(contrib[hi:] == 0), "contribution outside own +- halo"

        # --- fold: ring rows go to the neighbours
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(contrib[Y0 - top:Y0])), rank - 1))
            r_up = torch.empty((bot, pvec.shape[1]), dtype=torch.float64)
            reqs.append(dist.irecv(r_up, rank - 1))
        if rank + 1 < world:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(contrib[Y1:Y1 + bot])), rank + 1))
            r_dn = torch.empty((top, pvec.shape[1]), dtype=torch.float64)
            reqs.append(dist.irecv(r_dn, rank + 1))
        for r_ in reqs:
            r_.wait()
        own = contrib[Y0:Y1].copy()
        if rank > 0:
            own[:bot] += r_up.numpy()
        if rank + 1 < world:
            own[Y1 - top - Y0:] += r_dn.numpy()
        ref = O.normal(P, vo, om, m, pvec)[Y0:Y1]
        err = float(np.abs(own - ref).max() / np.abs(ref).max())
        # scalars: <p, Mp> partials sum to the global value (the library's allreduce)
        part = torch.tensor([float(np.vdot(pvec[Y0:Y1], own))], dtype=torch.float64)
        dist.all_reduce(part)
        full = float(np.vdot(pvec, O.normal(P, vo, om, m, pvec)))
        out[rank] = (err, abs(part.item() - full) / abs(full))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_exchange_schedule():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        err, serr = out[r]
        assert err < 1e-12, (r, err)
        assert serr < 1e-12, (r, serr)
