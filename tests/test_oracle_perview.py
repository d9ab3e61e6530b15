"""Pin P22 of the oracle's per-view disparity mode (P:L580-582 'for each
perspective theta_k, we need to find the disparity map omega_k'; reading A34 in DESIGN.md §3).

* equal maps omega_k = omega reproduce the shared mode exactly (the pinned A12 special case);
* view k of the per-view stack equals the shared-mode operator run with omega_k as the shared
  map (catches a view using another view's map or a q-vs-p stride in the map stack);
* the exact adjoint: <A x, r> = <x, A^T r> in per-view mode;
* the occlusion weight w_o uses the reference view's map omega_0 (the map on theta_0's grid).
CPU only."""
import numpy as np

import oracle as O
from lfsr_synth import random_instance


def per_view_maps(om, nv, seed):
    g = np.random.default_rng(seed)
    return np.stack([np.clip(om + 0.3 * g.standard_normal(om.shape), -1.5, 1.5) for _ in range(nv)])


def test_P22_per_view_disparity(oracle_lib):
    nv, h, w, z = 4, 6, 7, 2
    y, vo, om, x = random_instance(71, nv, h, w, z)
    kw = dict(n_views=nv, lr_h=h, lr_w=w, scale=z, ref_view=2)
    Ps, Pv = O.Params(**kw), O.Params(disp_per_view=1, **kw)
    # equal maps == shared mode
    same = np.stack([om] * nv)
    assert np.array_equal(O.apply_A(Pv, vo, same, x), O.apply_A(Ps, vo, om, x))
    r = np.random.default_rng(1).standard_normal((nv, h, w))
    assert np.array_equal(O.apply_AT(Pv, vo, same, r), O.apply_AT(Ps, vo, om, r))
    # view k uses omega_k
    oms = per_view_maps(om, nv, 5)
    Av = O.apply_A(Pv, vo, oms, x)
    ATv = O.apply_AT(Pv, vo, oms, r)
    at_sum = np.zeros_like(ATv)
    for k in range(nv):
        P1 = O.Params(n_views=1, lr_h=h, lr_w=w, scale=z, ref_view=0)
        assert np.array_equal(Av[k], O.apply_A(P1, vo[k:k + 1], oms[k], x)[0])
        at_sum += O.apply_AT(P1, vo[k:k + 1], oms[k], r[k:k + 1])
    assert np.allclose(ATv, at_sum, rtol=0, atol=1e-13)
    # adjoint identity
    lhs, rhs = float(np.vdot(Av, r)), float(np.vdot(x, ATv))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)
    # w_o from omega_0 (the reference view's map)
    wo_v, b_v, p_v = O.setup_wo(Pv, y, vo, oms)
    wo_s, b_s, p_s = O.setup_wo(Ps, y, vo, oms[Pv.ref_view])
    assert np.array_equal(wo_v, wo_s) and np.array_equal(p_v, p_s)
    # a whole ADMM iterate is consistent with the equal-maps special case
    a = O.admm(Pv, y, vo, same, 2)
    b = O.admm(Ps, y, vo, om, 2)
    assert np.array_equal(a.x_iters, b.x_iters)
