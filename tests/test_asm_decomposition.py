"""CPU check of the algebra behind the assembled data operator (reading A39), in
fp64 numpy, against the fp64 oracle's normal operator:

    c_A sum_k A_k^T A_k p  =  sum_h st[h] . p(. + d_h)  +  sum_{h>0} st[h](. - d_h) p(. - d_h)
                              + c_A sum_{irregular (k,i)} a_{k,i} (a_{k,i} . p)

where a_{k,i} = sum_{u,v} g[u] g[v] bil_k(zeta i + (u, v)) is the row of the stacked A (positions
outside Omega dropped, A11; bilinear sample at z + dtheta_k omega(z), replicate-clamped, A12/A13),
a row is regular when its cells fit a (2R+2)^2 window, and st[h][a] = c_A sum_{regular} a[a] a[a+d_h]
over the stored half window d_h (dy = 0, dx >= 0, or dy > 0).  The rows are built here from the
paper's definitions (not from the CUDA path, which this file does not import); the oracle supplies
the operator they must reproduce (with m = 0 its NLTV term vanishes).
"""
import numpy as np
import pytest

import oracle as O
import lfsr_synth as S


def rows_of(P, view_offsets, omega):
    """Every row a_{k,i} as (cells, weights) in fp64, from P:L577-583 / A11-A14."""
    z, H, W, h, w = P.scale, P.H, P.W, P.lr_h, P.lr_w
    g = O.blur_taps(z)
    R = (len(g) - 1) // 2
    rows = []
    for k in range(P.n_views):
        drho, dtau = float(view_offsets[k][0]), float(view_offsets[k][1])
        for iy in range(h):
            for ix in range(w):
                acc = {}
                for u in range(-R, R + 1):
                    Y = z * iy + u
                    if not 0 <= Y < H:
                        continue
                    for v in range(-R, R + 1):
                        X = z * ix + v
                        if not 0 <= X < W:
                            continue
                        o = float(omega[Y, X])
                        sy = min(max(Y + dtau * o, 0.0), H - 1.0)
                        sx = min(max(X + drho * o, 0.0), W - 1.0)
                        y0, x0 = int(np.floor(sy)), int(np.floor(sx))
                        y1, x1 = min(y0 + 1, H - 1), min(x0 + 1, W - 1)
                        fy, fx = sy - y0, sx - x0
                        gg = g[u + R] * g[v + R]
                        for (yy, xx, wt) in ((y0, x0, (1 - fy) * (1 - fx)), (y0, x1, (1 - fy) * fx),
                                             (y1, x0, fy * (1 - fx)), (y1, x1, fy * fx)):
                            acc[(yy, xx)] = acc.get((yy, xx), 0.0) + gg * wt
                rows.append(acc)
    return rows, R


def split_apply(P, rows, R, p):
    """The decomposition: half stencil of the regular rows + the irregular rows as rows."""
    H, W = P.H, P.W
    cA = P.lambda2 + 0.5 * P.theta * P.lambda1 ** 2
    WRr, SR = 2 * R + 2, 2 * R + 1
    NSW = 2 * SR + 1
    NH = (NSW * NSW + 1) // 2
    st = np.zeros((NH, H, W))
    irregular = []
    for acc in rows:
        ys = [c[0] for c in acc]
        xs = [c[1] for c in acc]
        if max(ys) - min(ys) < WRr and max(xs) - min(xs) < WRr:
            for (ay, ax), wa in acc.items():
                for (by, bx), wb in acc.items():
                    dy, dx = by - ay, bx - ax
                    if dy < 0 or (dy == 0 and dx < 0):
                        continue                      # the other half: read at the neighbour
                    assert abs(dy) <= SR and abs(dx) <= SR
                    st[dy * NSW + dx, ay, ax] += cA * wa * wb
        else:
            irregular.append(acc)
    q = np.zeros((H, W))
    pad = SR
    pp = np.pad(p, pad)
    for hh in range(NH):
        dy = (hh + SR) // NSW
        dx = hh - dy * NSW
        q += st[hh] * pp[pad + dy:pad + dy + H, pad + dx:pad + dx + W]          # M[a][a + d] p(a + d)
        if hh > 0:                                                              # M[a][a - d] = st[h][a - d]
            sh = np.pad(st[hh], pad)[pad - dy:pad - dy + H, pad - dx:pad - dx + W]
            q += sh * pp[pad - dy:pad - dy + H, pad - dx:pad - dx + W]
    for acc in irregular:
        t = cA * sum(wt * p[c] for c, wt in acc.items())
        for c, wt in acc.items():
            q[c] += t * wt
    return q, len(irregular)


@pytest.mark.parametrize("seed,nv,h,w,z", [(21, 9, 10, 13, 2), (22, 9, 8, 9, 3), (23, 4, 6, 7, 4)])
def test_assembled_split_reproduces_normal_operator(seed, nv, h, w, z):
    y, vo, om, _ = S.random_instance(seed, nv, h, w, z, grid=3 if nv == 9 else None)
    P = O.Params(n_views=nv, lr_h=h, lr_w=w, scale=z, ref_view=nv // 2)
    rows, R = rows_of(P, vo, om)
    p = np.random.default_rng(seed).uniform(-1, 1, (P.H, P.W))
    q, n_irr = split_apply(P, rows, R, p)
    ref = O.normal(P, vo, om, np.zeros((P.H, P.W)), p)     # m = 0: the data part c_A sum A^T A p
    err = np.linalg.norm(q - ref) / np.linalg.norm(ref)
    print("zeta %d: %d of %d rows irregular, rel err %.2e" % (z, n_irr, len(rows), err))
    assert 0 < n_irr < len(rows)      # the instance exercises both parts (a depth edge, A11 borders)
    assert err < 1e-12
