"""Pin P24 of the oracle's user blur kernel (P:L962 'the motion blur can be
modelled by a convolutional kernel as a realization of the linear operator B'; reading A36):
the Gaussian outer product reproduces the default B; the impulse response of an asymmetric
kernel fixes the convolution orientation; B^T is B's transpose; A_k with a kernel is the
literal composition D B W_k.  CPU only."""
import numpy as np

import oracle as O
import lfsr_synth as S
from lfsr_synth import random_instance


def test_P24_user_psf(oracle_lib):
    k = np.random.default_rng(2).uniform(0, 1, (5, 5))
    k /= k.sum()
    x = np.zeros((15, 17))
    x[7, 8] = 1.0
    b = O.apply_Bk(x, k)
    assert np.array_equal(b[5:10, 6:11], k)           # (B x)(Y,X) = sum k[u][v] x(Y-u, X-v)
    xr = np.random.default_rng(3).standard_normal((13, 11))
    tr = np.random.default_rng(4).standard_normal((13, 11))
    lhs, rhs = np.vdot(O.apply_Bk(xr, k), tr), np.vdot(xr, O.apply_Bk(tr, k, transpose=True))
    assert abs(lhs - rhs) <= 1e-13 * max(abs(lhs), 1.0)
    for z in (2, 3):
        y, vo, om, xx = random_instance(80 + z, 3, 6, 7, z)
        taps = O.blur_taps(z)
        Pg = O.Params(n_views=3, lr_h=6, lr_w=7, scale=z, ref_view=1)
        Pk = O.Params(n_views=3, lr_h=6, lr_w=7, scale=z, ref_view=1, psf=np.outer(taps, taps))
        assert np.allclose(O.apply_A(Pk, vo, om, xx), O.apply_A(Pg, vo, om, xx), rtol=0, atol=1e-14)
        r = np.random.default_rng(z).standard_normal((3, 6, 7))
        assert np.allclose(O.apply_AT(Pk, vo, om, r), O.apply_AT(Pg, vo, om, r), rtol=0, atol=1e-14)
        km = S.motion_psf(2 * (len(taps) // 2) + 1).astype(np.float64)
        Pm = O.Params(n_views=3, lr_h=6, lr_w=7, scale=z, ref_view=1, psf=km)
        Am = O.apply_A(Pm, vo, om, xx)
        for v in range(3):
            lit = O.apply_D(O.apply_Bk(O.apply_W(xx, om, vo[v, 0], vo[v, 1]), km), z)
            assert np.allclose(Am[v], lit, rtol=0, atol=1e-14)
        ATm = O.apply_AT(Pm, vo, om, r)
        assert abs(np.vdot(Am, r) - np.vdot(xx, ATm)) <= 1e-12 * abs(np.vdot(Am, r))
