"""zdc_fold_weights (host fp64, library) vs the oracle fold (NumPy LAPACK SVD).  Independent
implementations (TSQR + one-sided Jacobi vs LAPACK gesdd); R compared after canonical signs on
the separated synthetic spectra (reading c5), tolerance 1e-10 (north star)."""
import numpy as np
import pytest

import oracle as O
import paper_2408_04107_b200 as zdc
import zdc_synth as Z
from zdc_synth import Dims


@pytest.mark.parametrize("dims,n_calib", [(Z.dims_of(1), 512), (Dims(1, 128, 4, 2, 32), 300),
                                          (Dims(1, 256, 8, 1, 64), 200), (Dims(1, 64, 2, 2, 32), 24)])
def test_fold_matches_oracle(dims, n_calib):
    w = Z.layer_weights(dims, 1, 0)
    xc = Z.calibration(dims, 1, 0, n_calib)
    lib = zdc.fold_weights(dims, w.wq, w.wk, w.wv, w.wo, xc)
    ref = O.fold_layer(dims, w.wq, w.wk, w.wv, w.wo, xc)
    for key in ("sigma_qk", "sigma_vl"):
        assert np.max(np.abs(lib[key] - ref[key])) <= 1e-10 * np.max(ref[key]), key
    for key in ("r_qk", "r_vl"):
        assert np.max(np.abs(lib[key] - ref[key])) <= 1e-10, (key, np.max(np.abs(lib[key] - ref[key])))
    for key in ("wq_f", "wk_f", "wv_f", "wo_f"):
        assert np.max(np.abs(lib[key] - ref[key])) <= 1e-10 * np.max(np.abs(ref[key])), key
    dh = dims.d_head
    for g in range(dims.n_kv_heads):
        assert np.max(np.abs(lib["r_qk"][g].T @ lib["r_qk"][g] - np.eye(dh))) <= 1e-10


def test_fold_identity_case():
    """P10 through the library: diagonal calibration Gram with distinct entries -> R = I."""
    dims = Dims(1, 16, 2, 1, 8)
    d, dh, n = 16, 8, 64
    q, _ = np.linalg.qr(np.random.default_rng(5).standard_normal((n, d)))
    xc = np.sqrt(n) * q
    E = np.vstack([np.eye(dh), np.zeros((d - dh, dh))])
    c = np.linspace(2.0, 0.5, dh)
    wq = np.hstack([0.9 * E @ np.diag(c), 0.7 * E @ np.diag(c)])
    wk = 1.1 * E @ np.diag(c)
    wv = E @ np.diag(np.linspace(1.5, 0.3, dh))
    wo = np.vstack([np.diag(np.linspace(1.2, 0.2, dh)) @ E.T] * 2)
    f = zdc.fold_weights(dims, wq, wk, wv, wo, xc)
    assert np.max(np.abs(f["r_qk"][0] - np.eye(dh))) <= 1e-14
    assert np.max(np.abs(f["r_vl"][0] - np.eye(dh))) <= 1e-14
    assert np.max(np.abs(f["wo_f"] - wo)) <= 1e-14


def test_fold_errors():
    dims = Dims(1, 16, 2, 2, 8)
    w = Z.layer_weights(dims, 1, 0)
    with pytest.raises(zdc.ZdcError) as e:
        zdc.fold_weights(dims, w.wq, w.wk, w.wv, w.wo, np.ones((3, 16)))
    assert e.value.status == -2
    bad = w.wq.copy()
    bad[0, 0] = np.nan
    with pytest.raises(zdc.ZdcError) as e:
        zdc.fold_weights(dims, bad, w.wk, w.wv, w.wo, np.ones((16, 16)))
    assert e.value.status == -1
