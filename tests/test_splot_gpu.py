"""sPlot on the GPU against the reference's contracts (pkg/tests/test_splot.py)
and a brute-force numpy accumulation of the same sums (test-side check)."""

from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _model(hk, n_sig, n_bkg, mean=5.0, sigma=0.5, tau=3.0):
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", mean, step=0.1), hk.Parameter("sigma", sigma, step=0.05, lower=1e-4))
    e = hk.shape_exponential(hk.Parameter("tau", tau, step=0.2, lower=1e-4))
    return hk.add_pdfs([hk.Parameter("n_sig", n_sig, step=60.0, lower=0.0),
                        hk.Parameter("n_bkg", n_bkg, step=80.0, lower=0.0)],
                       [hk.make_pdf(g, hk.gaussian_norm(g), region), hk.make_pdf(e, hk.exponential_norm(e), region)])


@pytest.fixture(scope="module")
def fitted(hk, cuda):
    model = _model(hk, 4000.0, 6000.0)
    data = hk.generate_model_sample(model, hk.RngKey(71, 2))
    res = hk.fit(model, data, ["x0"])
    assert res.status is hk.FitStatus.CONVERGED
    return model, data


def test_single_species_matrix_is_the_yield(hk, cuda):
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 1.0))
    n = hk.Parameter("n", 1000.0, lower=0.0)
    model = hk.add_pdfs([n], [hk.make_pdf(g, hk.gaussian_norm(g), region)])
    data = hk.generate_model_sample(model, hk.RngKey(3, 2), poisson=False)
    hk.fit(model, data, ["x0"])
    V = hk.splot_matrix(model, data, ["x0"])
    assert V.shape == (1, 1) and V[0, 0] == pytest.approx(n.value, rel=1e-9)
    table = hk.splot_weights(model, data, ["x0"], V)
    assert np.max(np.abs(np.asarray(table.column("sw_n")) - 1.0)) < 1e-9


def test_matrix_matches_bruteforce_and_is_symmetric(hk, fitted):
    model, data = fitted
    V = hk.splot_matrix(model, data, ["x0"])
    x = np.asarray(data.column("x0"))
    p = np.stack([pdf.value((x,)) for _, pdf in model.components], axis=1)
    dens = p @ np.array([y.value for y, _ in model.components])
    ref = np.linalg.inv((p / dens[:, None]).T @ (p / dens[:, None]))
    assert np.max(np.abs((V - ref) / ref)) < 1e-8
    assert abs(V[0, 1] - V[1, 0]) <= 1e-10 * abs(V[0, 1])


def test_weights_sum_to_one_and_to_the_yields(hk, fitted):
    model, data = fitted
    V = hk.splot_matrix(model, data, ["x0"])
    t = hk.splot_weights(model, data, ["x0"], V)
    assert t.schema.names == ("sw_n_sig", "sw_n_bkg")
    s, b = np.asarray(t.column("sw_n_sig")), np.asarray(t.column("sw_n_bkg"))
    ps = model.param_set()
    assert np.max(np.abs(s + b - 1.0)) < 1e-9
    assert abs(np.sum(s) - ps["n_sig"].value) < 1e-6 * ps["n_sig"].value
    assert abs(np.sum(b) - ps["n_bkg"].value) < 1e-6 * ps["n_bkg"].value


def test_rejections(hk, cuda, fitted):
    model, data = fitted
    unfitted = _model(hk, 100.0, 20000.0)
    with pytest.raises(ValueError, match="optimum"):
        hk.splot_matrix(unfitted, data, ["x0"])
    region = hk.BoundedRegion(((0.0, 10.0),))
    g = hk.shape_gaussian(hk.Parameter("mean", 5.0), hk.Parameter("sigma", 1.0))
    pdf = hk.make_pdf(g, hk.gaussian_norm(g), region)
    twins = hk.add_pdfs([hk.Parameter("a", 50.0), hk.Parameter("b", 50.0)], [pdf, pdf])
    x = hk.ColumnStore.from_columns(hk.ColumnSchema.real64("x0"), [np.linspace(3.0, 7.0, 100)])
    with pytest.raises(ValueError):
        hk.splot_matrix(twins, x, ["x0"])
    with pytest.raises(ValueError, match="2x2"):
        hk.splot_weights(model, data, ["x0"], np.eye(3))
    V = hk.splot_matrix(model, data, ["x0"])
    a = hk.splot_weights(model, data, ["x0"], V, workers=1)
    b = hk.splot_weights(model, data, ["x0"], V, workers=8)
    assert np.array_equal(a.column("sw_n_sig"), b.column("sw_n_sig"))
    assert math.isfinite(float(V[0, 0]))
