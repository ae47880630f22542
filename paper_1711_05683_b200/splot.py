"""sPlot unfolding with the data pass on the GPU (reference splot.py:1-117).

V^-1_nj = sum_e pdf_n(x_e) pdf_j(x_e) / density(x_e)^2 is the same ratio
accumulation as the yield polish (hk_yield_partials); the k x k inversion and
the optimum / conditioning checks are host numpy, as in the reference.  The
per-event weights sw_n(e) = sum_j V_nj pdf_j(x_e) / density(x_e) are one
kernel (hk_splot_weights) writing device columns.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from . import _lib
from .fitting import ExtendedModel, _observable, lower_model, ratio_sums
from .store import ColumnSchema, ColumnStore

_STATIONARITY_TOL = 1e-6   # splot.py:30
_CONDITION_LIMIT = 1e12    # splot.py:32


def _density_error(model: ExtendedModel, store: ColumnStore, observable_columns, row: int):
    x = _observable(store, observable_columns, model)
    cell = _lib.empty(1)
    _lib.check(_lib.lib().hk_model_density(_lib.ptr(x[row:row + 1]), 1, lower_model(model),
                                           _lib.ptr(cell), _lib.stream_ptr()), "hk_model_density")
    d = np.float64(float(cell.item()))
    return ValueError(f"model density {d!r} is not positive at event {row}")


def splot_matrix(model: ExtendedModel, store: ColumnStore, observable_columns: Sequence[str],
                 workers: int | None = 1) -> np.ndarray:
    """sWeights covariance matrix V (splot.py:45-87)."""
    g, vinv, bad = ratio_sums(model, store, observable_columns)
    if bad[1] != _lib.HK_NO_BAD_ROW:
        raise _density_error(model, store, observable_columns, bad[1])
    residual = float(np.max(np.abs(g - 1.0)))
    if residual > _STATIONARITY_TOL:
        raise ValueError(f"yields are not at the extended-ML optimum "
                         f"(stationarity residual {residual:.3g}); fit before computing sWeights")
    if np.linalg.cond(vinv) > _CONDITION_LIMIT:
        raise ValueError("accumulated sWeights matrix is numerically singular; "
                         "the model species are degenerate on this data")
    return np.linalg.inv(vinv)


def splot_weights(model: ExtendedModel, store: ColumnStore, observable_columns: Sequence[str],
                  V: np.ndarray, workers: int | None = 1) -> ColumnStore:
    """Per-event sWeights table, columns sw_<species> (splot.py:90-117), on the GPU."""
    k = len(model.components)
    V = np.asarray(V, dtype=float)
    if V.shape != (k, k):
        raise ValueError(f"V must be {k}x{k}, got {V.shape}")
    if k > 4:
        raise NotImplementedError("device sWeights support up to 4 species")
    x = _observable(store, observable_columns, model)
    n = len(store)
    cols = [_lib.empty(n) for _ in range(k)]
    bad = _lib.bad_cells(1)
    vflat = np.ascontiguousarray(V.ravel())
    _lib.check(_lib.lib().hk_splot_weights(_lib.ptr(x), n, lower_model(model),
                                           vflat.ctypes.data_as(_lib.ctypes.POINTER(_lib.ctypes.c_double)),
                                           _lib.ptr_array(cols), _lib.ptr(bad), _lib.stream_ptr()),
               "hk_splot_weights")
    (first,) = _lib.read_bad(bad)
    if first != _lib.HK_NO_BAD_ROW:
        raise _density_error(model, store, observable_columns, first)
    schema = ColumnSchema.real64(*(f"sw_{name}" for name in model.species()))
    return ColumnStore._from_device(schema, cols)
