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
from .fitting import (DENSITY, DIV0, ExtendedModel, _closed_form, _density_at, _observables, fcn_exception,
                      first_problem, lower_density, lower_model, ratio_sums)
from .store import ColumnSchema, ColumnStore

_STATIONARITY_TOL = 1e-6   # splot.py:30
_CONDITION_LIMIT = 1e12    # splot.py:32


def _density_error(model: ExtendedModel, store: ColumnStore, observable_columns, row: int):
    obs = _observables(store, observable_columns, model)
    if _closed_form(model):
        cell = _lib.empty(1)
        _lib.check(_lib.lib().hk_model_density(_lib.ptr(obs[0][row:row + 1]), 1, lower_model(model),
                                               _lib.ptr(cell), _lib.stream_ptr()), "hk_model_density")
        d = np.float64(float(cell.item()))
    else:
        d = _density_at(lower_density(model), obs, row)
    return ValueError(f"model density {d!r} is not positive at event {row}")


def _raise_first(model, store, observable_columns, div0_row: int, bad_row: int) -> None:
    problem = first_problem(div0_row, bad_row)
    if problem is None:
        return
    row, kind = problem
    if kind == DIV0:
        obs = _observables(store, observable_columns, model)
        raise fcn_exception(row, DIV0, tuple(np.float64(float(c[row])) for c in obs))
    assert kind == DENSITY
    raise _density_error(model, store, observable_columns, row)


def splot_matrix(model: ExtendedModel, store: ColumnStore, observable_columns: Sequence[str],
                 workers: int | None = 1) -> np.ndarray:
    """sWeights covariance matrix V (splot.py:45-87)."""
    g, vinv, bad = ratio_sums(model, store, observable_columns)
    _raise_first(model, store, observable_columns, bad[2], bad[1])
    residual = float(np.max(np.abs(g - 1.0)))
    if residual > _STATIONARITY_TOL:
        raise ValueError(f"yields are not at the extended-ML optimum "
                         f"(stationarity residual {residual:.3g}); fit before computing sWeights")
    if np.linalg.cond(vinv) > _CONDITION_LIMIT:
        raise ValueError("accumulated sWeights matrix is numerically singular; "
                         "the model species are degenerate on this data")
    return np.linalg.inv(vinv)


def _weights_passes(model: ExtendedModel, obs, n: int, V: np.ndarray, cols: list) -> list:
    """sWeights for more species than one pass pins: per block of up to
    HK_MAX_COMPONENTS - 1 species s (fewer when the numerators would exceed a
    program's HK_MAX_PROGRAM ops), a pass whose slot 0 is the density and
    whose further slots are the numerators sum_j V[s, j] pdf_j, accumulated
    left to right as hk_splot_weights_program does (splot.py:114); an
    identity V' then writes numerator / density.  Slot 0's output goes to a
    scratch column.  Returns the first-bad rows of the first pass."""
    from .fitting import _lower_pass
    k = len(model.components)
    B = _lib.HK_MAX_COMPONENTS - 1
    scratch = _lib.empty(n)
    flags = None
    a = 0
    while a < k:
        species = list(range(a, min(a + B, k)))

        def numerators(pdfs, species=species):
            out = []
            for s in species:
                num = None
                for j in range(k):
                    term = ("mul", pdfs[j], ("const", float(V[s, j])))
                    num = term if num is None else ("add", num, term)
                out.append(num)
            return out

        try:
            dm = _lower_pass(model, numerators)
        except NotImplementedError:
            if B == 1:                  # one numerator does not fit a program
                raise
            B //= 2                     # fewer numerators per pass (HK_MAX_PROGRAM ops)
            continue
        a += len(species)
        Kp = dm.n_comp
        ident = np.zeros((Kp, Kp))
        ident[1:, 1:] = np.eye(Kp - 1)
        vflat = np.ascontiguousarray(ident.ravel())
        vptr = vflat.ctypes.data_as(_lib.ctypes.POINTER(_lib.ctypes.c_double))
        bad = _lib.bad_cells(3)
        _lib.check(_lib.lib().hk_splot_weights_program(_lib.ptr_array(obs), n, dm, vptr,
                                                       _lib.ptr_array([scratch] + [cols[s] for s in species]),
                                                       _lib.ptr(bad), _lib.stream_ptr()),
                   "hk_splot_weights_program")
        got = _lib.read_bad(bad)
        flags = got if flags is None else flags
    return flags


def splot_weights(model: ExtendedModel, store: ColumnStore, observable_columns: Sequence[str],
                  V: np.ndarray, workers: int | None = 1) -> ColumnStore:
    """Per-event sWeights table, columns sw_<species> (splot.py:90-117), on the GPU."""
    k = len(model.components)
    V = np.asarray(V, dtype=float)
    if V.shape != (k, k):
        raise ValueError(f"V must be {k}x{k}, got {V.shape}")
    obs = _observables(store, observable_columns, model)
    n = len(store)
    cols = [_lib.empty(n) for _ in range(k)]
    vflat = np.ascontiguousarray(V.ravel())
    vptr = vflat.ctypes.data_as(_lib.ctypes.POINTER(_lib.ctypes.c_double))
    if k > _lib.HK_MAX_COMPONENTS:
        flags = _weights_passes(model, obs, n, V, cols)
    elif _closed_form(model) and k <= 4:
        bad = _lib.bad_cells(1)
        _lib.check(_lib.lib().hk_splot_weights(_lib.ptr(obs[0]), n, lower_model(model), vptr,
                                               _lib.ptr_array(cols), _lib.ptr(bad), _lib.stream_ptr()),
                   "hk_splot_weights")
        flags = [_lib.HK_NO_BAD_ROW, *_lib.read_bad(bad), _lib.HK_NO_BAD_ROW]
    else:
        bad = _lib.bad_cells(3)
        _lib.check(_lib.lib().hk_splot_weights_program(_lib.ptr_array(obs), n, lower_density(model), vptr,
                                                       _lib.ptr_array(cols), _lib.ptr(bad), _lib.stream_ptr()),
                   "hk_splot_weights_program")
        flags = _lib.read_bad(bad)
    _raise_first(model, store, observable_columns, flags[2], flags[1])
    schema = ColumnSchema.real64(*(f"sw_{name}" for name in model.species()))
    return ColumnStore._from_device(schema, cols)
